"""Single-query design measurements on the GPU (round 2): the read-only HBM roofline (probe
kernel) vs buffer size, the fused single-query call at configs[1] and n_k sweep, and a decode
batch (B*H = 16 heads x 2^20 keys) under each heads-per-CTA / CTAs-per-SM / L2-hint variant.
Each timing: L2 read-flush, then CUDA events around one call, median of 30."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_05682_b200 import api

flush = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
sink = torch.empty((), device="cuda")


def timeit(fn, iters=30):
    ts = []
    for i in range(iters + 3):
        torch.sum(flush, dim=0, out=sink)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts), min(ts)


res = {"read_probe": [], "sq": [], "decode": []}
big = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
for mb in ((268, 1024, 4096) if "--quick" in sys.argv else (64, 128, 268, 512, 1024, 4096)):
    nb = mb << 20 if mb != 268 else 268435456
    buf = big[:nb]
    for ctas in (148, 296, 592):
        med, mn = timeit(lambda: api.debug_read_probe(buf, ctas))
        res["read_probe"].append({"bytes": nb, "ctas": ctas, "us": med, "gbs": nb / med / 1e3, "gbs_best": nb / mn / 1e3})
        print("read", mb, "MB ctas", ctas, f"{med:.1f} us {nb / med / 1e3:.0f} GB/s (best {nb / mn / 1e3:.0f})", flush=True)
del big

def sq_case(B, H, n_k, label, key):
    q = torch.empty((B, H, 64), dtype=torch.bfloat16, device="cuda")
    k = torch.empty((B, n_k, H, 64), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    for t, tid in ((q, 1), (k, 2), (v, 3)):
        api.mea_fill_synthetic(t, 0, tid)
    out = torch.empty((B, H, 64), dtype=torch.bfloat16, device="cuda")
    nbytes = 2 * B * H * n_k * 64 * 2
    ref = None
    hcs = (1, 2, 4, 8, 16) if H > 1 else (1,)
    variants = [(0, hc, cps, l2) for hc in hcs for cps in (1,) for l2 in (1, 0)]
    for tma, hc, cps, l2 in variants:
        if True:
            if True:
                api.debug_set_option("sq_heads_per_cta", hc)
                api.debug_set_option("sq_ctas_per_sm", cps)
                api.debug_set_option("sq_l2_256", l2)
                ws = torch.empty(api.mea_single_query_workspace_size(B, H, n_k, 64, api.MEA_BF16), dtype=torch.uint8,
                                 device="cuda")
                med, mn = timeit(lambda: api.mea_single_query_fwd(q, k, v, out=out, workspace=ws))
                if ref is None:
                    ref = out.float().clone()
                diff = (out.float() - ref).abs().max().item()
                r = {"label": label, "B": B, "H": H, "n_k": n_k, "tma": tma, "hc": hc, "ctas_per_sm": cps,
                     "l2_256": l2, "us": med, "gbs": nbytes / med / 1e3, "gbs_best": nbytes / mn / 1e3, "diff": diff}
                res[key].append(r)
                print(label, f"tma={tma} hc={hc} cps={cps} l2={l2}: {med:.1f} us {nbytes / med / 1e3:.0f} GB/s "
                      f"(best {nbytes / mn / 1e3:.0f}) diff {diff:.1e}", flush=True)
    api.debug_set_option("sq_heads_per_cta", 0)
    api.debug_set_option("sq_ctas_per_sm", 0)
    api.debug_set_option("sq_l2_256", 1)


for lg in (18, 20, 22, 24):
    sq_case(1, 1, 1 << lg, f"cfg2 n_k=2^{lg}", "sq")
sq_case(1, 16, 1 << 20, "decode B*H=16 n_k=2^20", "decode")
outp = [a for a in sys.argv[1:] if not a.startswith("--")]
json.dump(res, open(outp[0] if outp else "gpurun_out/sq_probe.json", "w"), indent=1)
