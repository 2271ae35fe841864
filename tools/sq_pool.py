"""Single query: static key ranges vs a dynamic pool of CTA-step chunks (knob sq_static_pct),
configs[1] n_k sweep and a decode batch; median of 30 event-timed calls, L2 flushed before each.
Also the timing of an empty launch (the per-call floor).

    python tools/sq_pool.py [out.json]
"""
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


res = []
x = torch.zeros(1, device="cuda")
med, mn = timeit(lambda: x.add_(1))
print(f"tiny torch kernel: {med:.2f} us (min {mn:.2f})")
res.append({"case": "tiny kernel", "us": med})
for B, H, lg in ((1, 1, 18), (1, 1, 20), (1, 1, 22), (1, 1, 24), (1, 16, 20), (4, 8, 16)):
    n_k = 1 << lg
    q = torch.empty((B, H, 64), dtype=torch.bfloat16, device="cuda")
    k = torch.empty((B, n_k, H, 64), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    for t, tid in ((q, 1), (k, 2), (v, 3)):
        api.mea_fill_synthetic(t, 0, tid)
    out = torch.empty((B, H, 64), dtype=torch.float32, device="cuda")
    nbytes = 2 * B * H * n_k * 64 * 2
    ref = None
    for pct in (100, 90, 80, 75, 60, 50, 0):
        api.debug_set_option("sq_static_pct", pct)
        ws = torch.empty(api.mea_single_query_workspace_size(B, H, n_k, 64, api.MEA_BF16), dtype=torch.uint8,
                         device="cuda")
        med, mn = timeit(lambda: api.mea_single_query_fwd(q, k, v, out=out, workspace=ws))
        if ref is None:
            ref = out.clone()
        diff = (out - ref).abs().max().item()
        r = {"B": B, "H": H, "n_k": n_k, "static_pct": pct, "us": med, "us_min": mn, "gbs": nbytes / med / 1e3,
             "diff_vs_static": diff}
        res.append(r)
        print(f"B={B} H={H} n_k=2^{lg} static={pct:3d}%: {med:8.2f} us (min {mn:8.2f}) {nbytes / med / 1e3:6.0f} GB/s "
              f"diff {diff:.1e}", flush=True)
    api.debug_set_option("sq_static_pct", 75)
outp = [a for a in sys.argv[1:] if not a.startswith("--")]
json.dump(res, open(outp[0] if outp else "gpurun_out/sq_pool.json", "w"), indent=1)
