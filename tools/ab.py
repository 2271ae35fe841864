"""Interleaved A/B timing of library builds (tools/build_variant.sh) on one workload at configs[2]'s
shape (B=1, H=16, n=16384, bf16): calls alternate build by build so every build sees the same
clock / power state, with a 512 MiB L2 read-flush before each call; results are compared with the
first build's (experiments only; parity is tests/).

    [COOL_MS=ms] CASE=fwd|fwd_paper|fwd_causal|bwd|bwd_causal|bwd_det|bwd_nolse|fwd128|bwd128|sq|sq16 ITERS=30 python tools/ab.py A.so B.so ...
(sq: configs[1], one query over 2^20 keys; sq16: the 16-head decode batch; TFLOP/s column = GB/s / 1000)
"""
import ctypes, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_05682_b200 import _lib, api

case = os.environ.get("CASE", "fwd")
iters = int(os.environ.get("ITERS", "30"))
cool_ms = float(os.environ.get("COOL_MS", "0"))
libs = sys.argv[1:]
d = 128 if case.endswith("128") else 64
n, H = 16384, 16
q = torch.empty((1, n, H, d), dtype=torch.bfloat16, device="cuda")
k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
for t, tid in ((q, 1), (k, 2), (v, 3), (do, 4)):
    api.mea_fill_synthetic(t, 0, tid)
causal = "causal" in case
fwd = api.mea_attention_fwd_causal if causal else api.mea_attention_fwd
out, lse = fwd(q, k, v, want_lse=True)
flush = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
sink = torch.empty((), device="cuda")
fns = {}
for path in libs:
    lib = ctypes.CDLL(path)
    for name, (r, args) in _lib.SIGNATURES.items():
        if hasattr(lib, name):
            f = getattr(lib, name)
            f.restype, f.argtypes = r, args
    fns[path] = lib
res = {p: [] for p in libs}
outs = {}
vis = (n * (n + 1) / 2) if causal else n * n
flops = (4 if case.startswith("fwd") else 10) * vis * d * H


if case.startswith("sq"):
    hs = 16 if case == "sq16" else 1
    sq_q = torch.empty((1, hs, 64), dtype=torch.bfloat16, device="cuda")
    sq_k = torch.empty((1, 1 << 20, hs, 64), dtype=torch.bfloat16, device="cuda")
    sq_v = torch.empty_like(sq_k)
    for t, tid in ((sq_q, 1), (sq_k, 2), (sq_v, 3)):
        api.mea_fill_synthetic(t, 0, tid)
    sq_ws = torch.empty(api.mea_single_query_workspace_size(1, hs, 1 << 20, 64, api.MEA_BF16), dtype=torch.uint8,
                        device="cuda")
    flops = 2 * hs * (1 << 20) * 64 * 2   # bytes (the column reads GB/s / 1000)


def call():
    if case.startswith("sq"):
        return (api.mea_single_query_fwd(sq_q, sq_k, sq_v, workspace=sq_ws, out_dtype=torch.float32),)
    if case == "fwd_paper":   # configs[2]'s literal schedule: query chunk 1024, key chunk 4096
        return (api.mea_attention_fwd(q, k, v, q_chunk=1024, k_chunk=4096),)
    if case.startswith("fwd"):
        return (fwd(q, k, v),)
    if case == "bwd_nolse":   # lse recomputed by the statistics pass B0
        return api.mea_attention_bwd(q, k, v, out, do)
    bwd = {"bwd": api.mea_attention_bwd, "bwd128": api.mea_attention_bwd, "bwd_det": api.mea_attention_bwd_deterministic,
           "bwd_causal": api.mea_attention_bwd_causal}[case]
    return bwd(q, k, v, out, do, lse=lse)


for i in range(iters + 2):
    for path in libs:
        _lib._lib = fns[path]
        if cool_ms:   # idle before each call: the board leaves its power cap, clocks return to max
            torch.cuda.synchronize()
            time.sleep(cool_ms / 1e3)
        torch.sum(flush, dim=0, out=sink)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        r = call()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            res[path].append(e0.elapsed_time(e1))
        outs[path] = r
ref = outs[libs[0]]
for path in libs[1:]:
    diff = max((a.float() - b.float()).abs().max().item() for a, b in zip(outs[path], ref))
    print(f"{os.path.basename(path)}: max|diff| vs first {diff:.3e}")
base = statistics.median(res[libs[0]])
for path, ts in res.items():
    ms = statistics.median(ts)
    if case.startswith("sq"):   # microsecond calls: the event clock ticks in ~1 us, report the mean too
        print(f"{case:10s} {os.path.basename(path):24s} median {ms * 1e3:.2f} us, mean {statistics.mean(ts) * 1e3:.2f} us "
              f"(min {min(ts) * 1e3:.2f})")
        continue
    print(f"{case:10s} {os.path.basename(path):24s} {ms:.3f} ms (min {min(ts):.3f}, {100 * (ms / base - 1):+.1f}%)  "
          f"{flops / ms / 1e9:.1f} TFLOP/s")
