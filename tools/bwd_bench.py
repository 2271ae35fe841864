"""Time backward variants (separate .so builds, tools/build_variant.sh) at configs[3] (B=1, H=16,
n=16384, d=64 bf16, lse given). Calls are interleaved variant by variant so every variant sees
the same clock / power state; gradients are compared with the first variant's (experiments only;
parity is tests/).

    ITERS=30 python tools/bwd_bench.py exp_so/exp_a.so exp_so/exp_b.so [...]
"""
import ctypes, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_05682_b200 import _lib, api

libs = sys.argv[1:]
q = torch.empty((1, 16384, 16, 64), dtype=torch.bfloat16, device="cuda")
k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
for t, tid in ((q, 1), (k, 2), (v, 3), (do, 4)): api.mea_fill_synthetic(t, 0, tid)
out, lse = api.mea_attention_fwd(q, k, v, want_lse=True)
fns = {}
for path in libs:
    lib = ctypes.CDLL(path)
    for name, (r, args) in _lib.SIGNATURES.items():
        if not hasattr(lib, name): continue
        f = getattr(lib, name); f.restype = r; f.argtypes = args
    fns[path] = lib
grads = {p: tuple(torch.empty_like(q) for _ in range(3)) for p in libs}
res = {p: [] for p in libs}
ITERS = int(os.environ.get("ITERS", "30"))
for i in range(ITERS + 2):
    for path in libs:
        _lib._lib = fns[path]
        dq, dk, dv = grads[path]
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        fn = api.mea_attention_bwd_deterministic if os.environ.get("DET") == "1" else api.mea_attention_bwd
        e0.record(); fn(q, k, v, out, do, lse=lse, dq=dq, dk=dk, dv=dv); e1.record()
        torch.cuda.synchronize()
        if i >= 2: res[path].append(e0.elapsed_time(e1))
ref = [x.float() for x in grads[libs[0]]]
for path in libs[1:]:
    g = [x.float() for x in grads[path]]
    print(f"{os.path.basename(path)}: max|diff| vs first dq {(g[0]-ref[0]).abs().max().item():.3e} "
          f"dk {(g[1]-ref[1]).abs().max().item():.3e} dv {(g[2]-ref[2]).abs().max().item():.3e}")
base = statistics.median(res[libs[0]])
for path, ts in res.items():
    ms = statistics.median(ts)
    print(f"{os.path.basename(path):24s} bwd {ms:.3f} ms (min {min(ts):.3f}, {100 * (ms / base - 1):+.1f}%)  "
          f"{10*16384*16384*64*16/ms/1e9:.1f} TFLOP/s")
