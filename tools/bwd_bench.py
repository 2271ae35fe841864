"""Time backward variants (separate .so builds, tools/build_variant.sh) at configs[3] and compare
their gradients with the first library's (sanity check for experiments; parity is tests/).

    python tools/bwd_bench.py exp_so/exp_base.so exp_so/exp_X.so [...]
"""
import ctypes, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_05682_b200 import _lib, api
q = torch.empty((1, 16384, 16, 64), dtype=torch.bfloat16, device="cuda")
k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
for t, tid in ((q, 1), (k, 2), (v, 3), (do, 4)): api.mea_fill_synthetic(t, 0, tid)
out, lse = api.mea_attention_fwd(q, k, v, want_lse=True)
first = None
res = {p: [] for p in sys.argv[1:]}
for rnd in range(3):
    for path in sys.argv[1:]:
        lib = ctypes.CDLL(path)
        for name, (r, args) in _lib.SIGNATURES.items():
            f = getattr(lib, name); f.restype = r; f.argtypes = args
        _lib._lib = lib
        for i in range(8):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); g = api.mea_attention_bwd(q, k, v, out, do, lse=lse); e1.record()
            torch.cuda.synchronize()
            if i >= 2: res[path].append(e0.elapsed_time(e1))
        if rnd == 0:
            g = [x.float() for x in g]
            if first is None:
                first = g
            else:
                print(f"{os.path.basename(path)}: max|diff| vs first dq {(g[0]-first[0]).abs().max().item():.3e} "
                      f"dk {(g[1]-first[1]).abs().max().item():.3e} dv {(g[2]-first[2]).abs().max().item():.3e}")
for path, ts in res.items():
    ms = statistics.median(ts)
    print(f"{os.path.basename(path):24s} bwd {ms:.3f} ms (min {min(ts):.3f})  {10*16384*16384*64*16/ms/1e9:.1f} TFLOP/s")
