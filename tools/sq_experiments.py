"""Time single-query variants (separate .so builds) at configs[1] (n_k = 2^20) and 2^22, interleaved,
L2 read-flush before each call; outputs compared with the first variant."""
import ctypes, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_05682_b200 import _lib, api
libs = sys.argv[1:]
fns = {}
for path in libs:
    lib = ctypes.CDLL(path)
    for name, (r, args) in _lib.SIGNATURES.items():
        if not hasattr(lib, name): continue
        f = getattr(lib, name); f.restype = r; f.argtypes = args
    fns[path] = lib
flush = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
sink = torch.empty((), device="cuda")
for n_k in (1 << 20, 1 << 22):
    q = torch.empty((1, 1, 64), dtype=torch.bfloat16, device="cuda")
    k = torch.empty((1, n_k, 1, 64), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    for t, tid in ((q, 1), (k, 2), (v, 3)): api.mea_fill_synthetic(t, 0, tid)
    outs = {p: torch.empty((1, 1, 64), dtype=torch.bfloat16, device="cuda") for p in libs}
    res = {p: [] for p in libs}
    for it in range(42):
        for path in libs:
            _lib._lib = fns[path]
            torch.sum(flush, dim=0, out=sink)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); api.mea_single_query_fwd(q, k, v, out=outs[path]); e1.record()
            torch.cuda.synchronize()
            if it >= 2: res[path].append(e0.elapsed_time(e1) * 1e3)
    ref = outs[libs[0]].float()
    for path in libs:
        us = statistics.median(res[path])
        print(f"n_k=2^{n_k.bit_length()-1} {os.path.basename(path):20s} {us:7.2f} us  {4 * n_k * 64 / us / 1e3:6.0f} GB/s  "
              f"diff {(outs[path].float() - ref).abs().max().item():.1e}")
