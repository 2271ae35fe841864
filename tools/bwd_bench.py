import ctypes, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_05682_b200 import _lib, api
q = torch.empty((1, 16384, 16, 64), dtype=torch.bfloat16, device="cuda")
k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
for t, tid in ((q, 1), (k, 2), (v, 3), (do, 4)): api.mea_fill_synthetic(t, 0, tid)
out, lse = api.mea_attention_fwd(q, k, v, want_lse=True)
for path in sys.argv[1:]:
    lib = ctypes.CDLL(path)
    for name, (res, args) in _lib.SIGNATURES.items():
        f = getattr(lib, name); f.restype = res; f.argtypes = args
    _lib._lib = lib
    ts = []
    for i in range(8):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); api.mea_attention_bwd(q, k, v, out, do, lse=lse); e1.record()
        torch.cuda.synchronize()
        if i >= 2: ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    print(f"{os.path.basename(path):24s} bwd {ms:.3f} ms  {10*16384*16384*64*16/ms/1e9:.1f} TFLOP/s")
