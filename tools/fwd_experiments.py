"""Time forward-kernel variants (built with -D flags into separate .so files) at cfg3."""
import ctypes, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_05682_b200 import _lib, api

libs = sys.argv[1:]
dev = torch.device("cuda", 0)
for H in (16, 1):
    q = torch.empty((1, 16384, H, 64), dtype=torch.bfloat16, device=dev)
    k, v = torch.empty_like(q), torch.empty_like(q)
    for t, tid in ((q, 1), (k, 2), (v, 3)):
        api.mea_fill_synthetic(t, 0, tid)
    out = torch.empty_like(q)
    for path in libs:
        lib = ctypes.CDLL(path)
        for name, (res, args) in _lib.SIGNATURES.items():
            f = getattr(lib, name); f.restype = res; f.argtypes = args
        _lib._lib = lib
        ts = []
        for i in range(12):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); api.mea_attention_fwd(q, k, v, out=out); e1.record()
            torch.cuda.synchronize()
            if i >= 2: ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        print(f"H={H:2d} {os.path.basename(path):30s} {ms:8.3f} ms  {4*16384*16384*64*H/ms/1e9:8.1f} TFLOP/s")
