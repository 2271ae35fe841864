import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from paper_2112_05682_b200 import _lib, api
lib = ctypes.CDLL(sys.argv[1])
for name, (res, args) in _lib.SIGNATURES.items():
    f = getattr(lib, name); f.restype = res; f.argtypes = args
_lib._lib = lib
q = torch.empty((1, 16384, 16, 64), dtype=torch.bfloat16, device="cuda")
k, v = torch.empty_like(q), torch.empty_like(q)
for t, tid in ((q, 1), (k, 2), (v, 3)): api.mea_fill_synthetic(t, 0, tid)
lse = torch.zeros((1, 16, 16384), dtype=torch.float32, device="cuda")
for _ in range(3): out = api.mea_attention_fwd(q, k, v, lse=lse)
torch.cuda.synchronize()
ts = lse.view(torch.int64)[0, 0, :4*16*8].cpu().numpy().reshape(4, 16, 8).astype(np.int64)
base = ts[0, 0, 0]
names = ["wait_S", "compute", "xchg", "tail", "store+arrive"]
for w in range(4):
    for i in range(4):
        r = ts[w, i, :6] - base
        print(f"qt{w//2} half{w%2} t={i+8}", " ".join(f"{x:7d}" for x in r), "| dt:", " ".join(f"{n}={x}" for n, x in zip(names, np.diff(r))))
