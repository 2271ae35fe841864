import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from paper_2112_05682_b200 import _lib, api
lib = ctypes.CDLL(sys.argv[1])
for name, (res, args) in _lib.SIGNATURES.items():
    f = getattr(lib, name); f.restype = res; f.argtypes = args
_lib._lib = lib
q = torch.empty((1, 16384, 16, 64), dtype=torch.bfloat16, device="cuda")
k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
for t, tid in ((q, 1), (k, 2), (v, 3), (do, 4)): api.mea_fill_synthetic(t, 0, tid)
out, lse = api.mea_attention_fwd(q, k, v, want_lse=True)
dq = torch.zeros_like(q)
for _ in range(2): api.mea_attention_bwd(q, k, v, out, do, lse=lse, dq=dq)
torch.cuda.synchronize()
ts = dq.view(torch.int64).flatten()[:2*16*8].cpu().numpy().reshape(2, 16, 8).astype(np.int64)
base = ts[0, 0, 0]
names = ["wait_S", "ld", "compute", "wait_dsfree", "store+arrive"]
for g in range(2):
    for i in range(4):
        r = ts[g, i, :6] - base
        print(f"colhalf{g} t={i+8}", " ".join(f"{x:7d}" for x in r), "| dt:", " ".join(f"{n}={x}" for n, x in zip(names, np.diff(r))))
