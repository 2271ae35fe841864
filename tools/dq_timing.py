"""Per-tile timeline of the dQ kernel (build with -DMEA_EXP_TIMING; the probes overwrite dq):
one CTA, both column halves, key tiles 8..23, and the means. Usage:
    python tools/dq_timing.py exp_so/exp_t.so [d]
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from paper_2112_05682_b200 import _lib, api
lib = ctypes.CDLL(sys.argv[1])
for name, (res, args) in _lib.SIGNATURES.items():
    if not hasattr(lib, name): continue
    f = getattr(lib, name); f.restype = res; f.argtypes = args
_lib._lib = lib
d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
q = torch.empty((1, 16384, 16, d), dtype=torch.bfloat16, device="cuda")
k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
for t, tid in ((q, 1), (k, 2), (v, 3), (do, 4)): api.mea_fill_synthetic(t, 0, tid)
out, lse = api.mea_attention_fwd(q, k, v, want_lse=True)
dq = torch.zeros_like(q)
for _ in range(2): api.mea_attention_bwd_deterministic(q, k, v, out, do, lse=lse, dq=dq)
torch.cuda.synchronize()
ts = dq.view(torch.int64).flatten()[:2*16*8].cpu().numpy().reshape(2, 16, 8).astype(np.int64)
names = ["wait_S", "ld", "compute", "wait_dsfree", "store+arrive"]
for g in range(2):
    dd = np.diff(ts[g, :, :6], axis=1).mean(axis=0)
    print(f"colhalf{g} period {np.diff(ts[g, :, 0]).mean():6.0f} | " + " ".join(f"{n}={x:.0f}" for n, x in zip(names, dd)))
