"""Per-tile softmax timeline of the forward kernel (build with -DMEA_EXP_TIMING; the probes
overwrite lse): for one CTA, query tile qt, row half, key tiles 8..23.

    python tools/fwd_timing.py exp_so/exp_ftime.so
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
q = torch.empty((1, 16384, 16, 64), dtype=torch.bfloat16, device="cuda")
k, v = torch.empty_like(q), torch.empty_like(q)
for t, tid in ((q, 1), (k, 2), (v, 3)): api.mea_fill_synthetic(t, 0, tid)
lse = torch.zeros((1, 16, 16384), dtype=torch.float32, device="cuda")
for _ in range(3): out = api.mea_attention_fwd(q, k, v, lse=lse)
torch.cuda.synchronize()
ts = lse.view(torch.int64)[0, 0, :4*16*8].cpu().numpy().reshape(4, 16, 8).astype(np.int64)
base = ts[0, 0, 0]
for w in range(4):
    for i in range(3):
        r = ts[w, i, [0, 1, 4, 5]] - base
        print(f"qt{w//2} half{w%2} t={i+8}", " ".join(f"{x:7d}" for x in r))
print("means over 16 tiles (cycles):")
for w in range(4):
    r = ts[w, :, [0, 1, 4, 5]].T
    d = np.diff(r, axis=1).mean(axis=0)
    print(f"  qt{w//2} half{w%2} period {np.diff(ts[w, :, 0]).mean():6.0f} | wait_S={d[0]:.0f} "
          f"compute={d[1]:.0f} pv_wait+store+arrive={d[2]:.0f}")
