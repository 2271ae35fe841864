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
allts = lse.view(torch.int64)[0, 0, :1024 + 128].cpu().numpy().astype(np.int64)
ts = allts[:512].reshape(4, 16, 8)
its = allts[512:768].reshape(2, 16, 8)
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
print("softmax t: top, s_full(t) seen, compute done, -, p_full arrived")
for w in (0, 2):
    for i in range(4):
        print(f"  qt{w//2} t={i+8}", " ".join(f"{x - base:7d}" for x in ts[w, i, [0, 1, 4, 2, 5]]))
print("issuer t: fwd_sm100a: top, kv_full(t+1), s_loaded(t), QK(t+1) issued, p_full(t), PV(t) issued | fwd_db: p_full(t) seen, PV(t) issued, pv_done(t) seen, QK(t+2) issued")
for qt in range(2):
    for i in range(4):
        print(f"  qt{qt} t={i+8}", " ".join(f"{x - base:7d}" for x in its[qt, i, :6]))
ws = lse.view(torch.int64)[0, 0, 1024:1024 + 128].cpu().numpy().astype(np.int64).reshape(4, 16, 2)
if ws.min() > 0:
    print("per softmax warp (sw 0-7 = qt0, 8-15 = qt1): compute start (after ld wait) / p_full arrive")
    for i in range(4):
        print(f"  t={i+8} start ", " ".join(f"{x - base:6d}" for x in ws[i, :, 1]))
        print(f"  t={i+8} arrive", " ".join(f"{x - base:6d}" for x in ws[i, :, 0]))
