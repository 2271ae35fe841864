"""Per-tile timeline of the d = 64 forward (fwd_db: Q in TMEM, 64-key tiles; build with
-DMEA_EXP_TIMING, the probes overwrite lse): CTA 0, quarter-0 softmax warps (qt, sub), key
tiles 8..23; plus the two MMA issuers.

    python tools/fwd_timing3.py exp_so/exp_fttq.so
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
a = lse.view(torch.int64)[0, 0, :2048 + 256].cpu().numpy().astype(np.int64)
sw = a[:512].reshape(4, 16, 8)    # [qt*2+sub][t-8][probe]
iss = a[2048:2048 + 256].reshape(2, 16, 8)
base = sw[0, 0, 0]
names = ["top", "s_full", "ld+s_free", "compute", "pv_done", "arrive"]
print("softmax (quarter 0) per tile:", " | ".join(names), "(cycles from base)")
for w in range(4):
    for i in range(3):
        print(f"  qt{w//2} sub{w%2} t={i+8}", " ".join(f"{x - base:7d}" for x in sw[w, i, :6]))
print("means over 16 tiles: period | wait s_full | ld | compute | wait pv_done | store+arrive | loop")
for w in range(4):
    r = sw[w, :, :6].astype(np.float64)
    d = np.diff(r, axis=1).mean(axis=0)
    loop = (r[1:, 0] - r[:-1, 5]).mean()
    print(f"  qt{w//2} sub{w%2}  {np.diff(r[:, 0]).mean():6.0f} | " + " | ".join(f"{x:5.0f}" for x in d) + f" | {loop:5.0f}")
print("issuer t: s_free(t) seen, kv_full(t+2) seen, QK(t+2) issued, p_full(t) seen, fenced, PV(t) issued")
for qt in range(2):
    for i in range(4):
        print(f"  qt{qt} t={i+8}", " ".join(f"{x - base:7d}" for x in iss[qt, i, [0, 4, 1, 2, 5, 3]]))
