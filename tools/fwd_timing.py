"""Per-tile timeline of the d = 64 forward (fwd_db; build with -DMEA_EXP_TIMING, the probes
overwrite lse): CTA 0, the quarter-0 / sub-0 softmax warp of each query tile (lane 0), key tiles
8..23, and the two MMA issuers.

    tools/build_variant.sh ftime -DMEA_EXP_TIMING && python tools/fwd_timing.py exp_so/exp_ftime.so
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
a = lse.view(torch.int64)[0, 0, :1024].cpu().numpy().astype(np.int64)
sw = a[:256].reshape(2, 16, 8)     # softmax: [query tile][t - 8][probe]
iss = a[512:768].reshape(2, 16, 8)  # issuers: [query tile][t - 8][probe]
base = sw[0, 0, 0]
names = ["top", "S_t landed", "compute done", "S_{t+1} prefetched", "P_t stored + arrived"]
idx = [0, 1, 4, 2, 5]
print("softmax (quarter 0, sub 0, lane 0) per tile:", " | ".join(names), "(cycles from base)")
for qt in range(2):
    for i in range(4):
        print(f"  qt{qt} t={i + 8}", " ".join(f"{x - base:7d}" for x in sw[qt, i, idx]))
print("means over 16 tiles: period | ld wait | compute | S_{t+1} wait + prefetch | P store + arrive | loop")
for qt in range(2):
    r = sw[qt, :, idx].astype(np.float64).T
    d = np.diff(r, axis=1).mean(axis=0)
    loop = (r[1:, 0] - r[:-1, 4]).mean()
    print(f"  qt{qt}  {np.diff(r[:, 0]).mean():6.0f} | " + " | ".join(f"{x:5.0f}" for x in d) + f" | {loop:5.0f}")
print("issuer t: p_full(t) seen, PV(t) issued, pv_done(t) seen, QK(t+2) issued")
for qt in range(2):
    for i in range(4):
        print(f"  qt{qt} t={i + 8}", " ".join(f"{x - base:7d}" for x in iss[qt, i, :4]))
