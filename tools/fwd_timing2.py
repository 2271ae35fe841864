"""Per-step timeline of the d = 64 forward (fwd_db, 8 softmax warps each alternating both query
tiles; build with -DMEA_EXP_TIMING, the probes overwrite lse): for CTA 0, warps (quarter 0-1,
sub 0-1), key tiles 8..23, both query tiles; plus the two MMA issuers.

    python tools/fwd_timing2.py exp_so/exp_ftime.so
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
sw = a[:1024].reshape(4, 16, 2, 8)    # [quarter*2+sub][t-8][qt][probe]
iss = a[2048:2048 + 256].reshape(2, 16, 8)
base = sw[0, 0, 0, 0]
print("softmax warp (quarter, sub) step (t, qt): start | compute done | ld_wait done | s_full(t+1) seen | arrive done   (cycles from base)")
for w in range(4):
    for i in range(3):
        for qt in range(2):
            r = sw[w, i, qt, :5] - base
            print(f"  q{w//2} s{w%2} t={i+8} qt{qt}", " ".join(f"{x:7d}" for x in r))
print("means over 16 steps per warp: step period (both tiles) | compute | ld_wait | s_full wait | store+arrive | gap to next")
for w in range(4):
    st = sw[w, :, :, :5].astype(np.float64)
    per = np.diff(st[:, 0, 0]).mean()
    comp = (st[:, :, 1] - st[:, :, 0]).mean(); ldw = (st[:, :, 2] - st[:, :, 1]).mean()
    sfw = (st[:, :, 3] - st[:, :, 2]).mean(); arr = (st[:, :, 4] - st[:, :, 3]).mean()
    gap = np.concatenate([st[:, 1, 0] - st[:, 0, 4], st[1:, 0, 0] - st[:-1, 1, 4]]).mean()
    print(f"  q{w//2} s{w%2}  {per:7.0f} | {comp:6.0f} | {ldw:5.0f} | {sfw:5.0f} | {arr:5.0f} | {gap:5.0f}")
print("issuer t: p_full(t) seen, PV(t) issued, pv_done(t) seen, QK(t+2) issued")
for qt in range(2):
    for i in range(4):
        print(f"  qt{qt} t={i+8}", " ".join(f"{x - base:7d}" for x in iss[qt, i, :4]))
