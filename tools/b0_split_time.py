"""B0 (statistics pass, lse = NULL) vs the forward: per-kernel event times of the backward with
lse recomputed and of the forward at configs[2]/[3] shape.

    python tools/b0_split_time.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, statistics
from paper_2112_05682_b200 import api
q = torch.empty((1, 16384, 16, 64), dtype=torch.bfloat16, device="cuda")
k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
for t, tid in ((q, 1), (k, 2), (v, 3), (do, 4)): api.mea_fill_synthetic(t, 0, tid)
out, lse = api.mea_attention_fwd(q, k, v, want_lse=True)
for _ in range(3): api.mea_attention_bwd(q, k, v, out, do)
torch.cuda.synchronize()
api.profile_enable(True); api.profile_read()
for _ in range(10): api.mea_attention_bwd(q, k, v, out, do)
torch.cuda.synchronize()
p = api.profile_read(); api.profile_enable(False)
for n,(c,ms) in p.items(): print(n, c, ms/c)
api.profile_enable(True); api.profile_read()
for _ in range(10): api.mea_attention_fwd(q, k, v, out=out, lse=lse)
torch.cuda.synchronize()
p = api.profile_read(); api.profile_enable(False)
for n,(c,ms) in p.items(): print(n, c, ms/c)
