import os, sys
sys.path.insert(0, '/root/repo')
import torch
from paper_2112_05682_b200 import api
for d in (64, 128):
    n, H = 16384, 16
    q = torch.empty((1, n, H, d), dtype=torch.bfloat16, device="cuda")
    k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
    for t, tid in ((q, 1), (k, 2), (v, 3), (do, 4)): api.mea_fill_synthetic(t, 0, tid)
    out, lse = api.mea_attention_fwd(q, k, v, want_lse=True)
    for _ in range(2): api.mea_attention_bwd_deterministic(q, k, v, out, do, lse=lse)
    torch.cuda.synchronize()
    api.profile_enable(True); api.profile_read()
    for _ in range(5): api.mea_attention_bwd_deterministic(q, k, v, out, do, lse=lse)
    torch.cuda.synchronize()
    pr = api.profile_read(); api.profile_enable(False)
    print(d, {k: round(ms / c, 3) for k, (c, ms) in pr.items()})
