"""Per-kernel event times of mea_attention_bwd at configs[3] (library launch profiler)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_05682_b200 import api
q = torch.empty((1, 16384, 16, 64), dtype=torch.bfloat16, device="cuda")
k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
for t, tid in ((q, 1), (k, 2), (v, 3), (do, 4)): api.mea_fill_synthetic(t, 0, tid)
out, lse = api.mea_attention_fwd(q, k, v, want_lse=True)
for _ in range(2): api.mea_attention_bwd(q, k, v, out, do, lse=lse)
torch.cuda.synchronize()
api.profile_enable(True); api.profile_read()
for _ in range(5): api.mea_attention_bwd(q, k, v, out, do, lse=lse)
r = api.profile_read()
for name, (cnt, ms) in sorted(r.items()):
    print(f"{name:16s} {ms / cnt:.3f} ms")
