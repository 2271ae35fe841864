"""configs[1] single query (n_k = 2^20, d = 64, bf16): event-timed calls with an L2 flush between
(for ncu launch lists / duration comparison)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_05682_b200 import api
n_k = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
q = torch.empty((1, 1, 64), dtype=torch.bfloat16, device="cuda")
k = torch.empty((1, n_k, 1, 64), dtype=torch.bfloat16, device="cuda")
v = torch.empty_like(k)
for t, tid in ((q, 1), (k, 2), (v, 3)):
    api.mea_fill_synthetic(t, 0, tid)
out = torch.empty((1, 1, 64), dtype=torch.bfloat16, device="cuda")
ws = torch.empty(api.mea_single_query_workspace_size(1, 1, n_k, 64, api.MEA_BF16), dtype=torch.uint8, device="cuda")
flush = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
sink = torch.empty((), device="cuda")
ts = []
for i in range(25):
    torch.sum(flush, dim=0, out=sink)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); api.mea_single_query_fwd(q, k, v, out=out, workspace=ws); e1.record()
    torch.cuda.synchronize()
    if i >= 5:
        ts.append(e0.elapsed_time(e1) * 1e3)
print(f"n_k={n_k}: median {statistics.median(ts):.2f} us, min {min(ts):.2f} us, "
      f"{4 * n_k * 64 / statistics.median(ts) / 1e3:.0f} GB/s")
