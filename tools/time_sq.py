"""Time mea_single_query_fwd at configs[1] (n_k = 2^20, d = 64, bf16) end to end (both kernels),
with a read-based L2 flush before every call."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_05682_b200 import api

n_k = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
BH = int(sys.argv[2]) if len(sys.argv) > 2 else 1
q = torch.empty((1, BH, 64), dtype=torch.bfloat16, device="cuda")
k = torch.empty((1, n_k, BH, 64), dtype=torch.bfloat16, device="cuda")
v = torch.empty_like(k)
for t, tid in ((q, 1), (k, 2), (v, 3)):
    api.mea_fill_synthetic(t, 0, tid)
o = torch.empty((1, BH, 64), dtype=torch.bfloat16, device="cuda")
ws = torch.empty(api.mea_single_query_workspace_size(1, BH, n_k, 64, api.MEA_BF16), dtype=torch.uint8, device="cuda")
flush = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
sink = torch.empty((), device="cuda")
ts = []
for i in range(25):
    torch.sum(flush, dim=0, out=sink)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); api.mea_single_query_fwd(q, k, v, out=o, workspace=ws); e1.record()
    torch.cuda.synchronize()
    if i >= 5: ts.append(e0.elapsed_time(e1) * 1e3)
us = statistics.median(ts)
b = 2 * n_k * BH * 64 * 2
print(f"n_k={n_k} BH={BH}: {us:.1f} us  {b / us / 1e3:.0f} GB/s  (min {min(ts):.1f} us)")
