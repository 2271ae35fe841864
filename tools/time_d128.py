"""Time the d = 128 forward (and d = 64 for comparison) at B=1, H=16, n=16384, bf16."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_05682_b200 import api

flush = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
sink = torch.empty((), device="cuda")
for d in (64, 128):
    n, H = 16384, 16
    q = torch.empty((1, n, H, d), dtype=torch.bfloat16, device="cuda")
    k, v = torch.empty_like(q), torch.empty_like(q)
    for t, tid in ((q, 1), (k, 2), (v, 3)):
        api.mea_fill_synthetic(t, 0, tid)
    out = torch.empty_like(q)
    lse = torch.empty((1, H, n), dtype=torch.float32, device="cuda")
    ts = []
    for i in range(23):
        torch.sum(flush, dim=0, out=sink)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); api.mea_attention_fwd(q, k, v, out=out, lse=lse); e1.record()
        torch.cuda.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    print(f"d={d}: {ms:.3f} ms (min {min(ts):.3f})  {4 * n * n * d * H / ms / 1e9:.1f} TFLOP/s")
