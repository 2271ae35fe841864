"""Time forward and backward at d = 64 and d = 128 (B=1, H=16, n=16384, bf16, lse given), with a
512 MiB L2 read-flush before each call."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_05682_b200 import api

flush = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
sink = torch.empty((), device="cuda")


def timed(fn, iters=12):
    fn(); fn()
    ts = []
    for _ in range(iters):
        torch.sum(flush, dim=0, out=sink)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), min(ts)


for d in (64, 128):
    n, H = 16384, 16
    q = torch.empty((1, n, H, d), dtype=torch.bfloat16, device="cuda")
    k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
    for t, tid in ((q, 1), (k, 2), (v, 3), (do, 4)):
        api.mea_fill_synthetic(t, 0, tid)
    out = torch.empty_like(q)
    lse = torch.empty((1, H, n), dtype=torch.float32, device="cuda")
    fl = 4 * n * n * d * H
    ms, mn = timed(lambda: api.mea_attention_fwd(q, k, v, out=out, lse=lse))
    print(f"d={d} fwd: {ms:.3f} ms (min {mn:.3f})  {fl / ms / 1e9:.1f} TFLOP/s")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
    ws = torch.empty(api.mea_attention_bwd_workspace_size(1, H, n, n, d, api.MEA_BF16, True), dtype=torch.uint8,
                     device="cuda")
    for name, fn in (("bwd", api.mea_attention_bwd), ("bwd_det", api.mea_attention_bwd_deterministic)):
        ms, mn = timed(lambda: fn(q, k, v, out, do, lse=lse, dq=dq, dk=dk, dv=dv, workspace=ws))
        print(f"d={d} {name}: {ms:.3f} ms (min {mn:.3f})  {2.5 * fl / ms / 1e9:.1f} TFLOP/s")
    del q, k, v, do, out, dq, dk, dv, ws
