"""fp32 forward: exact SIMT (MEA_F32) vs split-precision tensor cores (MEA_F32_SPLIT), B=1 H=16 d=64."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2112_05682_b200 import api
for n in (1024, 4096, 16384):
    H = 16
    q = torch.randn(1, n, H, 64, device="cuda"); k = torch.randn_like(q); v = torch.randn_like(q)
    out = torch.empty_like(q)
    for split in (False, True):
        if n == 16384 and not split:
            continue   # the SIMT kernel takes ~seconds here
        fn = lambda: api.mea_attention_fwd(q, k, v, out=out, f32_split=split)
        fn(); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        print(f"n={n} {'split TC' if split else 'exact SIMT'}: {ms:.3f} ms  {4 * n * n * 64 * H / ms / 1e9:.1f} TFLOP/s")
