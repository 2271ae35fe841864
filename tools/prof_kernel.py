"""Launch one hot-path call a few times at a BASELINE.json config (for ncu captures).

    python tools/prof_kernel.py fwd|fwd_kc|bwd|sq|fwd128|bwd128|fwd_causal|bwd_causal|sq_batch [--iters N]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2112_05682_b200 import api  # noqa: E402
from synth import gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("what", choices=["fwd", "fwd_kc", "bwd", "sq", "fwd128", "bwd128", "fwd_causal", "bwd_causal", "sq_batch"])
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--n", type=int, default=16384)
a = ap.parse_args()
dev = torch.device("cuda", 0)
H, D = 16, 64
if a.what in ("sq", "sq_batch"):
    hs = 16 if a.what == "sq_batch" else 1   # configs[1] (one head) or the 16-head decode batch
    q = torch.empty((1, hs, D), dtype=torch.bfloat16, device=dev)
    k = torch.empty((1, 1 << 20, hs, D), dtype=torch.bfloat16, device=dev)
    v = torch.empty_like(k)
    for t, tid in ((q, 1), (k, 2), (v, 3)):
        api.mea_fill_synthetic(t, 0, tid)
    for _ in range(a.iters):
        api.mea_single_query_fwd(q, k, v)
elif a.what in ("fwd128", "bwd128"):
    q = torch.empty((1, a.n, H, 128), dtype=torch.bfloat16, device=dev)
    k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
    for t, tid in ((q, 1), (k, 2), (v, 3), (do, 4)):
        api.mea_fill_synthetic(t, 0, tid)
    out, lse = api.mea_attention_fwd(q, k, v, want_lse=True)
    for _ in range(a.iters):
        if a.what == "fwd128":
            api.mea_attention_fwd(q, k, v, out=out, lse=lse)
        else:
            api.mea_attention_bwd(q, k, v, out, do, lse=lse)
else:
    q = torch.empty((1, a.n, H, D), dtype=torch.bfloat16, device=dev)
    k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
    for t, tid in ((q, 1), (k, 2), (v, 3), (do, 4)):
        api.mea_fill_synthetic(t, 0, tid)
    out, lse = api.mea_attention_fwd(q, k, v, want_lse=True)
    for _ in range(a.iters):
        if a.what == "fwd":
            api.mea_attention_fwd(q, k, v, out=out, lse=lse)
        elif a.what == "fwd_causal":
            api.mea_attention_fwd_causal(q, k, v, out=out, lse=lse)
        elif a.what == "bwd_causal":
            api.mea_attention_bwd_causal(q, k, v, out, do, lse=lse)
        elif a.what == "fwd_kc":
            api.mea_attention_fwd(q, k, v, out=out, lse=lse, q_chunk=1024, k_chunk=4096)
        else:
            api.mea_attention_bwd(q, k, v, out, do, lse=lse)
torch.cuda.synchronize()
print("ok")
