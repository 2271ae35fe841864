import sys, math
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import oracle as O
from tests import helpers as Hh
from paper_2112_05682_b200 import api
for (B, nq, nk, H) in [(1, 1, 1, 1), (1, 1, 300, 1), (1, 128, 128, 1), (1, 128, 1000, 1), (2, 300, 1000, 3)]:
    q, k, v = Hh.host_inputs(B, nq, nk, H, 64, seed=9, dtype="f32")
    for scale in (1/8, 0.5):
        ref, ref_lse = O.mha_forward(q, k, v, scale)
        out, lse = api.mea_attention_fwd(Hh.to_dev(q, torch.float32), Hh.to_dev(k, torch.float32), Hh.to_dev(v, torch.float32), scale=scale, want_lse=True)
        torch.cuda.synchronize()
        e = np.abs(out.double().cpu().numpy() - ref)
        el = np.abs(lse.double().cpu().numpy() - ref_lse)
        print(B, nq, nk, H, scale, f"out err {e.max():.2e} (mean {e.mean():.1e}, |ref| max {np.abs(ref).max():.2f}) lse err {el.max():.2e}")
