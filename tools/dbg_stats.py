"""Debug: the B0 statistics pass's lse (read back from the deterministic backward's workspace)
against the forward's lse, and run-to-run equality."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2112_05682_b200 import api
from tests import helpers as Hh
for (B, n_q, n_k, H) in [(1, 1000, 1500, 2), (1, 4096, 4096, 4), (2, 300, 5000, 1)]:
    q, k, v, do = Hh.host_inputs(B, n_q, n_k, H, 64, seed=24, with_dout=True)
    qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    out, lse = api.mea_attention_fwd(qd, kd, vd, want_lse=True)
    nb = api.mea_attention_bwd_deterministic_workspace_size(B, H, n_q, n_k, 64, api.MEA_BF16, False)
    nq_pad = (n_q + 127) // 128 * 128
    rows_pad = B * H * nq_pad
    al = lambda x: (x + 255) // 256 * 256
    off = al(rows_pad * 4) * 2
    res = []
    for it in range(3):
        ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
        api.mea_attention_bwd_deterministic(qd, kd, vd, out, dod, lse=None, workspace=ws)
        torch.cuda.synchronize()
        l2 = ws[off:off + B * H * n_q * 4].view(torch.float32).reshape(B, H, n_q).clone()
        res.append(l2)
    d01 = (res[0] - res[1]).abs().max().item(); d02 = (res[0] - res[2]).abs().max().item()
    dl = (res[0] - lse).abs()
    bad = torch.nonzero(dl > 1e-4)
    print((B, n_q, n_k, H), "run-to-run", d01, d02, "vs fwd lse max", dl.max().item(), "bad rows", bad.shape[0],
          bad[:10].tolist())
