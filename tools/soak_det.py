"""Soak of the deterministic backward (and its bitwise reproducibility) at lengths up to 3000:
random shapes, d 64/128, scales; element-wise bars as tests/test_gpu_fuzz.py (reading 16)."""
import math, sys
import numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle as O
from tests import helpers as Hh
from paper_2112_05682_b200 import api
N = int(sys.argv[1]) if len(sys.argv) > 1 else 40
fails = 0
for i in range(N):
    r = np.random.default_rng(123000 + i)
    d = int(r.choice([64, 128]))
    B, H = int(r.integers(1, 3)), int(r.integers(1, 3))
    n_q, n_k = int(r.integers(1, 3000)), int(r.integers(1, 3000))
    scale = float(r.choice([1 / math.sqrt(d), -0.1, 0.03]))
    q, k, v, do = Hh.host_inputs(B, n_q, n_k, H, d, seed=i, with_dout=True)
    qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    out, lse = api.mea_attention_fwd(qd, kd, vd, scale=scale, want_lse=True)
    g1 = api.mea_attention_bwd_deterministic(qd, kd, vd, out, dod, lse=lse, scale=scale)
    g2 = api.mea_attention_bwd_deterministic(qd, kd, vd, out, dod, lse=lse, scale=scale)
    torch.cuda.synchronize()
    same = all(torch.equal(a, b) for a, b in zip(g1, g2))
    gtol = Hh.TOL_BF16_GRAD * max(1.0, abs(scale) * math.sqrt(d))
    try:
        for x, ref, nm in zip(g1, O.mha_backward(q, k, v, do, scale), ("dq", "dk", "dv")):
            Hh.assert_close_bf16(x.double().cpu().numpy(), ref, abs_tol=gtol if nm != "dv" else Hh.TOL_BF16_GRAD,
                                 rel_tol=Hh.REL_NORM_GRAD * (max(1.0, abs(scale) * math.sqrt(d)) if nm != "dv" else 1.0),
                                 what=nm, strict=nm == "dv" or gtol == Hh.TOL_BF16_GRAD)
        ok = same
    except AssertionError as e:
        ok = False
        print(f"case {i}: d={d} B={B} H={H} n_q={n_q} n_k={n_k} scale={scale}: {e}")
    if not same:
        print(f"case {i}: not bitwise reproducible")
    fails += not ok
print(f"{N - fails} of {N} cases pass")
