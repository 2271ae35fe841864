"""Soak of the backward with lse = NULL (the statistics pass B0 recomputes lse) against the oracle
and against the same backward given the forward's lse: random shapes up to 3000, d 64/128, plain /
causal / padded (element-wise bars as tests/test_gpu_fuzz.py, reading 16)."""
import math, sys
import numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle as O
from tests import helpers as Hh
from paper_2112_05682_b200 import api
N = int(sys.argv[1]) if len(sys.argv) > 1 else 40
fails = 0
for i in range(N):
    r = np.random.default_rng(321000 + i)
    d = int(r.choice([64, 128]))
    B, H = int(r.integers(1, 3)), int(r.integers(1, 3))
    n_q, n_k = int(r.integers(1, 3000)), int(r.integers(1, 3000))
    mode = str(r.choice(["plain", "causal", "padded"]))
    if mode == "causal":
        n_k = n_q
    scale = float(r.choice([1 / math.sqrt(d), -0.1, 0.03]))
    lens = [int(x) for x in r.integers(1, n_k + 1, size=B)] if mode == "padded" else [n_k] * B
    q, k, v, do = Hh.host_inputs(B, n_q, n_k, H, d, seed=i, with_dout=True)
    qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    kl = torch.tensor(lens, dtype=torch.int32, device="cuda")
    if mode == "plain":
        out, lse = api.mea_attention_fwd(qd, kd, vd, scale=scale, want_lse=True)
        bwd = lambda L: api.mea_attention_bwd(qd, kd, vd, out, dod, lse=L, scale=scale)
    elif mode == "causal":
        out, lse = api.mea_attention_fwd_causal(qd, kd, vd, scale=scale, want_lse=True)
        bwd = lambda L: api.mea_attention_bwd_causal(qd, kd, vd, out, dod, lse=L, scale=scale)
    else:
        out, lse = api.mea_attention_fwd_padded(qd, kd, vd, kl, scale=scale, want_lse=True)
        bwd = lambda L: api.mea_attention_bwd_padded(qd, kd, vd, out, dod, kl, lse=L, scale=scale)
    g_lse, g_b0 = bwd(lse), bwd(None)
    torch.cuda.synchronize()
    gtol = Hh.TOL_BF16_GRAD * max(1.0, abs(scale) * math.sqrt(d))
    try:
        for b in range(B):
            L = lens[b]
            refs = O.mha_backward(q[b:b + 1], k[b:b + 1, :L], v[b:b + 1, :L], do[b:b + 1], scale, causal=mode == "causal")
            for gi, (x, ref, nm) in enumerate(zip(g_b0, refs, ("dq", "dk", "dv"))):
                x = x[b:b + 1].double().cpu().numpy()
                x = x if nm == "dq" else x[:, :L]
                Hh.assert_close_bf16(x, ref, abs_tol=gtol if nm != "dv" else Hh.TOL_BF16_GRAD,
                                     rel_tol=Hh.REL_NORM_GRAD * (max(1.0, abs(scale) * math.sqrt(d)) if nm != "dv" else 1.0),
                                     what=f"{nm} (lse NULL)", strict=nm == "dv" or gtol == Hh.TOL_BF16_GRAD)
        dmax = max((a.float() - c.float()).abs().max().item() for a, c in zip(g_lse, g_b0))
        ok = True
    except AssertionError as e:
        ok = False
        dmax = float("nan")
        print(f"case {i}: {mode} d={d} B={B} H={H} n_q={n_q} n_k={n_k} scale={scale} lens={lens}: {e}")
    fails += not ok
print(f"{N - fails} of {N} cases pass")
