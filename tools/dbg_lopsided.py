import sys, math, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle as O
from tests import helpers as Hh
from paper_2112_05682_b200 import api
for n_q in (2003, 20003, 60003, 200003):
    n_k, B, H, d = 3, 1, 2, 64
    q, k, v, do = Hh.host_inputs(B, n_q, n_k, H, d, seed=62, with_dout=True)
    qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    scale = 1 / math.sqrt(d)
    out, lse = api.mea_attention_fwd(qd, kd, vd, out_dtype=torch.float32, want_lse=True)
    ob = out.to(torch.bfloat16)
    g = api.mea_attention_bwd(qd, kd, vd, ob, dod, lse=lse)
    gd = api.mea_attention_bwd_deterministic(qd, kd, vd, ob, dod, lse=lse)
    torch.cuda.synchronize()
    rq, rk, rv = O.mha_backward(q, k, v, do, scale)
    # fp64 with out rounded to bf16 (delta) and dS rounded
    Ob = ob.double().cpu().numpy()
    ek = np.zeros_like(rk)
    for h in range(H):
        s = scale * q[0, :, h] @ k[0, :, h].T
        p = np.exp(s - s.max(1, keepdims=True)); p /= p.sum(1, keepdims=True)
        delta = (do[0, :, h] * Ob[0, :, h]).sum(1, keepdims=True)
        ds = torch.from_numpy(p * (do[0, :, h] @ v[0, :, h].T - delta)).to(torch.bfloat16).double().numpy()
        ek[0, :, h] = scale * ds.T @ q[0, :, h]
    for nm, x, r in (("fused", g[1], rk), ("det", gd[1], rk)):
        x = x.double().cpu().numpy()
        print(f"n_q={n_q} {nm} dk: max|got-exact| {np.abs(x - r).max():.4f}  max|got-emu| {np.abs(x - ek).max():.4f} "
              f"max|emu-exact| {np.abs(ek - r).max():.4f}  max|ref| {np.abs(r).max():.2f}")
    print(f"   dv fused max err {np.abs(g[2].double().cpu().numpy() - rv).max():.4f}, max|dv| {np.abs(rv).max():.1f}")
    for nm, x, r in (("dk", g[1], rk), ("dv", g[2], rv)):
        print(f"   {nm} relative norm error {Hh.rel_norm(x.double().cpu().numpy(), r):.2e}")
