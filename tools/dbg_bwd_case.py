"""Is a backward mismatch the kernel's or bf16's? For one fuzz case (padded or causal or plain),
compare the kernel's dq / dk with (a) the exact fp64 oracle and (b) fp64 arithmetic in which only
`out` (entering delta = dO . out) and dS are rounded to bf16, as the API's contract and the MMA
operand make them. Usage: python tools/dbg_bwd_case.py B n_q n_k H d scale mode seed [lens...]"""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle as O
from tests import helpers as Hh
from paper_2112_05682_b200 import api
B, n_q, n_k, H, d = (int(x) for x in sys.argv[1:6])
scale, mode, seed = float(sys.argv[6]), sys.argv[7], int(sys.argv[8])
lens = [int(x) for x in sys.argv[9:]] or [n_k] * B
if mode == "causal":
    n_k = n_q
q, k, v, do = Hh.host_inputs(B, n_q, n_k, H, d, seed=seed, with_dout=True)
qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
kl = torch.tensor(lens, dtype=torch.int32, device="cuda")
if mode == "padded":
    out, lse = api.mea_attention_fwd_padded(qd, kd, vd, kl, scale=scale, out_dtype=torch.float32, want_lse=True)
    g = api.mea_attention_bwd_padded(qd, kd, vd, out.to(torch.bfloat16), dod, kl, lse=lse, scale=scale)
elif mode == "causal":
    out, lse = api.mea_attention_fwd_causal(qd, kd, vd, scale=scale, out_dtype=torch.float32, want_lse=True)
    g = api.mea_attention_bwd_causal(qd, kd, vd, out.to(torch.bfloat16), dod, lse=lse, scale=scale)
else:
    out, lse = api.mea_attention_fwd(qd, kd, vd, scale=scale, out_dtype=torch.float32, want_lse=True)
    g = api.mea_attention_bwd(qd, kd, vd, out.to(torch.bfloat16), dod, lse=lse, scale=scale)
torch.cuda.synchronize()
gq, gk = g[0].double().cpu().numpy(), g[1].double().cpu().numpy()
ob = out.to(torch.bfloat16).double().cpu().numpy()
bf = lambda x: torch.from_numpy(x).to(torch.bfloat16).double().numpy()
for b in range(B):
    L = lens[b] if mode == "padded" else n_k
    rq, rk, _ = O.mha_backward(q[b:b + 1], k[b:b + 1, :L], v[b:b + 1, :L], do[b:b + 1], scale, causal=mode == "causal")
    eq, ek = np.zeros_like(rq), np.zeros_like(rk)
    for h in range(H):
        s = scale * (q[b, :, h] @ k[b, :L, h].T)
        if mode == "causal":
            s = np.where(np.tril(np.ones(s.shape, dtype=bool)), s, -np.inf)
        p = np.exp(s - s.max(1, keepdims=True)); p /= p.sum(1, keepdims=True)
        delta = (do[b, :, h] * ob[b, :, h]).sum(1, keepdims=True)
        ds = bf(p * (do[b, :, h] @ v[b, :L, h].T - delta))
        eq[0, :, h] = scale * ds @ k[b, :L, h]
        ek[0, :, h] = scale * ds.T @ q[b, :, h]
    for nm, got, ref, emu in (("dq", gq[b:b + 1], rq, eq), ("dk", gk[b:b + 1, :L], rk, ek)):
        print(f"b={b} {nm}: max|got-exact| {np.abs(got - ref).max():.4f}  max|emu-exact| {np.abs(emu - ref).max():.4f}  "
              f"max|got-emu| {np.abs(got - emu).max():.4f}  max|ref| {np.abs(ref).max():.3f}")
    for nm, got, ref, emu in (("dq", gq[b:b + 1], rq, eq), ("dk", gk[b:b + 1, :L], rk, ek)):
        print(f"b={b} {nm}: rel-norm got-exact {Hh.rel_norm(got, ref):.4f}  emu-exact {Hh.rel_norm(emu, ref):.4f}  "
              f"got-emu {Hh.rel_norm(got, emu):.4f}")
