import sys, math, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle as O
from tests import helpers as Hh
from paper_2112_05682_b200 import api
B, n, H, d, scale = 2, 6, 2, 128, 0.5
q, k, v, do = Hh.host_inputs(B, n, n, H, d, seed=766, with_dout=True)
qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
out, lse = api.mea_attention_fwd_causal(qd, kd, vd, scale=scale, out_dtype=torch.float32, want_lse=True)
outb = out.to(torch.bfloat16)
g = api.mea_attention_bwd_causal(qd, kd, vd, outb, dod, lse=lse, scale=scale)
torch.cuda.synchronize()
ref = O.mha_backward(q, k, v, do, scale, causal=True)
# emulate the kernel's roundings in fp64 with bf16 rounding of P and dS
def bf(x): return torch.tensor(x, dtype=torch.float64).to(torch.bfloat16).double().numpy()
Ob = outb.double().cpu().numpy(); L = lse.double().cpu().numpy()
emu = np.zeros_like(q)
for b in range(B):
    for h in range(H):
        s = q[b, :, h] @ k[b, :, h].T
        mask = np.tril(np.ones((n, n))) > 0
        P = np.where(mask, np.exp(s * scale - L[b, h][:, None]), 0.0)
        dP = do[b, :, h] @ v[b, :, h].T
        delta = (do[b, :, h] * Ob[b, :, h]).sum(-1)
        dS = bf(P * (dP - delta[:, None]))
        emu[b, :, h] = scale * dS @ k[b, :, h]
got = g[0].double().cpu().numpy()
def rn(a, r): return np.linalg.norm(a - r) / np.linalg.norm(r)
print("dq rel-norm got vs exact", rn(got, ref[0]), " emulated vs exact", rn(emu, ref[0]), " got vs emulated", rn(got, emu))
print("max abs got-exact", np.abs(got - ref[0]).max(), "norm exact", np.linalg.norm(ref[0]))
gd = api.mea_attention_bwd_deterministic(qd, kd, vd, outb, dod, lse=lse, scale=scale) if False else None
for b in range(B):
    print(f"b={b}: dq rel-norm got vs exact {rn(got[b], ref[0][b]):.4f}, emulated vs exact {rn(emu[b], ref[0][b]):.4f}, "
          f"got vs emulated {rn(got[b], emu[b]):.4f}, norm exact {np.linalg.norm(ref[0][b]):.3f}")
