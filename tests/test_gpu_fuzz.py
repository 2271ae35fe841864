"""Seeded random sweep over the whole entry-point surface against the float64 oracle (O1, O5,
O5t, O6 and their causal / truncated-key forms): shapes (ragged against every tile size: 96-key
and 128-key tiles, 128- and 256-row query blocks), head dims 64 / 128, scales of either sign and
zero, output dtypes, key chunks, query chunks, padding and causal masks. Each case is small enough
for the oracle; the point is breadth — a schedule or mask combination that breaks shows up here
even if no hand-written case hits it.
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle as O
from tests import helpers as Hh

pytestmark = pytest.mark.gpu

# MEA_FUZZ_CASES / MEA_FUZZ_BASE widen the sweep for a soak run (defaults: the 150 committed cases)
N_CASES = int(os.environ.get("MEA_FUZZ_CASES", "150"))
BASE = int(os.environ.get("MEA_FUZZ_BASE", "1000"))
NMAX = int(os.environ.get("MEA_FUZZ_NMAX", "0"))   # > 0: lengths up to NMAX instead of 520 / 700


def _case(i):
    r = np.random.default_rng(BASE + i)
    d = int(r.choice([64, 128]))
    B, H = int(r.integers(1, 3)), int(r.integers(1, 3))
    n_q, n_k = int(r.integers(1, NMAX or 520)), int(r.integers(1, NMAX or 700))
    scale = float(r.choice([1 / math.sqrt(d), 0.5, -0.2, 0.0, 0.02]))
    mode = str(r.choice(["plain", "chunks", "causal", "padded", "tree"]))
    out_f32 = bool(r.integers(0, 2))
    return dict(d=d, B=B, H=H, n_q=n_q, n_k=n_k, scale=scale, mode=mode, out_f32=out_f32,
                q_chunk=int(r.choice([0, 1, 300, 1024])), k_chunk=int(r.choice([1, 128, 200, 4096, -1])),
                lens=[int(x) for x in r.integers(0, n_k + 1, size=B)], seed=i)


@pytest.mark.parametrize("i", range(N_CASES))
def test_forward_and_backward_random_case(i):
    from paper_2112_05682_b200 import api
    c = _case(i)
    d, B, H, n_q, n_k, scale = c["d"], c["B"], c["H"], c["n_q"], c["n_k"], c["scale"]
    if c["mode"] == "causal":
        n_k = n_q
    q, k, v, do = Hh.host_inputs(B, n_q, n_k, H, d, seed=c["seed"], with_dout=True)
    qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    od = torch.float32 if c["out_f32"] else torch.bfloat16
    mode = c["mode"]
    lens = [min(L, n_k) for L in c["lens"]]
    if mode == "plain":
        out, lse = api.mea_attention_fwd(qd, kd, vd, scale=scale, out_dtype=od, want_lse=True)
    elif mode == "chunks":
        out, lse = api.mea_attention_fwd(qd, kd, vd, scale=scale, out_dtype=od, want_lse=True,
                                         q_chunk=c["q_chunk"], k_chunk=c["k_chunk"])
    elif mode == "tree":
        out, lse = api.mea_attention_fwd_tree(qd, kd, vd, scale=scale, out_dtype=od, want_lse=True,
                                              q_chunk=c["q_chunk"], k_chunk=c["k_chunk"])
    elif mode == "causal":
        out, lse = api.mea_attention_fwd_causal(qd, kd, vd, scale=scale, out_dtype=od, want_lse=True)
    else:
        kl = torch.tensor(lens, dtype=torch.int32, device="cuda")
        out, lse = api.mea_attention_fwd_padded(qd, kd, vd, kl, scale=scale, out_dtype=od, want_lse=True)
    torch.cuda.synchronize()
    got, glse = out.double().cpu().numpy(), lse.double().cpu().numpy()
    causal = mode == "causal"
    for b in range(B):
        L = lens[b] if mode == "padded" else n_k
        if L == 0:   # padded element with no keys: out 0, lse -inf
            assert (got[b] == 0).all() and np.isneginf(glse[b]).all()
            continue
        ref, ref_lse = O.mha_forward(q[b:b + 1], k[b:b + 1, :L], v[b:b + 1, :L], scale, causal=causal)
        Hh.assert_close_bf16(got[b:b + 1], ref, what=f"case {i} {mode} out")
        assert np.abs(glse[b:b + 1] - ref_lse).max() < 1e-3, f"case {i} {mode} lse"
    # backward on the modes that have one (the padded / causal / plain forward's)
    if mode in ("plain", "causal", "padded") and scale != 0.0 and all(L > 0 for L in lens):
        ob = out if out.dtype == torch.bfloat16 else out.to(torch.bfloat16)
        if mode == "plain":
            dq, dk, dv = api.mea_attention_bwd(qd, kd, vd, ob, dod, lse=lse, scale=scale)
        elif mode == "causal":
            dq, dk, dv = api.mea_attention_bwd_causal(qd, kd, vd, ob, dod, lse=lse, scale=scale)
        else:
            dq, dk, dv = api.mea_attention_bwd_padded(qd, kd, vd, ob, dod, kl, lse=lse, scale=scale)
        torch.cuda.synchronize()
        dq, dk, dv = (x.double().cpu().numpy() for x in (dq, dk, dv))
        # dq = scale dS K and dk = scale dS^T Q carry the bf16 rounding of dS (an MMA operand) times
        # `scale`: the north star's 5e-2 is stated at the standard scale 1/sqrt(d), so the bar
        # grows with |scale| sqrt(d) beyond it (reading 16)
        gtol = Hh.TOL_BF16_GRAD * max(1.0, abs(scale) * math.sqrt(d))
        for b in range(B):
            L = lens[b] if mode == "padded" else n_k
            rq, rk, rv = O.mha_backward(q[b:b + 1], k[b:b + 1, :L], v[b:b + 1, :L], do[b:b + 1], scale, causal=causal)
            # the relative-norm guard on dq / dk widens like their absolute bar (reading 16): the
            # bf16 roundings of out (in delta = dO . out) and of dS cancel against dP in peaked rows
            # (soak case 766 of MEA_FUZZ_BASE=40000 — d = 128, n = 6, causal, scale 0.5 — is 3.0 % off
            # for the kernel and for fp64 arithmetic with only out and dS rounded to bf16 alike,
            # tools/dbg_case766.py)
            gw = max(1.0, abs(scale) * math.sqrt(d))
            rel = {"dq": Hh.REL_NORM_GRAD * gw, "dk": Hh.REL_NORM_GRAD * gw, "dv": Hh.REL_NORM_GRAD}
            aq, ak, av = _operand_allowance(q[b:b + 1], k[b:b + 1, :L], v[b:b + 1, :L], do[b:b + 1], scale, causal)
            ex = {"dq": aq, "dk": ak, "dv": av}
            for g, r, nm in ((dq[b:b + 1], rq, "dq"), (dk[b:b + 1, :L], rk, "dk"), (dv[b:b + 1, :L], rv, "dv")):
                Hh.assert_close_bf16(g, r, abs_tol=gtol if nm != "dv" else Hh.TOL_BF16_GRAD, rel_tol=rel[nm], extra=ex[nm],
                                     strict=nm == "dv" or gtol == Hh.TOL_BF16_GRAD,
                                     what=f"case {i} {nm}")
            if L < n_k:
                assert (dk[b, L:] == 0).all() and (dv[b, L:] == 0).all()


def _operand_allowance(q, k, v, do, scale, causal):
    """First-order bound of what bf16 rounding of the backward's inputs can move dq and dk by
    (reading 16), element-wise, in fp64 from one batch element ([1, n, H, d]): dS is an
    MMA operand rounded to bf16 (|err| <= 2^-8 |dS|), and delta = dO . out is formed from the
    bf16-stored out (|err delta_i| <= 2^-8 (|dO| . |out|)_i, entering dS_ij as P_ij err delta_i);
    then |err dq| <= |scale| e |K| and |err dk| <= |scale| e^T |Q| with e the dS error bound;
    P is the dV MMA's bf16 operand, |err dv| <= 2^-8 P^T |dO|. Negligible for long rows; large for
    a few keys under many queries, where dk and dv sum many terms."""
    aq, ak, av = np.zeros_like(q), np.zeros_like(k), np.zeros_like(k)
    for h in range(q.shape[2]):
        qh, kh, vh, doh = q[0, :, h], k[0, :, h], v[0, :, h], do[0, :, h]
        s = scale * (qh @ kh.T)
        if causal:
            s = np.where(np.tril(np.ones(s.shape, dtype=bool)), s, -np.inf)
        p = np.exp(s - s.max(axis=1, keepdims=True))
        p /= p.sum(axis=1, keepdims=True)
        oh = p @ vh
        ds = p * (doh @ vh.T - (doh * oh).sum(axis=1, keepdims=True))
        e = 2.0 ** -8 * (np.abs(ds) + p * (np.abs(doh) * np.abs(oh)).sum(axis=1, keepdims=True))
        aq[0, :, h] = abs(scale) * (e @ np.abs(kh))
        ak[0, :, h] = abs(scale) * (e.T @ np.abs(qh))
        av[0, :, h] = 2.0 ** -8 * (p.T @ np.abs(doh))
    return aq, ak, av


N_OTHER = int(os.environ.get("MEA_FUZZ_OTHER_CASES", "60"))


@pytest.mark.parametrize("i", range(N_OTHER))
def test_other_entry_points_random_case(i):
    """Single query (bf16 d 64/128, f32), key-range partials merged, the deterministic backward
    and the fp32 forwards (exact SIMT and split-precision) on random shapes."""
    from paper_2112_05682_b200 import api
    r = np.random.default_rng(BASE + 4000 + i)
    kind = ["single_query", "partial_merge", "bwd_det", "f32"][i % 4]
    d = int(r.choice([64, 128]))
    B, H = int(r.integers(1, 3)), int(r.integers(1, 4))
    n_q, n_k = int(r.integers(1, 400)), int(r.integers(1, 3000))
    scale = float(r.choice([1 / math.sqrt(d), -0.1, 0.03]))
    if kind == "single_query":
        f32 = bool(r.integers(0, 2))
        q, k, v = Hh.host_inputs(B, 1, n_k, H, d, seed=i, dtype="f32" if f32 else "bf16")
        dt = torch.float32 if f32 else torch.bfloat16
        out = api.mea_single_query_fwd(Hh.to_dev(q[:, 0], dt), Hh.to_dev(k, dt), Hh.to_dev(v, dt), scale=scale,
                                       out_dtype=torch.float32)
        torch.cuda.synchronize()
        got = out.double().cpu().numpy()
        for b in range(B):
            for h in range(H):
                ref = O.naive(q[b, 0, h][None], k[b, :, h], v[b, :, h], scale)[0][0]
                if f32:
                    Hh.assert_close_f32(got[b, h], ref)
                else:
                    Hh.assert_close_bf16(got[b, h], ref)
    elif kind == "partial_merge":
        q, k, v = Hh.host_inputs(B, n_q, n_k, H, d, seed=i)
        cuts = sorted({0, n_k, *[int(x) for x in r.integers(0, n_k + 1, size=int(r.integers(0, 4)))]})
        qd = Hh.to_dev(q, torch.bfloat16)
        parts = [api.mea_attention_partial_fwd(qd, Hh.to_dev(k[:, a:b_], torch.bfloat16),
                                               Hh.to_dev(v[:, a:b_], torch.bfloat16), scale=scale)
                 for a, b_ in zip(cuts[:-1], cuts[1:])]
        out = api.mea_merge_partials(torch.stack([p_[0].reshape(-1) for p_ in parts]),
                                     torch.stack([p_[1].reshape(-1) for p_ in parts]),
                                     torch.stack([p_[2].reshape(-1, d) for p_ in parts]), B, n_q * H,
                                     out_dtype=torch.float32).reshape(B, n_q, H, d)
        torch.cuda.synchronize()
        Hh.assert_close_bf16(out.double().cpu().numpy(), O.mha_forward(q, k, v, scale)[0])
    elif kind == "bwd_det":
        n_k = min(n_k, 800)
        q, k, v, do = Hh.host_inputs(B, n_q, n_k, H, d, seed=i, with_dout=True)
        qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
        out, lse = api.mea_attention_fwd(qd, kd, vd, scale=scale, want_lse=True)
        g = api.mea_attention_bwd_deterministic(qd, kd, vd, out, dod, lse=lse if i % 8 else None, scale=scale)
        torch.cuda.synchronize()
        gtol = Hh.TOL_BF16_GRAD * max(1.0, abs(scale) * math.sqrt(d))
        for x, ref, nm in zip(g, O.mha_backward(q, k, v, do, scale), ("dq", "dk", "dv")):
            Hh.assert_close_bf16(x.double().cpu().numpy(), ref, abs_tol=gtol, rel_tol=Hh.REL_NORM_GRAD, what=nm,
                                 strict=nm == "dv" or gtol == Hh.TOL_BF16_GRAD)
    else:
        n_q, n_k = min(n_q, 200), min(n_k, 600)
        split = d == 64 and bool(r.integers(0, 2))
        q, k, v = Hh.host_inputs(B, n_q, n_k, H, d, seed=i, dtype="f32")
        out, lse = api.mea_attention_fwd(Hh.to_dev(q, torch.float32), Hh.to_dev(k, torch.float32),
                                         Hh.to_dev(v, torch.float32), scale=scale, want_lse=True, f32_split=split)
        torch.cuda.synchronize()
        ref, ref_lse = O.mha_forward(q, k, v, scale)
        got = out.double().cpu().numpy()
        if split:   # the split-precision bound (tests/test_gpu_forward.py): 1e-5 + 3 2^-18 max|v|
            assert np.abs(got - ref).max() <= 1e-5 + 3 * 2.0 ** -18 * np.abs(v).max()
        else:
            Hh.assert_close_f32(got, ref)
        assert np.abs(lse.double().cpu().numpy() - ref_lse).max() < 1e-5
