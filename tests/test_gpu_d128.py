"""GPU parity of head dimension 128 ("d=64 first; d=128 NEXT"): the forward
(fwd128_sm100a.cu) and the backward (bwd_det_sm100a.cu / bwd_dq_sm100a.cu at D = 128)
against the float64 oracle (O1) on the same generated inputs: shapes over several query and key
tiles with ragged tails, both output dtypes and scales, the rescale stress case, configs[2]'s
length at d = 128 on sampled rows, and the key-chunk schedule. Causal attention at d = 128:
tests/test_gpu_causal.py.
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
from tests import helpers as Hh

pytestmark = pytest.mark.gpu
D = 128


def _run(q, k, v, scale=None, out_dtype=None, **kw):
    from paper_2112_05682_b200 import api
    out, lse = api.mea_attention_fwd(Hh.to_dev(q, torch.bfloat16), Hh.to_dev(k, torch.bfloat16),
                                     Hh.to_dev(v, torch.bfloat16), scale=scale, out_dtype=out_dtype, want_lse=True,
                                     **kw)
    torch.cuda.synchronize()
    return out.double().cpu().numpy(), lse.double().cpu().numpy()


@pytest.mark.parametrize("B,n_q,n_k,H", [(1, 1, 1, 1), (1, 17, 129, 2), (2, 300, 1000, 3), (1, 1000, 17, 1),
                                         (1, 256, 4097, 2)])
def test_d128_forward_matches_oracle(B, n_q, n_k, H):
    q, k, v = Hh.host_inputs(B, n_q, n_k, H, D, seed=41)
    ref, ref_lse = O.mha_forward(q, k, v, 1 / math.sqrt(D))
    got, lse = _run(q, k, v)
    Hh.assert_close_bf16(got, ref)
    assert np.abs(lse - ref_lse).max() < 1e-3


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_d128_out_dtypes_and_scales(out_dtype):
    q, k, v = Hh.host_inputs(1, 200, 333, 2, D, seed=42)
    for scale in (1.0 / 16, 0.0, -0.05):
        ref, ref_lse = O.mha_forward(q, k, v, scale)
        got, lse = _run(q, k, v, scale=scale, out_dtype=out_dtype)
        Hh.assert_close_bf16(got, ref)
        assert np.abs(lse - ref_lse).max() < 1e-3


def test_d128_monotone_scores_rescale_every_tile():
    n = 900
    u = np.zeros(D); u[0] = 1.0
    k = (np.arange(n)[:, None] / n * 8.0) * u[None, :]
    q = np.tile(8.0 * u, (5, 1))
    v = Hh.host_inputs(1, 1, n, 1, D, seed=43)[2][0, :, 0]
    k_b = torch.tensor(k).bfloat16().double().numpy()
    ref, _ = O.naive(q, k_b, v, 1.0)
    got, _ = _run(q[None, :, None], k_b[None, :, None], v[None, :, None], scale=1.0)
    Hh.assert_close_bf16(got[0, :, 0], ref)


def test_d128_long_sequence_sampled_rows():
    """n = 16384 (configs[2]'s length), H = 8, d = 128: full launch, sampled rows vs O1."""
    from paper_2112_05682_b200 import api
    from synth import gen
    B, n, H = 1, 16384, 8
    q = torch.empty((B, n, H, D), dtype=torch.bfloat16, device="cuda")
    k, v = torch.empty_like(q), torch.empty_like(q)
    for t, tid in ((q, gen.TENSOR_Q), (k, gen.TENSOR_K), (v, gen.TENSOR_V)):
        api.mea_fill_synthetic(t, 0, tid)
    out, lse = api.mea_attention_fwd(q, k, v, want_lse=True)
    torch.cuda.synchronize()
    rows = np.array([0, 127, 128, 9999, 16383])
    kk = gen.normal_tensor((B, n, H, D), 0, gen.TENSOR_K, "bf16").astype(np.float64)
    vv = gen.normal_tensor((B, n, H, D), 0, gen.TENSOR_V, "bf16").astype(np.float64)
    for h in (0, 7):
        qr = gen.rows_of((B, n, H, D), 0, gen.TENSOR_Q, 0, rows, h)
        ref, ref_lse = O.naive(qr, kk[0, :, h], vv[0, :, h], 1 / math.sqrt(D))
        Hh.assert_close_bf16(out[0, rows, h].double().cpu().numpy(), ref)
        assert np.abs(lse[0, h, rows].double().cpu().numpy() - ref_lse).max() < 1e-3


def test_d128_key_chunk_schedule():
    """Figure 1's key-chunk summaries at d = 128 (fwd128 split mode + merge_rows), with and without
    query-chunk windows, equal the oracle."""
    q, k, v = Hh.host_inputs(2, 300, 1100, 2, D, seed=46)
    ref, ref_lse = O.mha_forward(q, k, v, 0.1)
    for qc, kc in ((0, 256), (128, 300), (1000, 128)):
        got, lse = _run(q, k, v, scale=0.1, q_chunk=qc, k_chunk=kc)
        Hh.assert_close_bf16(got, ref)
        assert np.abs(lse - ref_lse).max() < 1e-3


@pytest.mark.parametrize("B,n_q,n_k,H,lse_given", [(1, 130, 300, 2, True), (2, 257, 129, 1, True),
                                                   (1, 1, 1, 1, True), (1, 200, 333, 2, False)])
def test_d128_backward_matches_oracle(B, n_q, n_k, H, lse_given):
    """d = 128 backward (two-kernel path: dK/dV on 64-query tiles, dQ on 128-key tiles) vs O6."""
    from paper_2112_05682_b200 import api
    q, k, v, do = Hh.host_inputs(B, n_q, n_k, H, D, seed=44, with_dout=True)
    scale = 1 / math.sqrt(D)
    dq_r, dk_r, dv_r = O.mha_backward(q, k, v, do, scale)
    qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    out, lse = api.mea_attention_fwd(qd, kd, vd, want_lse=True)
    for fn in (api.mea_attention_bwd, api.mea_attention_bwd_deterministic):
        dq, dk, dv = fn(qd, kd, vd, out, dod, lse=lse if lse_given else None)
        torch.cuda.synchronize()
        for got, ref, name in ((dq, dq_r, "dq"), (dk, dk_r, "dk"), (dv, dv_r, "dv")):
            Hh.assert_close_bf16(got.double().cpu().numpy(), ref, abs_tol=Hh.TOL_BF16_GRAD,
                                 rel_tol=Hh.REL_NORM_GRAD, what=name)


def test_d128_backward_sampled_rows_n4096():
    from paper_2112_05682_b200 import api
    B, n, H = 1, 4096, 2
    q, k, v, do = Hh.host_inputs(B, n, n, H, D, seed=45, with_dout=True)
    qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    out, lse = api.mea_attention_fwd(qd, kd, vd, want_lse=True)
    dq, dk, dv = api.mea_attention_bwd(qd, kd, vd, out, dod, lse=lse)
    torch.cuda.synchronize()
    qr, kr = np.array([0, 63, 64, 2049, 4095]), np.array([0, 127, 128, 3000, 4095])
    for h in range(H):
        sq, sk, sv = O.backward_rows(q[0, :, h], k[0, :, h], v[0, :, h], do[0, :, h], 1 / math.sqrt(D), qr, kr)
        for got, ref, name in ((dq[0, qr, h], sq, "dq"), (dk[0, kr, h], sk, "dk"), (dv[0, kr, h], sv, "dv")):
            Hh.assert_close_bf16(got.double().cpu().numpy(), ref, abs_tol=Hh.TOL_BF16_GRAD,
                                 rel_tol=Hh.REL_NORM_GRAD, what=name)


@pytest.mark.parametrize("scale", [0.0, 0.05, 0.3, -0.1])
def test_d128_fused_backward_scales(scale):
    """The fused d = 128 backward (bwd128_sm100a.cu: lse per column, any scale incl. 0 and
    negative) against O6, next to the deterministic two-kernel path."""
    from paper_2112_05682_b200 import api
    q, k, v, do = Hh.host_inputs(1, 200, 300, 2, D, seed=46, with_dout=True)
    dq_r, dk_r, dv_r = O.mha_backward(q, k, v, do, scale)
    qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    out, lse = api.mea_attention_fwd(qd, kd, vd, scale=scale, want_lse=True)
    strict = abs(scale) <= 1 / math.sqrt(D)
    for fn in (api.mea_attention_bwd, api.mea_attention_bwd_deterministic):
        dq, dk, dv = fn(qd, kd, vd, out, dod, lse=lse, scale=scale)
        torch.cuda.synchronize()
        for got, ref, name in ((dq, dq_r, "dq"), (dk, dk_r, "dk"), (dv, dv_r, "dv")):
            Hh.assert_close_bf16(got.double().cpu().numpy(), ref, abs_tol=Hh.TOL_BF16_GRAD * max(1.0, abs(scale) * math.sqrt(D)),
                                 rel_tol=Hh.REL_NORM_GRAD, what=name, strict=strict)


def test_d128_full_size_sampled_rows_bench_config():
    """The bench's d = 128 extras at configs[2]/[3] shape (B=1 H=16 n=16384 d=128 bf16, device-
    generated inputs, the launch configuration bench.py times): forward and the fused backward
    on sampled rows of 2 heads against O1 / O6."""
    from paper_2112_05682_b200 import api
    from synth import gen
    B, n, H = 1, 16384, 16
    shape = (B, n, H, D)
    ts = [torch.empty(shape, dtype=torch.bfloat16, device="cuda") for _ in range(4)]
    for t, tid in zip(ts, (gen.TENSOR_Q, gen.TENSOR_K, gen.TENSOR_V, gen.TENSOR_DO)):
        api.mea_fill_synthetic(t, 0, tid)
    q, k, v, do = ts
    out, lse = api.mea_attention_fwd(q, k, v, want_lse=True)
    dq, dk, dv = api.mea_attention_bwd(q, k, v, out, do, lse=lse)
    torch.cuda.synchronize()
    rows = np.array([0, 1, 63, 64, 127, 128, 8191, 16383])
    scale = 1 / math.sqrt(D)
    for h in (0, 9):
        hq, hk, hv, hdo = (gen.rows_of(shape, 0, tid, 0, np.arange(n), h)
                           for tid in (gen.TENSOR_Q, gen.TENSOR_K, gen.TENSOR_V, gen.TENSOR_DO))
        ro, rl = O.naive(hq[rows], hk, hv, scale)
        Hh.assert_close_bf16(out[0, rows, h].double().cpu().numpy(), ro)
        assert np.abs(lse[0, h, rows].double().cpu().numpy() - rl).max() < 1e-3
        rq, rk, rv = O.backward_rows(hq, hk, hv, hdo, scale, rows, rows)
        Hh.assert_close_bf16(dq[0, rows, h].double().cpu().numpy(), rq, Hh.TOL_BF16_GRAD, Hh.REL_NORM_GRAD, "dq")
        Hh.assert_close_bf16(dk[0, rows, h].double().cpu().numpy(), rk, Hh.TOL_BF16_GRAD, Hh.REL_NORM_GRAD, "dk")
        Hh.assert_close_bf16(dv[0, rows, h].double().cpu().numpy(), rv, Hh.TOL_BF16_GRAD, Hh.REL_NORM_GRAD, "dv")
