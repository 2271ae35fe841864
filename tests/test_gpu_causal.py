"""GPU parity of causal attention (query i attends keys j <= i) —
mea_attention_fwd_causal / mea_attention_bwd_causal against the float64 oracle's causal
definition (O1/O6 with ``causal=True``, pinned in tests/test_oracle.py) on the same generated
inputs. Sizes cover one tile, several 256-row blocks with ragged tails, and configs[2]'s shape on
sampled rows; bf16 tolerances as for the non-causal path.
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
from tests import helpers as Hh

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,n,H", [(1, 17, 2), (2, 300, 1), (1, 513, 2)])
def test_causal_d128_forward_and_backward(B, n, H):
    """d = 128: fwd128 with the diagonal mask, and the two-kernel backward starting each key tile
    at its diagonal (dK/dV) / stopping each query block at its diagonal (dQ)."""
    from paper_2112_05682_b200 import api
    q, k, v, do = Hh.host_inputs(B, n, n, H, 128, seed=35, with_dout=True)
    scale = 1 / math.sqrt(128)
    ref, ref_lse = O.mha_forward(q, k, v, scale, causal=True)
    dq_r, dk_r, dv_r = O.mha_backward(q, k, v, do, scale, causal=True)
    qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    out, lse = api.mea_attention_fwd_causal(qd, kd, vd, want_lse=True)
    dq, dk, dv = api.mea_attention_bwd_causal(qd, kd, vd, out, dod, lse=lse)
    torch.cuda.synchronize()
    Hh.assert_close_bf16(out.double().cpu().numpy(), ref)
    assert np.abs(lse.double().cpu().numpy() - ref_lse).max() < 1e-3
    for got, r, name in ((dq, dq_r, "dq"), (dk, dk_r, "dk"), (dv, dv_r, "dv")):
        Hh.assert_close_bf16(got.double().cpu().numpy(), r, abs_tol=Hh.TOL_BF16_GRAD, rel_tol=Hh.REL_NORM_GRAD,
                             what=name)


def _fwd(q, k, v, scale):
    from paper_2112_05682_b200 import api
    out, lse = api.mea_attention_fwd_causal(Hh.to_dev(q, torch.bfloat16), Hh.to_dev(k, torch.bfloat16),
                                            Hh.to_dev(v, torch.bfloat16), scale=scale, want_lse=True)
    torch.cuda.synchronize()
    return out.double().cpu().numpy(), lse.double().cpu().numpy()


@pytest.mark.parametrize("B,n,H", [(1, 1, 1), (1, 17, 2), (2, 300, 3), (1, 513, 1), (1, 1000, 2), (1, 1024, 1)])
def test_causal_forward_matches_oracle(B, n, H):
    q, k, v = Hh.host_inputs(B, n, n, H, 64, seed=31)
    ref, ref_lse = O.mha_forward(q, k, v, 0.125, causal=True)
    got, lse = _fwd(q, k, v, 0.125)
    Hh.assert_close_bf16(got, ref)
    assert np.abs(lse - ref_lse).max() < 1e-3
    np.testing.assert_allclose(got[:, 0], np.asarray(torch.tensor(v[:, 0]).bfloat16().double()), atol=0)  # row 0 = v_0


def test_causal_forward_stress_monotone_scores():
    """Scores growing along the keys: every tile rescales, and the diagonal tile's masked keys
    hold the largest raw scores (they must not leak into the max or the sums)."""
    n, d = 700, 64
    u = np.zeros(d); u[0] = 1.0
    k = (np.arange(n)[:, None] / n * 8.0) * u[None, :]
    q = np.tile(8.0 * u, (n, 1))
    v = Hh.host_inputs(1, 1, n, 1, d, seed=32)[2][0, :, 0]
    k_b = torch.tensor(k).bfloat16().double().numpy()
    ref, _ = O.naive(q, k_b, v, 1.0, causal=True)
    got, _ = _fwd(q[None, :, None], k_b[None, :, None], v[None, :, None], 1.0)
    Hh.assert_close_bf16(got[0, :, 0], ref)


@pytest.mark.parametrize("B,n,H,lse_given", [(1, 130, 2, True), (2, 300, 1, True), (1, 600, 2, False),
                                             (1, 1, 1, True)])
def test_causal_backward_matches_oracle(B, n, H, lse_given):
    from paper_2112_05682_b200 import api
    q, k, v, do = Hh.host_inputs(B, n, n, H, 64, seed=33, with_dout=True)
    scale = 0.125
    dq_r, dk_r, dv_r = O.mha_backward(q, k, v, do, scale, causal=True)
    qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    out, lse = api.mea_attention_fwd_causal(qd, kd, vd, scale=scale, want_lse=True)
    dq, dk, dv = api.mea_attention_bwd_causal(qd, kd, vd, out, dod, lse=lse if lse_given else None, scale=scale)
    torch.cuda.synchronize()
    for got, ref, name in ((dq, dq_r, "dq"), (dk, dk_r, "dk"), (dv, dv_r, "dv")):
        Hh.assert_close_bf16(got.double().cpu().numpy(), ref, abs_tol=Hh.TOL_BF16_GRAD, rel_tol=Hh.REL_NORM_GRAD,
                             what=name)


def test_causal_rejects_unsupported():
    from paper_2112_05682_b200 import api
    q = torch.zeros(1, 8, 1, 64, dtype=torch.bfloat16, device="cuda")
    k = torch.zeros(1, 9, 1, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        api.mea_attention_fwd_causal(q, k, k)
    with pytest.raises(api.MeaError):
        api.mea_attention_fwd_causal(q.float(), q.float(), q.float())


def test_causal_config3_shape_sampled_rows():
    """configs[2]'s shape (H = 16, n = 16384): the full launch, sampled rows of two heads vs
    the oracle's causal rows (prefix lengths 1 ... 16384), incl. block and tile boundaries."""
    from paper_2112_05682_b200 import api
    from synth import gen
    B, n, H, d = 1, 16384, 16, 64
    q = torch.empty((B, n, H, d), dtype=torch.bfloat16, device="cuda")
    k, v = torch.empty_like(q), torch.empty_like(q)
    for t, tid in ((q, gen.TENSOR_Q), (k, gen.TENSOR_K), (v, gen.TENSOR_V)):
        api.mea_fill_synthetic(t, 0, tid)
    out, lse = api.mea_attention_fwd_causal(q, k, v, want_lse=True)
    torch.cuda.synchronize()
    rows = np.array([0, 1, 127, 128, 255, 256, 8191, 12345, 16383])
    kk = gen.normal_tensor((B, n, H, d), 0, gen.TENSOR_K, "bf16").astype(np.float64)
    vv = gen.normal_tensor((B, n, H, d), 0, gen.TENSOR_V, "bf16").astype(np.float64)
    qq = gen.normal_tensor((B, n, H, d), 0, gen.TENSOR_Q, "bf16").astype(np.float64)
    for h in (0, 15):
        ref, ref_lse = O.naive(qq[0, :, h], kk[0, :, h], vv[0, :, h], 1 / math.sqrt(d), rows=rows, causal=True)
        Hh.assert_close_bf16(out[0, rows, h].double().cpu().numpy(), ref)
        assert np.abs(lse[0, h, rows].double().cpu().numpy() - ref_lse).max() < 1e-3


def test_causal_backward_sampled_rows_n4096():
    """Backward at n = 4096 (16 key tiles, triangular work), sampled dq / dk / dv rows vs O6."""
    from paper_2112_05682_b200 import api
    B, n, H, d = 1, 4096, 2, 64
    q, k, v, do = Hh.host_inputs(B, n, n, H, d, seed=34, with_dout=True)
    qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    out, lse = api.mea_attention_fwd_causal(qd, kd, vd, want_lse=True)
    dq, dk, dv = api.mea_attention_bwd_causal(qd, kd, vd, out, dod, lse=lse)
    torch.cuda.synchronize()
    qr = np.array([0, 127, 128, 2049, 4095])
    kr = np.array([0, 1, 128, 3000, 4095])
    for h in range(H):
        sq, sk, sv = O.backward_rows(q[0, :, h], k[0, :, h], v[0, :, h], do[0, :, h], 1 / math.sqrt(d), qr, kr,
                                     causal=True)
        Hh.assert_close_bf16(dq[0, qr, h].double().cpu().numpy(), sq, abs_tol=Hh.TOL_BF16_GRAD,
                             rel_tol=Hh.REL_NORM_GRAD, what="dq")
        Hh.assert_close_bf16(dk[0, kr, h].double().cpu().numpy(), sk, abs_tol=Hh.TOL_BF16_GRAD,
                             rel_tol=Hh.REL_NORM_GRAD, what="dk")
        Hh.assert_close_bf16(dv[0, kr, h].double().cpu().numpy(), sv, abs_tol=Hh.TOL_BF16_GRAD,
                             rel_tol=Hh.REL_NORM_GRAD, what="dv")
