"""GPU parity of key padding (masks needed to use the library on a padded batch):
mea_attention_fwd_padded / mea_attention_bwd_padded against the float64 oracle applied to each
batch element's unpadded keys k[b, :L_b], v[b, :L_b] (O1 / O6 — masking a key is removing it from
the definition), on the same generated inputs; padded keys must get dk = dv = 0
exactly, and a batch element with no keys out = 0, lse = -inf.
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
from tests import helpers as Hh

pytestmark = pytest.mark.gpu


def _lens(x):
    return torch.tensor(x, dtype=torch.int32, device="cuda")


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("B,n_q,n_k,H,lens", [(3, 300, 1000, 2, [1000, 1, 517]), (2, 129, 96, 1, [95, 96]),
                                              (2, 257, 2000, 2, [1999, 1300])])
def test_padded_forward_matches_oracle(d, B, n_q, n_k, H, lens):
    from paper_2112_05682_b200 import api
    q, k, v = Hh.host_inputs(B, n_q, n_k, H, d, seed=51)
    scale = 1 / math.sqrt(d)
    out, lse = api.mea_attention_fwd_padded(Hh.to_dev(q, torch.bfloat16), Hh.to_dev(k, torch.bfloat16),
                                            Hh.to_dev(v, torch.bfloat16), _lens(lens), want_lse=True,
                                            out_dtype=torch.float32)
    torch.cuda.synchronize()
    out, lse = out.double().cpu().numpy(), lse.double().cpu().numpy()
    for b, L in enumerate(lens):
        ref, ref_lse = O.mha_forward(q[b:b + 1], k[b:b + 1, :L], v[b:b + 1, :L], scale)
        Hh.assert_close_bf16(out[b:b + 1], ref)
        assert np.abs(lse[b:b + 1] - ref_lse).max() < 1e-3


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("out_dtype", [torch.bfloat16, torch.float32])
def test_padded_forward_empty_batch_element(d, out_dtype):
    from paper_2112_05682_b200 import api
    B, n, H = 2, 200, 2
    q, k, v = Hh.host_inputs(B, n, n, H, d, seed=52)
    out, lse = api.mea_attention_fwd_padded(Hh.to_dev(q, torch.bfloat16), Hh.to_dev(k, torch.bfloat16),
                                            Hh.to_dev(v, torch.bfloat16), _lens([0, 150]), want_lse=True,
                                            out_dtype=out_dtype)
    torch.cuda.synchronize()
    assert (out[0] == 0).all() and torch.isinf(lse[0]).all() and (lse[0] < 0).all()
    ref, _ = O.mha_forward(q[1:], k[1:, :150], v[1:, :150], 1 / math.sqrt(d))
    Hh.assert_close_bf16(out[1:].double().cpu().numpy(), ref)


@pytest.mark.parametrize("d,lse_given", [(64, True), (64, False), (128, True), (128, False)])
def test_padded_backward_empty_batch_element(d, lse_given):
    """A batch element with no keys: its dq, dk and dv are exactly 0 (P = 0 everywhere, and the
    recomputed lse is -inf), the other element matches the oracle."""
    from paper_2112_05682_b200 import api
    B, n, H = 2, 200, 2
    lens = [0, 150]
    q, k, v, do = Hh.host_inputs(B, n, n, H, d, seed=54, with_dout=True)
    qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    kl = _lens(lens)
    out, lse = api.mea_attention_fwd_padded(qd, kd, vd, kl, want_lse=True)
    dq, dk, dv = api.mea_attention_bwd_padded(qd, kd, vd, out, dod, kl, lse=lse if lse_given else None)
    torch.cuda.synchronize()
    for x, nm in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
        assert (x[0] == 0).all(), f"{nm} of the empty element"
        assert (x[1, 150:] == 0).all() if nm != "dq" else True
    dq, dk, dv = (x.double().cpu().numpy() for x in (dq, dk, dv))
    rq, rk, rv = O.mha_backward(q[1:], k[1:, :150], v[1:, :150], do[1:], 1 / math.sqrt(d))
    for got, ref, nm in ((dq[1:], rq, "dq"), (dk[1:, :150], rk, "dk"), (dv[1:, :150], rv, "dv")):
        Hh.assert_close_bf16(got, ref, abs_tol=Hh.TOL_BF16_GRAD, rel_tol=Hh.REL_NORM_GRAD, what=nm)


@pytest.mark.parametrize("d,lse_given", [(64, True), (64, False), (128, True)])
def test_padded_backward_matches_oracle(d, lse_given):
    from paper_2112_05682_b200 import api
    B, n_q, n_k, H = 3, 300, 700, 2
    lens = [700, 129, 1]
    q, k, v, do = Hh.host_inputs(B, n_q, n_k, H, d, seed=53, with_dout=True)
    scale = 1 / math.sqrt(d)
    qd, kd, vd, dod = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    kl = _lens(lens)
    out, lse = api.mea_attention_fwd_padded(qd, kd, vd, kl, want_lse=True)
    dq, dk, dv = api.mea_attention_bwd_padded(qd, kd, vd, out, dod, kl, lse=lse if lse_given else None)
    torch.cuda.synchronize()
    dq, dk, dv = (x.double().cpu().numpy() for x in (dq, dk, dv))
    for b, L in enumerate(lens):
        rq, rk, rv = O.mha_backward(q[b:b + 1], k[b:b + 1, :L], v[b:b + 1, :L], do[b:b + 1], scale)
        for got, ref, nm in ((dq[b:b + 1], rq, "dq"), (dk[b:b + 1, :L], rk, "dk"), (dv[b:b + 1, :L], rv, "dv")):
            Hh.assert_close_bf16(got, ref, abs_tol=Hh.TOL_BF16_GRAD, rel_tol=Hh.REL_NORM_GRAD, what=nm)
        assert (dk[b, L:] == 0).all() and (dv[b, L:] == 0).all()


def test_padded_full_lengths_equal_unpadded():
    """kv_lens = n_k everywhere is the unpadded call, bit for bit (same kernels, no key masked)."""
    from paper_2112_05682_b200 import api
    B, n, H, d = 2, 1000, 2, 64
    q, k, v, do = (Hh.to_dev(x, torch.bfloat16) for x in Hh.host_inputs(B, n, n, H, d, seed=54, with_dout=True))
    kl = _lens([n, n])
    a, la = api.mea_attention_fwd_padded(q, k, v, kl, want_lse=True)
    b_, lb = api.mea_attention_fwd(q, k, v, want_lse=True)
    assert torch.equal(a, b_) and torch.equal(la, lb)
    ga = api.mea_attention_bwd_padded(q, k, v, a, do, kl, lse=la)
    gb = api.mea_attention_bwd(q, k, v, b_, do, lse=lb)
    for x, y in zip(ga, gb):
        assert (x.float() - y.float()).abs().max().item() < 2e-2  # dQ reduction order may differ


def test_padded_rejects_bad_arguments():
    from paper_2112_05682_b200 import api
    q = torch.zeros(2, 8, 1, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(TypeError):
        api.mea_attention_fwd_padded(q, q, q, torch.tensor([8, 8], dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError):
        api.mea_attention_fwd_padded(q, q, q, _lens([8]))
    with pytest.raises(api.MeaError):
        api.mea_attention_fwd_padded(q.float(), q.float(), q.float(), _lens([8, 8]))
