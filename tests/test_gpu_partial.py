"""GPU parity of the key-range building blocks of sharded self-attention:
mea_attention_partial_fwd (the stream triple (m*, s*, v*) of every query row over one key range,
PAPER.md:85-90) and mea_merge_partials over the ranges, against the float64
oracle (O5 partial_triple / merge, O1 naive) on the same generated inputs.

The reference max m* of the kernel may lag the true max (lazy rescale, reading 9), so
the triple is compared through the quantities that do not depend on it: v*/s* (attention over
the range) and m* + log s* (the range's log-sum-exp).
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
from tests import helpers as Hh

pytestmark = pytest.mark.gpu


def _partial(q, k, v, scale):
    from paper_2112_05682_b200 import api
    m, s, vs = api.mea_attention_partial_fwd(Hh.to_dev(q, torch.bfloat16), Hh.to_dev(k, torch.bfloat16),
                                             Hh.to_dev(v, torch.bfloat16), scale=scale)
    torch.cuda.synchronize()
    return m, s, vs


@pytest.mark.parametrize("B,n_q,n_k,H", [(1, 1, 1, 1), (2, 300, 129, 2), (1, 257, 1000, 3)])
def test_partial_triple_matches_oracle(B, n_q, n_k, H):
    q, k, v = Hh.host_inputs(B, n_q, n_k, H, 64, seed=21)
    scale = 0.125
    m, s, vs = _partial(q, k, v, scale)
    m, s, vs = (x.double().cpu().numpy() for x in (m, s, vs))
    for b in range(B):
        for h in range(H):
            rm, rs, rv = O.partial_triple(q[b, :, h], k[b, :, h], v[b, :, h], scale)
            Hh.assert_close_bf16(vs[b, :, h] / s[b, :, h, None], rv / rs[:, None])
            assert np.abs((m[b, :, h] + np.log(s[b, :, h])) - (rm + np.log(rs))).max() < 1e-3


def test_partial_d128_ranges_merge_to_full_attention():
    """d = 128 (fwd128's triple epilogue): two ragged key ranges merged == attention over all keys."""
    from paper_2112_05682_b200 import api
    B, n_q, n_k, H, d = 1, 200, 700, 2, 128
    q, k, v = Hh.host_inputs(B, n_q, n_k, H, d, seed=24)
    ref, _ = O.mha_forward(q, k, v, 1 / math.sqrt(d))
    qd = Hh.to_dev(q, torch.bfloat16)
    parts = [api.mea_attention_partial_fwd(qd, Hh.to_dev(k[:, a:b], torch.bfloat16), Hh.to_dev(v[:, a:b], torch.bfloat16))
             for a, b in ((0, 300), (300, n_k))]
    out = api.mea_merge_partials(torch.stack([p_[0].reshape(-1) for p_ in parts]),
                                 torch.stack([p_[1].reshape(-1) for p_ in parts]),
                                 torch.stack([p_[2].reshape(-1, d) for p_ in parts]), B, n_q * H,
                                 out_dtype=torch.float32).reshape(B, n_q, H, d)
    torch.cuda.synchronize()
    Hh.assert_close_bf16(out.double().cpu().numpy(), ref)


def test_key_ranges_merge_to_full_attention():
    """Ragged key ranges, one of them empty, merged == attention over all keys."""
    from paper_2112_05682_b200 import api
    B, n_q, n_k, H = 2, 333, 1100, 2
    q, k, v = Hh.host_inputs(B, n_q, n_k, H, 64, seed=22)
    scale = 1 / 8
    ref, _ = O.mha_forward(q, k, v, scale)
    cuts = [0, 129, 129, 700, n_k]   # ranges [0,129), [129,129) empty, [129,700), [700,1100)
    parts = [_partial(q, k[:, a:b], v[:, a:b], scale) for a, b in zip(cuts[:-1], cuts[1:])]
    M = torch.stack([p[0].reshape(-1) for p in parts])
    S = torch.stack([p[1].reshape(-1) for p in parts])
    V = torch.stack([p[2].reshape(-1, 64) for p in parts])
    assert torch.isinf(parts[1][0]).all() and (parts[1][1] == 0).all() and (parts[1][2] == 0).all()
    for od in (torch.float32, torch.bfloat16):
        out = api.mea_merge_partials(M, S, V, B, n_q * H, out_dtype=od).reshape(B, n_q, H, 64)
        torch.cuda.synchronize()
        Hh.assert_close_bf16(out.double().cpu().numpy(), ref)


def test_sharded_self_attention_single_rank_equals_forward():
    """dist.sharded_self_attention without a process group (world 1): partial + merge over all
    keys == mea_attention_fwd within the bf16 tolerance; both against the oracle."""
    from paper_2112_05682_b200 import api, dist as mdist
    B, n_q, n_k, H = 1, 600, 2000, 2
    q, k, v = Hh.host_inputs(B, n_q, n_k, H, 64, seed=23)
    ref, _ = O.mha_forward(q, k, v, 1 / 8)
    qd, kd, vd = (Hh.to_dev(x, torch.bfloat16) for x in (q, k, v))
    a = mdist.sharded_self_attention(qd, kd, vd, scale=1 / 8)
    b = api.mea_attention_fwd(qd, kd, vd, scale=1 / 8)
    torch.cuda.synchronize()
    Hh.assert_close_bf16(a.double().cpu().numpy(), ref)
    assert (a.float() - b.float()).abs().max().item() < 1e-2


def test_partial_large_rows_sampled():
    """configs[2] shape (H = 16, n = 16384) split in two key halves: merged rows equal the oracle
    on sampled rows (full-size launch, the merge over 262144 rows)."""
    from paper_2112_05682_b200 import api
    from synth import gen
    B, n, H, d = 1, 16384, 16, 64
    q = torch.empty((B, n, H, d), dtype=torch.bfloat16, device="cuda")
    k, v = torch.empty_like(q), torch.empty_like(q)
    for t, tid in ((q, gen.TENSOR_Q), (k, gen.TENSOR_K), (v, gen.TENSOR_V)):
        api.mea_fill_synthetic(t, 0, tid)
    half = 9000
    p0 = api.mea_attention_partial_fwd(q, k[:, :half].contiguous(), v[:, :half].contiguous())
    p1 = api.mea_attention_partial_fwd(q, k[:, half:].contiguous(), v[:, half:].contiguous())
    out = api.mea_merge_partials(torch.stack([p0[0].reshape(-1), p1[0].reshape(-1)]),
                                 torch.stack([p0[1].reshape(-1), p1[1].reshape(-1)]),
                                 torch.stack([p0[2].reshape(-1, d), p1[2].reshape(-1, d)]), B, n * H,
                                 out_dtype=torch.float32).reshape(B, n, H, d)
    torch.cuda.synchronize()
    rows = np.array([0, 127, 128, 5000, 16383])
    kk = gen.normal_tensor((B, n, H, d), 0, gen.TENSOR_K, "bf16").astype(np.float64)
    vv = gen.normal_tensor((B, n, H, d), 0, gen.TENSOR_V, "bf16").astype(np.float64)
    for h in (0, 15):
        qr = gen.rows_of((B, n, H, d), 0, gen.TENSOR_Q, 0, rows, h)
        ref, _ = O.naive(qr, kk[0, :, h], vv[0, :, h], 1 / math.sqrt(d))
        Hh.assert_close_bf16(out[0, rows, h].double().cpu().numpy(), ref)


@pytest.mark.parametrize("d", [64, 128])
def test_packed_partials_merge_to_full_attention(d):
    """Packed records {v*, m, s} (the all-gather layout): self-attention over ragged key ranges,
    one empty, and single-query ranges, merged by mea_merge_triples == the oracle."""
    from paper_2112_05682_b200 import api
    B, n_q, n_k, H = 2, 150, 900, 2
    q, k, v = Hh.host_inputs(B, n_q, n_k, H, d, seed=25)
    scale = 1 / math.sqrt(d)
    ref, _ = O.mha_forward(q, k, v, scale)
    qd = Hh.to_dev(q, torch.bfloat16)
    cuts = [0, 300, 300, n_k]
    recs = torch.stack([api.mea_attention_partial_fwd_packed(qd, Hh.to_dev(k[:, a:b], torch.bfloat16),
                                                             Hh.to_dev(v[:, a:b], torch.bfloat16), scale=scale)
                        for a, b in zip(cuts[:-1], cuts[1:])])
    assert recs.shape == (3, B * n_q * H, d + 4)
    assert torch.isinf(recs[1, :, d]).all() and (recs[1, :, d + 1] == 0).all() and (recs[1, :, :d] == 0).all()
    out = api.mea_merge_triples(recs, out_dtype=torch.float32).reshape(B, n_q, H, d)
    torch.cuda.synchronize()
    Hh.assert_close_bf16(out.double().cpu().numpy(), ref)
    # the unpacked triple of one range carries the same numbers
    m, s, vs = api.mea_attention_partial_fwd(qd, Hh.to_dev(k[:, 300:], torch.bfloat16),
                                             Hh.to_dev(v[:, 300:], torch.bfloat16), scale=scale)
    torch.cuda.synchronize()
    assert torch.equal(recs[2, :, d], m.reshape(-1)) and torch.equal(recs[2, :, d + 1], s.reshape(-1))
    assert torch.equal(recs[2, :, :d], vs.reshape(-1, d))
    # single query: packed per-(b, h) records over key ranges
    qs = qd[:, 0].contiguous()
    srecs = torch.stack([api.mea_single_query_partial_packed(qs, Hh.to_dev(k[:, a:b], torch.bfloat16),
                                                             Hh.to_dev(v[:, a:b], torch.bfloat16), scale=scale)
                         for a, b in zip(cuts[:-1], cuts[1:])])
    sout = api.mea_merge_triples(srecs, out_dtype=torch.float32).reshape(B, H, d)
    torch.cuda.synchronize()
    sref = np.stack([[O.naive(q[b, 0, h][None], k[b, :, h], v[b, :, h], scale)[0][0] for h in range(H)]
                     for b in range(B)])
    Hh.assert_close_bf16(sout.double().cpu().numpy(), sref)
