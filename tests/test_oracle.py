"""Pins for the float64 oracle (DESIGN.md "Oracle pins" P1-P10).

Each test checks the oracle against something other than itself: closed forms,
special cases, invariants, independent algorithms (brute force on tiny inputs),
an independent library implementation (torch float64 SDPA / autograd), and
finite differences. "P:n" = PAPER.md line n, "S:n" = SPEC.md line n.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle as O
from synth import gen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")


def _rand(rng, *shape):
    return rng.standard_normal(shape)


# ---------------------------------------------------------------- P4 closed forms
def test_closed_forms_golden():
    data = json.load(open(GOLDEN))
    for case in data["cases"]:
        q, k, v = (np.array(case[x]) for x in ("q", "k", "v"))
        if "expected" in case:
            want = np.array([[case["expected"]]])
        elif "expected_vec" in case:
            want = np.array([case["expected_vec"]])
        else:  # scores [3,1,5]
            e = math.e
            want = np.array([[(1 * e**3 + 2 * e + 3 * e**5) / (e**3 + e + e**5)]])
        for fn in (lambda: O.naive(q, k, v, case["scale"])[0],
                   lambda: O.sequential(q, k, v, case["scale"])[0],
                   lambda: O.chunked(q, k, v, case["scale"], 1, 1),
                   lambda: O.stream_finalize(O.single_query(q[0], k, v, case["scale"]))[None]):
            np.testing.assert_allclose(fn(), want, rtol=1e-14, atol=1e-14, err_msg=case["name"])


def test_stream_states_golden():
    data = json.load(open(GOLDEN))["stream_states"]
    st = O.stream_init(2)
    assert st[1] == 0.0 and st[2] == -math.inf and not st[0].any()     # P:87 / S:163
    for (score, vi), after in zip(data["updates"], data["after"]):
        st = O.stream_update(st, score, np.array(vi))
        assert list(st[0]) == after["v_star"]
        assert st[1] == after["s_star"] and st[2] == after["m_star"]
    assert list(O.stream_finalize(st)) == data["finalized"]


def test_empty_keys_is_an_error():
    with pytest.raises(O.EmptyKeysError):
        O.stream_finalize(O.stream_init(3))
    with pytest.raises(O.EmptyKeysError):
        O.naive(np.ones((2, 3)), np.ones((0, 3)), np.ones((0, 3)), 1.0)
    with pytest.raises(O.EmptyKeysError):
        O.sequential(np.ones((2, 3)), np.ones((0, 3)), np.ones((0, 3)), 1.0)


# ---------------------------------------------------------------- P2 / P3 special cases
def test_single_key_returns_value_exactly(rng):
    q, k, v = _rand(rng, 5, 4), _rand(rng, 1, 4), _rand(rng, 1, 6)
    for out in (O.naive(q, k, v, 0.5)[0], O.sequential(q, k, v, 0.5)[0], O.chunked(q, k, v, 0.5, 2, 3)):
        assert np.array_equal(out, np.repeat(v, 5, axis=0))


def test_identical_keys_or_zero_scale_give_mean(rng):
    q, v = _rand(rng, 6, 4), _rand(rng, 9, 3)
    k = np.repeat(_rand(rng, 1, 4), 9, axis=0)
    np.testing.assert_allclose(O.naive(q, k, v, 0.7)[0], np.repeat(v.mean(0, keepdims=True), 6, 0), atol=1e-14)
    k2 = _rand(rng, 9, 4)
    np.testing.assert_allclose(O.sequential(q, k2, v, 0.0)[0], np.repeat(v.mean(0, keepdims=True), 6, 0), atol=1e-14)
    np.testing.assert_allclose(O.naive(np.zeros((2, 4)), k2, v, 1.0)[0], np.repeat(v.mean(0, keepdims=True), 2, 0), atol=1e-14)


# ---------------------------------------------------------------- P1 brute force
@pytest.mark.parametrize("n_q,n_k,d", [(1, 1, 1), (3, 7, 2), (17, 33, 8), (40, 64, 16), (5, 129, 3)])
def test_definition_sequential_chunked_agree(rng, n_q, n_k, d):
    q, k, v = _rand(rng, n_q, d), _rand(rng, n_k, d), _rand(rng, n_k, d)
    scale = 1 / math.sqrt(d)
    ref, lse = O.naive(q, k, v, scale)
    np.testing.assert_allclose(O.sequential(q, k, v, scale)[0], ref, atol=1e-12, rtol=0)
    for kc in (1, 3, 7, n_k, 4096):
        for qc in (1, 3, n_q, 1024):
            np.testing.assert_allclose(O.chunked(q, k, v, scale, qc, kc), ref, atol=1e-12, rtol=0)
    for i in range(n_q):   # the literal per-query stream
        np.testing.assert_allclose(O.stream_finalize(O.single_query(q[i], k, v, scale)), ref[i], atol=1e-12)


def test_definition_matches_independent_pure_python(rng):
    """Brute force in plain Python floats (math.exp, math.fsum), no numpy, tiny sizes."""
    q, k, v = _rand(rng, 4, 3), _rand(rng, 6, 3), _rand(rng, 6, 2)
    ref, lse = O.naive(q, k, v, 0.9)
    for i in range(4):
        s = [0.9 * math.fsum(q[i][f] * k[j][f] for f in range(3)) for j in range(6)]
        w = [math.exp(x) for x in s]                  # scores are O(1): no overflow here
        z = math.fsum(w)
        for f in range(2):
            assert abs(math.fsum(w[j] * v[j][f] for j in range(6)) / z - ref[i, f]) < 1e-13
        assert abs(math.log(z) - lse[i]) < 1e-13      # P9: lse = log sum exp


def test_definition_matches_torch_sdpa_f64(rng):
    """Independent library implementation (torch CPU float64 math SDPA)."""
    B, n_q, n_k, H, d = 2, 37, 53, 3, 16
    q, k, v = _rand(rng, B, n_q, H, d), _rand(rng, B, n_k, H, d), _rand(rng, B, n_k, H, d)
    out, lse = O.mha_forward(q, k, v, 1 / math.sqrt(d))
    t = lambda x: torch.from_numpy(x).permute(0, 2, 1, 3)      # [B,H,n,d]
    ref = torch.nn.functional.scaled_dot_product_attention(t(q), t(k), t(v)).permute(0, 2, 1, 3).numpy()
    np.testing.assert_allclose(out, ref, atol=1e-12, rtol=0)
    s = torch.einsum("bhqd,bhkd->bhqk", t(q), t(k)) / math.sqrt(d)
    np.testing.assert_allclose(lse, torch.logsumexp(s, dim=-1).numpy(), atol=1e-12, rtol=0)


def test_merge_over_disjoint_key_ranges(rng):
    q, k, v = _rand(rng, 9, 5), _rand(rng, 50, 5), _rand(rng, 50, 4)
    ref = O.naive(q, k, v, 0.4)[0]
    cuts = [0, 0, 7, 8, 30, 50, 50]        # includes empty ranges
    parts = [O.partial_triple(q, k[a:b], v[a:b], 0.4) for a, b in zip(cuts[:-1], cuts[1:])]
    m, s, vs = (np.stack([p[i] for p in parts]) for i in range(3))
    np.testing.assert_allclose(O.merge(m, s, vs), ref, atol=1e-12)
    # the stream state equals the closed-form triple
    vst, sst, mst = O.sequential(q, k, v, 0.4)[1]
    m1, s1, v1 = O.partial_triple(q, k, v, 0.4)
    np.testing.assert_allclose(mst, m1, atol=1e-13)
    np.testing.assert_allclose(sst, s1, rtol=1e-12)
    np.testing.assert_allclose(vst, v1, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("n_k,kc", [(1, 1), (7, 1), (50, 7), (64, 1), (65, 8), (200, 13)])
def test_tree_summarization_equals_definition_with_log_memory(rng, n_k, kc):
    """O5t against the definition (O1): same out and lse; and the binary counter never
    holds more than floor(log2(chunks)) + 2 summaries (the O(log n) claim), which a flat
    Figure 1 merge (chunks summaries) exceeds as soon as chunks > 3."""
    q, k, v = _rand(rng, 6, 5), _rand(rng, n_k, 5), _rand(rng, n_k, 3)
    ref, ref_lse = O.naive(q, k, v, 0.7)
    out, lse, alive = O.tree_summarize(q, k, v, 0.7, kc)
    np.testing.assert_allclose(out, ref, atol=1e-12)
    np.testing.assert_allclose(lse, ref_lse, atol=1e-12)
    chunks = -(-n_k // kc)
    assert alive <= int(math.floor(math.log2(chunks))) + 2
    if chunks == 2 ** 6:   # all levels full just before the last carry: the bound is attained
        assert alive == 7
    # merge2 of a summary with an empty one is the identity; merge2 is the P = 2 case of O5
    a = O.partial_triple(q, k, v, 0.7)
    e = O.partial_triple(q, k[:0], v[:0], 0.7)
    for x, y in zip(O.merge2(a, e), a):
        np.testing.assert_allclose(x, y, atol=1e-15)
    b1, b2 = O.partial_triple(q, k[: n_k // 2], v[: n_k // 2], 0.7), O.partial_triple(q, k[n_k // 2:], v[n_k // 2:], 0.7)
    if n_k >= 2:
        m, s_, vs = O.merge2(b1, b2)
        np.testing.assert_allclose(vs / s_[:, None], O.merge(*(np.stack([b1[i], b2[i]]) for i in range(3))), atol=1e-12)


# ---------------------------------------------------------------- P5 / P6 shift and stability
def _shifted(q, k, c):
    """Append a feature so every score of every row gets +c exactly (scale 1)."""
    return (np.hstack([q, np.full((q.shape[0], 1), c)]), np.hstack([k, np.ones((k.shape[0], 1))]))


@pytest.mark.parametrize("c", [-50.0, -3.0, 2.5, 50.0])
def test_shift_invariance(rng, c):
    q, k, v = _rand(rng, 7, 4), _rand(rng, 11, 4), _rand(rng, 11, 3)
    ref = O.naive(q, k, v, 1.0)[0]
    qs, ks = _shifted(q, k, c)
    for out in (O.naive(qs, ks, v, 1.0)[0], O.sequential(qs, ks, v, 1.0)[0], O.chunked(qs, ks, v, 1.0, 3, 4)):
        np.testing.assert_allclose(out, ref, atol=1e-12)


@pytest.mark.parametrize("c", [-1000.0, 1000.0])
def test_stability_at_huge_scores(rng, c):
    """with the max subtracted, scores near +-1000 are harmless; Eq.(1) is not."""
    q, k, v = _rand(rng, 5, 3), _rand(rng, 8, 3), _rand(rng, 8, 2)
    ref = O.naive(q, k, v, 1.0)[0]
    qs, ks = _shifted(q, k, c)
    for out in (O.naive(qs, ks, v, 1.0)[0], O.sequential(qs, ks, v, 1.0)[0], O.chunked(qs, ks, v, 1.0, 2, 3)):
        assert np.isfinite(out).all()
        np.testing.assert_allclose(out, ref, atol=1e-10)
    assert not np.isfinite(O.lazy_unstable(qs, ks, v, 1.0)).all()
    # small scores: Eq.(1) is exact (negative control is a real implementation)
    np.testing.assert_allclose(O.lazy_unstable(q, k, v, 1.0), ref, atol=1e-12)


def test_paper_overflow_threshold_f32():
    """"For scores >= 89 the exponentiation results in inf"."""
    out = O.lazy_unstable(np.array([[1.0]]), np.array([[89.0]]), np.array([[7.0]]), 1.0, dtype=np.float32)
    assert not np.isfinite(out).all()
    assert O.naive(np.array([[1.0]]), np.array([[89.0]]), np.array([[7.0]]), 1.0)[0][0, 0] == 7.0
    out = O.lazy_unstable(np.array([[1.0]]), np.array([[88.0], [0.0]]), np.array([[1.0], [0.5]]), 1.0, dtype=np.float32)
    assert np.isfinite(out).all()


# ---------------------------------------------------------------- P7 permutation
def test_permutation_invariance(rng):
    q, k, v = _rand(rng, 6, 4), _rand(rng, 23, 4), _rand(rng, 23, 5)
    perm = rng.permutation(23)
    a = O.sequential(q, k, v, 0.5)[0]
    b = O.sequential(q, k[perm], v[perm], 0.5)[0]
    np.testing.assert_allclose(a, b, atol=1e-12)


# ---------------------------------------------------------------- P8 gradients
@pytest.mark.parametrize("n_q,n_k,d", [(3, 5, 2), (8, 8, 4), (4, 16, 8)])
def test_backward_matches_finite_differences(rng, n_q, n_k, d):
    q, k, v, do = _rand(rng, n_q, d), _rand(rng, n_k, d), _rand(rng, n_k, d), _rand(rng, n_q, d)
    scale = 1 / math.sqrt(d)
    an = O.backward(q, k, v, do, scale)
    fd = O.fd_grad(q, k, v, do, scale)
    for a, f in zip(an, fd):
        assert np.abs(a - f).max() <= 1e-5 * max(1.0, np.abs(f).max())
        assert np.linalg.norm(a - f) <= 1e-5 * np.linalg.norm(f) + 1e-9


def test_backward_matches_torch_autograd(rng):
    n_q, n_k, d = 13, 21, 8
    q, k, v, do = _rand(rng, n_q, d), _rand(rng, n_k, d), _rand(rng, n_k, d), _rand(rng, n_q, d)
    tq, tk, tv = (torch.tensor(x, requires_grad=True) for x in (q, k, v))
    out = torch.softmax(0.3 * tq @ tk.T, dim=-1) @ tv
    out.backward(torch.from_numpy(do))
    for a, t in zip(O.backward(q, k, v, do, 0.3), (tq, tk, tv)):
        np.testing.assert_allclose(a, t.grad.numpy(), atol=1e-12)


def test_backward_special_cases(rng):
    q, k, v, do = _rand(rng, 4, 3), _rand(rng, 1, 3), _rand(rng, 1, 3), _rand(rng, 4, 3)
    dq, dk, dv = O.backward(q, k, v, do, 1.0)           # n_k = 1: weight is constant 1
    assert not dq.any() and not dk.any()
    np.testing.assert_allclose(dv, do.sum(0, keepdims=True), atol=1e-15)
    k2, v2 = _rand(rng, 6, 3), _rand(rng, 6, 3)
    for g in O.backward(q, k2, v2, np.zeros((4, 3)), 1.0):
        assert not g.any()
    # delta identity: sum_j P_ij dP_ij = dO_i . O_i
    out = O.naive(q, k2, v2, 1.0)[0]
    s = O.scores(q, k2, 1.0)
    p = np.exp(s - s.max(1, keepdims=True)); p /= p.sum(1, keepdims=True)
    np.testing.assert_allclose((p * (do @ v2.T)).sum(1), O.delta_rowsum(out, do), atol=1e-13)


# ---------------------------------------------------------------- P10 generator
def test_generator_statistics_and_determinism():
    x = gen.normal_tensor((4096, 64), 42, gen.TENSOR_Q, "f64")
    assert abs(x.mean()) < 0.05 and abs(x.std() - 1) < 0.05
    assert np.abs(x).max() < 6
    assert np.array_equal(x, gen.normal_tensor((4096, 64), 42, gen.TENSOR_Q, "f64"))
    assert not np.array_equal(x, gen.normal_tensor((4096, 64), 43, gen.TENSOR_Q, "f64"))
    # values are multiples of 2^-16 (exact in f32)
    assert np.array_equal(x * 65536, np.round(x * 65536))
    assert np.array_equal(x.astype(np.float32).astype(np.float64), x)


def test_generator_bf16_rounding_is_rne():
    x = np.array([1.0 + 2**-8, 1.0 + 3 * 2**-8, -(1.0 + 2**-8), 1.0 + 2**-8 + 2**-16])
    want = np.array([1.0, 1.0 + 2**-6, -1.0, 1.0 + 2**-7])
    np.testing.assert_array_equal(gen.round_to_bf16(x), want.astype(np.float32))
    t = torch.from_numpy(gen.normal_tensor((1000,), 3, 2, "f64")).to(torch.bfloat16).float().numpy()
    np.testing.assert_array_equal(gen.normal_tensor((1000,), 3, 2, "bf16"), t)


def test_generator_row_sampling_matches_full_tensor():
    shape = (2, 37, 3, 8)
    full = gen.normal_tensor(shape, 7, gen.TENSOR_K, "bf16")
    rows = np.array([0, 5, 36])
    np.testing.assert_array_equal(gen.rows_of(shape, 7, gen.TENSOR_K, 1, rows, 2), full[1, rows, 2])


def test_backward_rows_equals_full_backward(rng):
    n_q, n_k, d = 37, 29, 8
    q, k, v, do = _rand(rng, n_q, d), _rand(rng, n_k, d), _rand(rng, n_k, d), _rand(rng, n_q, d)
    dq, dk, dv = O.backward(q, k, v, do, 0.4)
    qr, kr = np.array([0, 5, 36]), np.array([1, 28])
    sq, sk, sv = O.backward_rows(q, k, v, do, 0.4, qr, kr, block=10)
    np.testing.assert_allclose(sq, dq[qr], atol=1e-12)
    np.testing.assert_allclose(sk, dk[kr], atol=1e-12)
    np.testing.assert_allclose(sv, dv[kr], atol=1e-12)


# ---------------------------------------------------------------- causal masking
def test_causal_rows_equal_the_stream_over_their_prefix(rng):
    """Causal row i == the paper's sequential stream algorithm (O3) over keys 0..i —
    a different algorithm on a sliced input, not the masked definition again. Row 0 = v_0."""
    n, d = 23, 8
    q, k, v = _rand(rng, n, d), _rand(rng, n, d), _rand(rng, n, d)
    out, lse = O.naive(q, k, v, 0.7, causal=True)
    for i in range(n):
        ref = O.sequential(q[i:i + 1], k[:i + 1], v[:i + 1], 0.7)[0]
        np.testing.assert_allclose(out[i], ref[0], atol=1e-12)
        assert abs(lse[i] - np.log(np.exp(0.7 * (q[i] @ k[:i + 1].T)).sum())) < 1e-12
    np.testing.assert_array_equal(out[0], v[0])
    sub, sub_lse = O.naive(q, k, v, 0.7, rows=[3, 17], causal=True)
    np.testing.assert_allclose(sub, out[[3, 17]], atol=1e-14)


def test_causal_matches_torch_sdpa_f64(rng):
    """Independent library implementation: torch float64 SDPA with is_causal=True."""
    B, n, H, d = 2, 33, 3, 16
    q, k, v = _rand(rng, B, n, H, d), _rand(rng, B, n, H, d), _rand(rng, B, n, H, d)
    out, _ = O.mha_forward(q, k, v, 1 / math.sqrt(d), causal=True)
    t = lambda x: torch.from_numpy(x).permute(0, 2, 1, 3)
    ref = torch.nn.functional.scaled_dot_product_attention(t(q), t(k), t(v), is_causal=True)
    np.testing.assert_allclose(out, ref.permute(0, 2, 1, 3).numpy(), atol=1e-12, rtol=0)


def test_causal_backward_matches_fd_and_autograd(rng):
    n, d = 9, 4
    q, k, v, do = _rand(rng, n, d), _rand(rng, n, d), _rand(rng, n, d), _rand(rng, n, d)
    an = O.backward(q, k, v, do, 0.5, causal=True)
    fd = O.fd_grad(q, k, v, do, 0.5, causal=True)
    for a, f in zip(an, fd):
        assert np.abs(a - f).max() <= 1e-5 * max(1.0, np.abs(f).max())
    tq, tk, tv = (torch.tensor(x, requires_grad=True) for x in (q, k, v))
    s = 0.5 * tq @ tk.T
    s = s.masked_fill(torch.triu(torch.ones(n, n, dtype=torch.bool), 1), float("-inf"))
    (torch.softmax(s, dim=-1) @ tv).backward(torch.from_numpy(do))
    for a, t in zip(an, (tq, tk, tv)):
        np.testing.assert_allclose(a, t.grad.numpy(), atol=1e-12)
    # the last key is seen by the last query only: dv_{n-1} = P_{n-1,n-1} dO_{n-1}
    p_last = np.exp(0.5 * q[-1] @ k.T - O.naive(q, k, v, 0.5, causal=True)[1][-1])[-1]
    np.testing.assert_allclose(an[2][-1], p_last * do[-1], atol=1e-12)
    qr, kr = np.array([0, 4, 8]), np.array([0, 3, 8])
    sq, sk, sv = O.backward_rows(q, k, v, do, 0.5, qr, kr, block=4, causal=True)
    np.testing.assert_allclose(sq, an[0][qr], atol=1e-12)
    np.testing.assert_allclose(sk, an[1][kr], atol=1e-12)
    np.testing.assert_allclose(sv, an[2][kr], atol=1e-12)


# ---------------------------------------------------------------- P8 on the library layout
def _autograd_mha(q, k, v, do, scale, causal):
    """torch float64 autograd of softmax attention on [B, n, H, d] (an independent library path:
    einsum over the head axis, no per-(b,h) slicing)."""
    tq, tk, tv = (torch.tensor(x, requires_grad=True) for x in (q, k, v))
    s = scale * torch.einsum("bqhd,bkhd->bhqk", tq, tk)
    if causal:
        n_q, n_k = q.shape[1], k.shape[1]
        s = s.masked_fill(torch.triu(torch.ones(n_q, n_k, dtype=torch.bool), 1), float("-inf"))
    out = torch.einsum("bhqk,bkhd->bqhd", torch.softmax(s, dim=-1), tv)
    out.backward(torch.from_numpy(do))
    return out.detach().numpy(), tq.grad.numpy(), tk.grad.numpy(), tv.grad.numpy()


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("n_q,n_k", [(7, 11), (9, 9)])
def test_mha_backward_matches_autograd_on_library_layout(rng, causal, n_q, n_k):
    """mha_backward (the reference of every GPU backward parity test) on [B, n, H, d] with B, H > 1
    against torch autograd: a swapped dk/dv, a wrong [b, :, h] slice or a
    transposed head/batch index fails here."""
    if causal and n_q != n_k:
        pytest.skip("causal needs n_q == n_k")
    B, H, d = 2, 3, 5
    q, k, v = _rand(rng, B, n_q, H, d), _rand(rng, B, n_k, H, d), _rand(rng, B, n_k, H, d)
    do = _rand(rng, B, n_q, H, d)
    v = v * np.arange(1, d + 1)          # dv and dk differ in scale: a dk <-> dv swap cannot pass
    out_ref, gq, gk, gv = _autograd_mha(q, k, v, do, 0.7, causal)
    out, _ = O.mha_forward(q, k, v, 0.7, causal=causal)
    np.testing.assert_allclose(out, out_ref, atol=1e-12, rtol=0)
    dq, dk, dv = O.mha_backward(q, k, v, do, 0.7, causal=causal)
    for got, ref, nm in ((dq, gq, "dq"), (dk, gk, "dk"), (dv, gv, "dv")):
        assert got.shape == ref.shape, nm
        np.testing.assert_allclose(got, ref, atol=1e-12, rtol=0, err_msg=nm)


def test_mha_backward_equals_per_head_backward(rng):
    """Each (b, h) slice of mha_backward is O6 on that slice alone, and different heads differ."""
    B, n_q, n_k, H, d = 2, 6, 4, 3, 4
    q, k, v, do = (_rand(rng, B, n, H, d) for n in (n_q, n_k, n_k, n_q))
    dq, dk, dv = O.mha_backward(q, k, v, do, 0.5)
    for b in range(B):
        for h in range(H):
            r = O.backward(q[b, :, h], k[b, :, h], v[b, :, h], do[b, :, h], 0.5)
            for got, ref in zip((dq[b, :, h], dk[b, :, h], dv[b, :, h]), r):
                np.testing.assert_array_equal(got, ref)
    assert np.abs(dq[0, :, 0] - dq[0, :, 1]).max() > 1e-3 and np.abs(dq[0] - dq[1]).max() > 1e-3
