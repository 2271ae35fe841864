"""Shared test helpers: seeded inputs (synth) and tolerance checks. No method arithmetic."""
import math

import numpy as np
import torch

from synth import gen

# BASELINE.json north_star tolerances
TOL_F32_ABS, TOL_F32_REL = 1e-5, 1e-4
TOL_BF16_OUT, TOL_BF16_GRAD = 2e-2, 5e-2
# extra relative-norm guards: absolute bars are loose at large n
REL_NORM_OUT, REL_NORM_GRAD = 1e-2, 2e-2


def host_inputs(B, n_q, n_k, H, d, seed=0, dtype="bf16", with_dout=False):
    """Generator values (f64 arrays holding the exact input values)."""
    q = gen.normal_tensor((B, n_q, H, d), seed, gen.TENSOR_Q, dtype).astype(np.float64)
    k = gen.normal_tensor((B, n_k, H, d), seed, gen.TENSOR_K, dtype).astype(np.float64)
    v = gen.normal_tensor((B, n_k, H, d), seed, gen.TENSOR_V, dtype).astype(np.float64)
    if with_dout:
        do = gen.normal_tensor((B, n_q, H, d), seed, gen.TENSOR_DO, dtype).astype(np.float64)
        return q, k, v, do
    return q, k, v


def to_dev(x, dtype):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dtype).cuda()


def rel_norm(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))


BF16_STORE = 2.0 ** -8   # one bf16 rounding of a stored result (half-ulp is 2^-9 relative)


STRICT_REF = 4.0   # |ref| up to which reading 17's 2^-8|ref| term must not be needed


def assert_close_bf16(got, ref, abs_tol=TOL_BF16_OUT, rel_tol=REL_NORM_OUT, what="out", strict=True, extra=None):
    """|got - ref| <= abs_tol + 2^-8 |ref| element-wise (reading 17: a value stored
    in bf16 is only defined to within its own rounding), plus a relative-norm guard.

    strict (default): ALSO the unmodified north-star bar (2e-2 outputs, 5e-2 gradients, no
    2^-8|ref| term) on every element with |ref| <= 4, i.e. where readings 16/17 claim no effect.
    Pass strict=False only where reading 16 applies (|scale| > 1/sqrt(d)).

    extra: an element-wise allowance (array like ref) added to both bars — the first-order bound
    of bf16-rounded MMA operands for a gradient (reading 16; tests/test_gpu_fuzz.py)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    diff = np.abs(got - ref)
    err = float(diff.max()) if diff.size else 0.0
    rn = rel_norm(got, ref)
    ex = 0.0 if extra is None else np.asarray(extra, dtype=np.float64)
    assert np.isfinite(got).all(), f"{what}: non-finite values"
    bad = diff > abs_tol + ex + BF16_STORE * np.abs(ref)
    assert not bad.any(), f"{what}: max abs err {err:.3e} > {abs_tol} + 2^-8|ref| at {int(bad.sum())} elements"
    if strict:
        bar = TOL_BF16_GRAD if abs_tol >= TOL_BF16_GRAD else TOL_BF16_OUT
        bar = min(bar, abs_tol)
        small = np.abs(ref) <= STRICT_REF
        if small.any():
            over = (diff - ex)[small]
            e_small = float(over.max())
            assert e_small <= bar, f"{what}: strict north-star bar {bar} broken where |ref| <= 4: {e_small:.3e}"
    if np.linalg.norm(ref) > 1e-6 * np.sqrt(ref.size):   # an exactly-zero reference has no relative scale
        if extra is not None:   # the allowance bounds each element's error, so its norm bounds the error's
            rel_tol = max(rel_tol, float(np.linalg.norm(ex) / np.linalg.norm(ref)))
        assert rn <= rel_tol, f"{what}: relative norm err {rn:.3e} > {rel_tol}"
    return err, rn


def assert_close_f32(got, ref, what="out"):
    got = np.asarray(got, dtype=np.float64)
    err = np.abs(got - ref)
    bad = err > TOL_F32_ABS + TOL_F32_REL * np.abs(ref)
    assert not bad.any(), f"{what}: max abs err {err.max():.3e} (abs {TOL_F32_ABS}, rel {TOL_F32_REL})"
    assert err.max() <= TOL_F32_ABS, f"{what}: max abs err {err.max():.3e} > {TOL_F32_ABS}"
    return float(err.max())
