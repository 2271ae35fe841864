"""Counter-based, integer-exact input generator (host side).

value(seed, tensor_id, i) for flat element index i of a tensor:

  1. base = mix64(seed * G + tensor_id * H)                 (all arithmetic mod 2^64)
  2. z_r  = mix64(base + (3*i + r + 1) * G)   for r = 0, 1, 2
  3. u_0..u_11 = the twelve 16-bit limbs of z_0, z_1, z_2 (low limb first)
  4. x = (sum_k u_k + 6) / 65536 - 6                        (Irwin-Hall(12) - 6)

mix64 is the splitmix64 finaliser; G = 0x9E3779B97F4A7C15, H = 0xD1B54A32D192ED03.
Step 4 is exact in binary floating point: x is a multiple of 2^-16 with |x| < 6, so
it has at most 19 significant bits and is representable in f32 and f64 exactly.
Rounding to bf16 is round-to-nearest-even of that exact value. Hence any
independent implementation (the CUDA one in csrc/gen_inputs.cu) is bit-identical.

x has mean 0 and variance 1 (12 uniforms of variance 1/12 each), bounded in
(-6, 6): the paper's "inputs drawn from a normal distribution with standard
deviation 1" (Sec. 5.1) with a bounded tail.

Tensor ids: q=1, k=2, v=3, dO=4.
"""
import numpy as np

TENSOR_Q, TENSOR_K, TENSOR_V, TENSOR_DO = 1, 2, 3, 4

_G = np.uint64(0x9E3779B97F4A7C15)
_H = np.uint64(0xD1B54A32D192ED03)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix64(z):
    z = z ^ (z >> np.uint64(30))
    z = z * _M1
    z = z ^ (z >> np.uint64(27))
    z = z * _M2
    return z ^ (z >> np.uint64(31))


def irwin_hall_values(seed, tensor_id, flat_idx):
    """Exact generator values (float64) for the given flat indices (any int array)."""
    with np.errstate(over="ignore"):
        s = np.array([seed], dtype=np.uint64)
        t = np.array([tensor_id], dtype=np.uint64)
        base = _mix64(s * _G + t * _H)
        idx = np.asarray(flat_idx, dtype=np.uint64)
        acc = np.zeros(idx.shape, dtype=np.uint64)
        mask = np.uint64(0xFFFF)
        for r in range(3):
            z = _mix64(base + (np.uint64(3) * idx + np.uint64(r + 1)) * _G)
            for c in range(4):
                acc += (z >> np.uint64(16 * c)) & mask
    # acc <= 12*65535 < 2^20: exact in f64; /65536 is exact; -6 is exact.
    return (acc.astype(np.float64) + 6.0) / 65536.0 - 6.0


def round_to_bf16(x):
    """Round-to-nearest-even of float values to bf16; returns float32 holding the bf16 value."""
    f = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    b = f.view(np.uint32).astype(np.uint64)
    rounded = ((b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) << np.uint64(16)
    return rounded.astype(np.uint32).view(np.float32).reshape(f.shape)


def bf16_bits_to_f32(bits):
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32)


def normal_tensor(shape, seed, tensor_id, dtype="bf16", chunk=1 << 22):
    """Full tensor in row-major order of ``shape``. dtype in {"bf16","f32","f64"}.

    Returns a numpy float32 (bf16-valued for "bf16") or float64 array.
    """
    n = int(np.prod(shape)) if len(shape) else 1
    out = np.empty(n, dtype=np.float64 if dtype == "f64" else np.float32)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        x = irwin_hall_values(seed, tensor_id, np.arange(lo, hi, dtype=np.uint64))
        if dtype == "bf16":
            out[lo:hi] = round_to_bf16(x)
        else:
            out[lo:hi] = x  # exact in f32 and f64
    return out.reshape(shape)


def rows_of(shape, seed, tensor_id, b, rows, h, dtype="bf16"):
    """Rows ``rows`` (array of sequence indices) of head h, batch b of a [B,n,H,d] tensor.

    Regenerates only the requested elements (used to check sampled rows of configs
    too large to copy back).
    """
    B, n, H, d = shape
    rows = np.asarray(rows, dtype=np.int64)
    flat = ((b * n + rows)[:, None] * H + h) * d + np.arange(d)[None, :]
    x = irwin_hall_values(seed, tensor_id, flat.astype(np.uint64))
    return round_to_bf16(x).astype(np.float64) if dtype == "bf16" else x
