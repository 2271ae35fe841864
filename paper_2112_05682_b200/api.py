"""Thin Python binding over libmea.so: same names as include/mea.h, torch tensors in.

Argument marshalling only — shapes, dtypes, pointers, the current CUDA stream and
workspace allocation (torch owns every buffer). Every step of the method runs in the
library's CUDA kernels. Layouts: q/out [B, n_q, H, d]; k/v [B, n_k, H, d]; lse
[B, H, n_q]; single-query q/out [B, H, d].
"""
import ctypes
import math

import torch

from . import _lib

MEA_F32, MEA_BF16 = 0, 1
_DT = {torch.float32: MEA_F32, torch.bfloat16: MEA_BF16}
_TORCH = {MEA_F32: torch.float32, MEA_BF16: torch.bfloat16}

MEA_OK = 0
STATUS = {0: "MEA_OK", 1: "MEA_ERR_INVALID_VALUE", 2: "MEA_ERR_EMPTY_KEYS", 3: "MEA_ERR_UNSUPPORTED",
          4: "MEA_ERR_MISALIGNED", 5: "MEA_ERR_WORKSPACE_TOO_SMALL", 6: "MEA_ERR_CUDA"}


class MeaError(RuntimeError):
    def __init__(self, status, detail):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {detail}")


class EmptyKeysError(MeaError, ValueError):
    pass


def _check(status):
    if status != MEA_OK:
        detail = _lib.load().mea_last_error_detail().decode()
        if status == 2:
            raise EmptyKeysError(status, detail)
        raise MeaError(status, detail)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _dtype(t):
    if t.dtype not in _DT:
        raise TypeError(f"unsupported dtype {t.dtype}; use bfloat16 or float32")
    return _DT[t.dtype]


def _cuda_contig(*ts):
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda:
            raise ValueError("libmea takes CUDA tensors (no CPU fallback)")
        if not t.is_contiguous():
            raise ValueError("tensors must be contiguous")


def _expect(t, shape, dtype, name):
    """Caller-supplied tensors are read by the kernels with the dtype / shape the call implies:
    reject anything else instead of reinterpreting bytes or writing out of bounds."""
    if t is None:
        return
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")


def _expect_out(out, shape):
    if out is not None:
        if out.dtype not in (torch.bfloat16, torch.float32):
            raise TypeError(f"out must be bfloat16 or float32, got {out.dtype}")
        _expect(out, shape, None, "out")


def _workspace(nbytes, device):
    if nbytes == 0:
        return None
    return torch.empty(nbytes, dtype=torch.uint8, device=device)


def version():
    return _lib.load().mea_version().decode()


# ------------------------------------------------------------------------ forward
def mea_attention_fwd_workspace_size(B, H, n_q, n_k, d, in_dtype, q_chunk=0, k_chunk=0):
    n = ctypes.c_size_t(0)
    _check(_lib.load().mea_attention_fwd_workspace_size(B, H, n_q, n_k, d, in_dtype, q_chunk, k_chunk,
                                                        ctypes.byref(n)))
    return n.value


MEA_F32_SPLIT = 2
MEA_CHUNK_SQRT_N = -1   # k_chunk: the paper's sqrt(n) key chunk


def mea_attention_fwd_tree_workspace_size(B, H, n_q, n_k, d, in_dtype=MEA_BF16, q_chunk=0, k_chunk=MEA_CHUNK_SQRT_N):
    n = ctypes.c_size_t(0)
    _check(_lib.load().mea_attention_fwd_tree_workspace_size(B, H, n_q, n_k, d, in_dtype, q_chunk, k_chunk,
                                                             ctypes.byref(n)))
    return n.value


def mea_attention_fwd_tree(q, k, v, scale=None, out=None, out_dtype=None, lse=None, want_lse=False,
                           q_chunk=0, k_chunk=MEA_CHUNK_SQRT_N, workspace=None):
    """The paper's chunked forward with multi-stage (tree) summarisation: key chunks
    summarised one after another per query chunk and merged like a binary counter, so only
    O(log(n_k / k_chunk)) summaries per query row are alive. bf16 inputs, d in {64, 128}."""
    _cuda_contig(q, k, v, out, lse)
    B, n_q, H, d = q.shape
    n_k = k.shape[1]
    if k.shape != (B, n_k, H, d) or v.shape != k.shape:
        raise ValueError(f"shape mismatch q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)}")
    if k.dtype != q.dtype or v.dtype != q.dtype:
        raise TypeError("q, k, v must share a dtype")
    dt = _dtype(q)
    _expect_out(out, (B, n_q, H, d))
    _expect(lse, (B, H, n_q), torch.float32, "lse")
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    if out is None:
        out = torch.empty((B, n_q, H, d), dtype=q.dtype if out_dtype is None else out_dtype, device=q.device)
    if want_lse and lse is None:
        lse = torch.empty((B, H, n_q), dtype=torch.float32, device=q.device)
    if workspace is None:
        workspace = _workspace(mea_attention_fwd_tree_workspace_size(B, H, n_q, n_k, d, dt, q_chunk, k_chunk),
                               q.device)
    _check(_lib.load().mea_attention_fwd_tree(
        _ptr(q), _ptr(k), _ptr(v), _ptr(out), B, H, n_q, n_k, d, dt, _dtype(out), scale, _ptr(lse),
        q_chunk, k_chunk, _ptr(workspace), workspace.numel() if workspace is not None else 0, _stream(q.device)))
    return (out, lse) if (want_lse or lse is not None) else out


def mea_attention_fwd(q, k, v, scale=None, out=None, out_dtype=None, lse=None, want_lse=False,
                      q_chunk=0, k_chunk=0, workspace=None, f32_split=False):
    """out = attention(q, k, v) (Figure 1). Returns out, or (out, lse).
    f32_split: float32 inputs on the tensor cores by split precision (MEA_F32_SPLIT, mea.h)."""
    _cuda_contig(q, k, v, out, lse)
    B, n_q, H, d = q.shape
    n_k = k.shape[1]
    if k.shape != (B, n_k, H, d) or v.shape != k.shape:
        raise ValueError(f"shape mismatch q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)}")
    dt = _dtype(q)
    if f32_split:
        if dt != MEA_F32:
            raise TypeError("f32_split needs float32 inputs")
        dt = MEA_F32_SPLIT
    if k.dtype != q.dtype or v.dtype != q.dtype:
        raise TypeError("q, k, v must share a dtype")
    _expect_out(out, (B, n_q, H, d))
    _expect(lse, (B, H, n_q), torch.float32, "lse")
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    if out is None:
        od = q.dtype if out_dtype is None else out_dtype
        out = torch.empty((B, n_q, H, d), dtype=od, device=q.device)
    if want_lse and lse is None:
        lse = torch.empty((B, H, n_q), dtype=torch.float32, device=q.device)
    if workspace is None:
        workspace = _workspace(mea_attention_fwd_workspace_size(B, H, n_q, n_k, d, dt, q_chunk, k_chunk), q.device)
    _check(_lib.load().mea_attention_fwd(
        _ptr(q), _ptr(k), _ptr(v), _ptr(out), B, H, n_q, n_k, d, dt, _dtype(out), scale, _ptr(lse),
        q_chunk, k_chunk, _ptr(workspace), workspace.numel() if workspace is not None else 0, _stream(q.device)))
    return (out, lse) if (want_lse or lse is not None) else out


def mea_attention_fwd_causal(q, k, v, scale=None, out=None, out_dtype=None, lse=None, want_lse=False):
    """Causal self-attention (query i sees keys j <= i); q, k, v [B, n, H, d] bf16, d = 64."""
    _cuda_contig(q, k, v, out, lse)
    B, n, H, d = q.shape
    if k.shape != q.shape or v.shape != q.shape:
        raise ValueError(f"causal attention needs q, k, v of one shape, got {tuple(q.shape)} {tuple(k.shape)}")
    if k.dtype != q.dtype or v.dtype != q.dtype:
        raise TypeError("q, k, v must share a dtype")
    _expect_out(out, (B, n, H, d))
    _expect(lse, (B, H, n), torch.float32, "lse")
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    if out is None:
        out = torch.empty((B, n, H, d), dtype=q.dtype if out_dtype is None else out_dtype, device=q.device)
    if want_lse and lse is None:
        lse = torch.empty((B, H, n), dtype=torch.float32, device=q.device)
    _check(_lib.load().mea_attention_fwd_causal(_ptr(q), _ptr(k), _ptr(v), _ptr(out), B, H, n, d, _dtype(q),
                                                _dtype(out), scale, _ptr(lse), _stream(q.device)))
    return (out, lse) if (want_lse or lse is not None) else out


def mea_attention_partial_fwd(q, k, v, scale=None):
    """Stream state (m*, s*, v*) of every query row over this call's keys (one key range of a
    sharded self-attention). Returns m [B,n_q,H], s [B,n_q,H] and vstar [B,n_q,H,d], float32,
    m in natural-log units; merge ranges with mea_merge_partials(..., B, n_q * H)."""
    _cuda_contig(q, k, v)
    B, n_q, H, d = q.shape
    n_k = k.shape[1]
    if k.shape != (B, n_k, H, d) or v.shape != k.shape:
        raise ValueError(f"shape mismatch q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)}")
    if k.dtype != q.dtype or v.dtype != q.dtype:
        raise TypeError("q, k, v must share a dtype")
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    m = torch.empty((B, n_q, H), dtype=torch.float32, device=q.device)
    s = torch.empty((B, n_q, H), dtype=torch.float32, device=q.device)
    vs = torch.empty((B, n_q, H, d), dtype=torch.float32, device=q.device)
    _check(_lib.load().mea_attention_partial_fwd(_ptr(q), _ptr(k), _ptr(v), _ptr(m), _ptr(s), _ptr(vs), B, H, n_q,
                                                 n_k, d, _dtype(q), scale, _stream(q.device)))
    return m, s, vs


# ------------------------------------------------------------------------ single query
def mea_single_query_workspace_size(B, H, n_k, d, in_dtype):
    n = ctypes.c_size_t(0)
    _check(_lib.load().mea_single_query_workspace_size(B, H, n_k, d, in_dtype, ctypes.byref(n)))
    return n.value


def mea_single_query_fwd(q, k, v, scale=None, out=None, out_dtype=None, workspace=None):
    """Single-query attention per (b,h). q [B,H,d]; k,v [B,n_k,H,d]."""
    _cuda_contig(q, k, v, out)
    B, H, d = q.shape
    n_k = k.shape[1]
    if k.shape != (B, n_k, H, d) or v.shape != k.shape:
        raise ValueError(f"shape mismatch q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)}")
    if k.dtype != q.dtype or v.dtype != q.dtype:
        raise TypeError("q, k, v must share a dtype")
    dt = _dtype(q)
    _expect_out(out, (B, H, d))
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    if out is None:
        out = torch.empty((B, H, d), dtype=q.dtype if out_dtype is None else out_dtype, device=q.device)
    if workspace is None:
        workspace = _workspace(mea_single_query_workspace_size(B, H, max(n_k, 0), d, dt), q.device)
    _check(_lib.load().mea_single_query_fwd(
        _ptr(q), _ptr(k), _ptr(v), _ptr(out), B, H, n_k, d, dt, _dtype(out), scale, _ptr(workspace),
        workspace.numel() if workspace is not None else 0, _stream(q.device)))
    return out


def mea_single_query_partial(q, k, v, scale=None, workspace=None):
    """Per-(b,h) stream triple (m*, s*, v*) over these keys; m in natural-log units."""
    _cuda_contig(q, k, v)
    B, H, d = q.shape
    n_k = k.shape[1]
    if k.shape != (B, n_k, H, d) or v.shape != k.shape:
        raise ValueError(f"shape mismatch q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)}")
    if k.dtype != q.dtype or v.dtype != q.dtype:
        raise TypeError("q, k, v must share a dtype")
    dt = _dtype(q)
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    m = torch.empty(B * H, dtype=torch.float32, device=q.device)
    s = torch.empty(B * H, dtype=torch.float32, device=q.device)
    vs = torch.empty(B * H * d, dtype=torch.float32, device=q.device)
    if workspace is None:
        workspace = _workspace(mea_single_query_workspace_size(B, H, n_k, d, dt), q.device)
    _check(_lib.load().mea_single_query_partial(
        _ptr(q), _ptr(k), _ptr(v), _ptr(m), _ptr(s), _ptr(vs), B, H, n_k, d, dt, scale, _ptr(workspace),
        workspace.numel() if workspace is not None else 0, _stream(q.device)))
    return m, s, vs.view(B * H, d)


def mea_merge_partials(m, s, vstar, B, H, out_dtype=torch.bfloat16, out=None):
    """Merge P stacked triples m [P,B*H], s [P,B*H], vstar [P,B*H,d] -> out [B,H,d]."""
    _cuda_contig(m, s, vstar, out)
    P = m.shape[0]
    d = vstar.shape[-1]
    _expect(m, (P, B * H), torch.float32, "m")
    _expect(s, (P, B * H), torch.float32, "s")
    _expect(vstar, (P, B * H, d), torch.float32, "vstar")
    _expect_out(out, (B, H, d))
    if out is None:
        out = torch.empty((B, H, d), dtype=out_dtype, device=m.device)
    _check(_lib.load().mea_merge_partials(_ptr(m), _ptr(s), _ptr(vstar), P, B, H, d, _ptr(out), _dtype(out),
                                          _stream(m.device)))
    return out


def triple_floats(d):
    """Floats per packed triple record {v*[d], m, s, pad, pad} (MEA_TRIPLE_FLOATS, mea.h)."""
    return d + 4


def mea_single_query_partial_packed(q, k, v, scale=None, triples=None, workspace=None):
    """Per-(b,h) stream triple over these keys as packed records [B*H, d+4] (v*, m, s; m natural
    log) — the buffer a rank hands to all_gather_into_tensor unchanged."""
    _cuda_contig(q, k, v, triples)
    B, H, d = q.shape
    n_k = k.shape[1]
    if k.shape != (B, n_k, H, d) or v.shape != k.shape:
        raise ValueError(f"shape mismatch q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)}")
    if k.dtype != q.dtype or v.dtype != q.dtype:
        raise TypeError("q, k, v must share a dtype")
    dt = _dtype(q)
    _expect(triples, (B * H, triple_floats(d)), torch.float32, "triples")
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    if triples is None:
        triples = torch.empty((B * H, triple_floats(d)), dtype=torch.float32, device=q.device)
    if workspace is None:
        workspace = _workspace(mea_single_query_workspace_size(B, H, n_k, d, dt), q.device)
    _check(_lib.load().mea_single_query_partial_packed(
        _ptr(q), _ptr(k), _ptr(v), _ptr(triples), B, H, n_k, d, dt, scale, _ptr(workspace),
        workspace.numel() if workspace is not None else 0, _stream(q.device)))
    return triples


def mea_attention_partial_fwd_packed(q, k, v, scale=None, triples=None):
    """Every query row's stream triple over these keys as packed records [B*n_q*H, d+4]
    (row (b, i, h)); bf16, d in {64, 128}."""
    _cuda_contig(q, k, v, triples)
    B, n_q, H, d = q.shape
    n_k = k.shape[1]
    if k.shape != (B, n_k, H, d) or v.shape != k.shape:
        raise ValueError(f"shape mismatch q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)}")
    if k.dtype != q.dtype or v.dtype != q.dtype:
        raise TypeError("q, k, v must share a dtype")
    _expect(triples, (B * n_q * H, triple_floats(d)), torch.float32, "triples")
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    if triples is None:
        triples = torch.empty((B * n_q * H, triple_floats(d)), dtype=torch.float32, device=q.device)
    _check(_lib.load().mea_attention_partial_fwd_packed(_ptr(q), _ptr(k), _ptr(v), _ptr(triples), B, H, n_q, n_k, d,
                                                        _dtype(q), scale, _stream(q.device)))
    return triples


def mea_merge_triples(triples, out_dtype=torch.bfloat16, out=None):
    """Merge stacked packed records triples [P, rows, d+4] -> out [rows, d]."""
    _cuda_contig(triples, out)
    if triples.dim() != 3 or triples.dtype != torch.float32:
        raise ValueError("triples must be float32 [P, rows, d + 4]")
    P, rows, w = triples.shape
    d = w - 4
    _expect_out(out, (rows, d))
    if out is None:
        out = torch.empty((rows, d), dtype=out_dtype, device=triples.device)
    _check(_lib.load().mea_merge_triples(_ptr(triples), P, rows, d, _ptr(out), _dtype(out), _stream(triples.device)))
    return out


# ------------------------------------------------------------------------ backward
def mea_attention_bwd_workspace_size(B, H, n_q, n_k, d, dtype, lse_given=True):
    n = ctypes.c_size_t(0)
    _check(_lib.load().mea_attention_bwd_workspace_size(B, H, n_q, n_k, d, dtype, int(bool(lse_given)),
                                                        ctypes.byref(n)))
    return n.value


def mea_attention_bwd_deterministic_workspace_size(B, H, n_q, n_k, d, dtype, lse_given=True):
    n = ctypes.c_size_t(0)
    _check(_lib.load().mea_attention_bwd_deterministic_workspace_size(B, H, n_q, n_k, d, dtype,
                                                                      int(bool(lse_given)), ctypes.byref(n)))
    return n.value


def _bwd(fn, ws_fn, q, k, v, out, dout, lse, scale, dq, dk, dv, workspace):
    _cuda_contig(q, k, v, out, dout, lse, dq, dk, dv)
    B, n_q, H, d = q.shape
    n_k = k.shape[1]
    dt = _dtype(q)
    # every tensor is read / written as q's dtype and the shapes below (an fp32 `out` from the
    # paper's fp32-output forward must be cast by the caller, it is not reinterpreted)
    for t, shape, nm in ((k, (B, n_k, H, d), "k"), (v, (B, n_k, H, d), "v"), (out, (B, n_q, H, d), "out"),
                         (dout, (B, n_q, H, d), "dout"), (dq, (B, n_q, H, d), "dq"), (dk, (B, n_k, H, d), "dk"),
                         (dv, (B, n_k, H, d), "dv")):
        _expect(t, shape, q.dtype, nm)
    _expect(lse, (B, H, n_q), torch.float32, "lse")
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    if workspace is None:
        workspace = _workspace(ws_fn(B, H, n_q, n_k, d, dt, lse is not None), q.device)
    _check(fn(_ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(dout), _ptr(dq), _ptr(dk), _ptr(dv), B, H, n_q, n_k, d, dt,
              scale, _ptr(lse), _ptr(workspace), workspace.numel() if workspace is not None else 0,
              _stream(q.device)))
    return dq, dk, dv


def mea_attention_bwd(q, k, v, out, dout, lse=None, scale=None, dq=None, dk=None, dv=None, workspace=None):
    """(dq, dk, dv) of out = attention(q, k, v) given dout (recompute-per-tile backward)."""
    return _bwd(_lib.load().mea_attention_bwd, mea_attention_bwd_workspace_size, q, k, v, out, dout, lse, scale,
                dq, dk, dv, workspace)


def mea_attention_bwd_causal(q, k, v, out, dout, lse=None, scale=None, dq=None, dk=None, dv=None, workspace=None):
    """(dq, dk, dv) of out = mea_attention_fwd_causal(q, k, v) given dout."""
    lib = _lib.load()
    fn = lambda q_, k_, v_, o_, do_, dq_, dk_, dv_, B, H, n_q, n_k, d, dt, sc, lse_, ws, nb, st: \
        lib.mea_attention_bwd_causal(q_, k_, v_, o_, do_, dq_, dk_, dv_, B, H, n_q, d, dt, sc, lse_, ws, nb, st)
    if q.shape != k.shape:
        raise ValueError("causal attention needs n_q == n_k")
    return _bwd(fn, mea_attention_bwd_workspace_size, q, k, v, out, dout, lse, scale, dq, dk, dv, workspace)


def _kv_lens_dev(kv_lens, q):
    if not (torch.is_tensor(kv_lens) and kv_lens.dtype == torch.int32 and kv_lens.is_cuda and kv_lens.is_contiguous()):
        raise TypeError("kv_lens must be a contiguous int32 CUDA tensor [B]")
    if kv_lens.shape != (q.shape[0],):
        raise ValueError(f"kv_lens must have shape [B] = [{q.shape[0]}], got {tuple(kv_lens.shape)}")
    return kv_lens


def mea_attention_fwd_padded(q, k, v, kv_lens, scale=None, out=None, out_dtype=None, lse=None, want_lse=False):
    """Attention with key padding: batch element b attends keys j < kv_lens[b] (int32 CUDA [B])."""
    _cuda_contig(q, k, v, out, lse)
    B, n_q, H, d = q.shape
    n_k = k.shape[1]
    if k.shape != (B, n_k, H, d) or v.shape != k.shape:
        raise ValueError(f"shape mismatch q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)}")
    kv_lens = _kv_lens_dev(kv_lens, q)
    if k.dtype != q.dtype or v.dtype != q.dtype:
        raise TypeError("q, k, v must share a dtype")
    _expect_out(out, (B, n_q, H, d))
    _expect(lse, (B, H, n_q), torch.float32, "lse")
    scale = 1.0 / math.sqrt(d) if scale is None else float(scale)
    if out is None:
        out = torch.empty((B, n_q, H, d), dtype=q.dtype if out_dtype is None else out_dtype, device=q.device)
    if want_lse and lse is None:
        lse = torch.empty((B, H, n_q), dtype=torch.float32, device=q.device)
    _check(_lib.load().mea_attention_fwd_padded(_ptr(q), _ptr(k), _ptr(v), _ptr(out), B, H, n_q, n_k, d, _dtype(q),
                                                _dtype(out), scale, _ptr(lse), _ptr(kv_lens), _stream(q.device)))
    return (out, lse) if (want_lse or lse is not None) else out


def mea_attention_bwd_padded(q, k, v, out, dout, kv_lens, lse=None, scale=None, dq=None, dk=None, dv=None,
                             workspace=None):
    """(dq, dk, dv) of out = mea_attention_fwd_padded(q, k, v, kv_lens) given dout."""
    lib = _lib.load()
    kv_lens = _kv_lens_dev(kv_lens, q)
    fn = lambda q_, k_, v_, o_, do_, dq_, dk_, dv_, B, H, n_q, n_k, d, dt, sc, lse_, ws, nb, st: \
        lib.mea_attention_bwd_padded(q_, k_, v_, o_, do_, dq_, dk_, dv_, B, H, n_q, n_k, d, dt, sc, lse_, _ptr(kv_lens),
                                     ws, nb, st)
    return _bwd(fn, mea_attention_bwd_workspace_size, q, k, v, out, dout, lse, scale, dq, dk, dv, workspace)


def mea_attention_bwd_deterministic(q, k, v, out, dout, lse=None, scale=None, dq=None, dk=None, dv=None,
                                    workspace=None):
    """Same as mea_attention_bwd, bitwise reproducible (no cross-CTA reduction), ~2 MiB workspace."""
    return _bwd(_lib.load().mea_attention_bwd_deterministic, mea_attention_bwd_deterministic_workspace_size, q, k,
                v, out, dout, lse, scale, dq, dk, dv, workspace)


# ------------------------------------------------------------------------ generator / debug
def mea_fill_synthetic(t, seed, tensor_id, offset=0):
    """Fill a CUDA tensor with the counter-based synthetic inputs (synth/gen.py), in place."""
    _cuda_contig(t)
    _check(_lib.load().mea_fill_synthetic(_ptr(t), t.numel(), _dtype(t), seed, tensor_id, offset,
                                          _stream(t.device)))
    return t


def mea_debug_umma_tile(a, b, v):
    _cuda_contig(a, b, v)
    s = torch.empty((128, 128), dtype=torch.float32, device=a.device)
    o = torch.empty((128, 64), dtype=torch.float32, device=a.device)
    _check(_lib.load().mea_debug_umma_tile(_ptr(a), _ptr(b), _ptr(v), _ptr(s), _ptr(o), _stream(a.device)))
    return s, o


def debug_set_option(name, value):
    """Experiment knobs of the library (mea_debug.h); defaults are the shipped design."""
    _check(_lib.load().mea_debug_set_option(name.encode(), int(value)))


def debug_read_probe(buf, ctas=0, sink=None):
    """Stream the bytes of a CUDA tensor with the read-only HBM probe (mea_debug.h)."""
    _cuda_contig(buf)
    if sink is None:
        sink = torch.empty(1, dtype=torch.float32, device=buf.device)
    nbytes = buf.numel() * buf.element_size()
    _check(_lib.load().mea_debug_read_probe(_ptr(buf), nbytes - nbytes % 16, ctas, _ptr(sink), _stream(buf.device)))
    return sink


# ------------------------------------------------------------------------ launch profiling
def profile_enable(on=True):
    _lib.load().mea_profile_enable(1 if on else 0)


def profile_read():
    """{kernel name: (launch count, total ms)} since the last read (synchronises)."""
    buf = ctypes.create_string_buffer(1 << 14)
    _check(_lib.load().mea_profile_read(buf, len(buf)))
    res = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split()
        res[name] = (int(cnt), float(ms))
    return res
