"""Float64 oracle: the attention definition and the paper's algorithms, written out.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Plain numpy, float64 unless a
function says otherwise. "P:n" = /root/reference/PAPER.md line n. Figure 1's
minted line m is P:(107+m).

Notation follows the paper: q (query), k_i / v_i (keys / values), s_i = dot(q, k_i)
(scores), v* / s* / m* (running value sum, weight sum and max). ``scale`` multiplies
every score: the paper's Secs. 1-3 use scale = 1; Figure 1 divides the
query by sqrt(d), i.e. scale = 1/sqrt(d). Callers pass it explicitly.

Single-head functions take q [n_q, d], k [n_k, d], v [n_k, d_v] arrays. The
multi-head wrappers take [B, n, H, d] arrays (the library's layout) and loop over
(b, h).

Pins: every function here is checked in tests/test_oracle.py against closed forms,
special cases, invariants, brute force and finite differences ("Oracle
pins"). None is "parity unpinned".
"""
import math

import numpy as np


class EmptyKeysError(ValueError):
    """Attention over an empty key list is undefined (no weights to normalise)."""


def _f64(x):
    return np.asarray(x, dtype=np.float64)


def _check(q, k, v):
    q, k, v = _f64(q), _f64(k), _f64(v)
    if k.shape[0] == 0:
        raise EmptyKeysError("attention over an empty key list")
    if k.shape[0] != v.shape[0] or q.shape[-1] != k.shape[-1]:
        raise ValueError("shape mismatch")
    return q, k, v


# ----------------------------------------------------------------------------------
# O1: the definition, with the max subtracted before exponentiating
#     ("In practice, the softmax is implemented by subtracting the maximum score",
#     P:78-79). Also returns lse_i = log sum_j e^{s_ij} (natural log).
# ----------------------------------------------------------------------------------
def scores(q, k, scale):
    """s_ij = scale * dot(q_i, k_j)   (scale from P:116)."""
    return scale * (_f64(q) @ _f64(k).T)


def causal_mask(s, rows):
    """Causal attention (not in the paper, which disabled packing to avoid masking, P:353;
    reimplementations added it): query i sees keys j <= i only (n_q == n_k, top-left
    alignment). Masked scores are -inf, so their weights e^{s - m} are exactly 0."""
    j = np.arange(s.shape[1])[None, :]
    return np.where(j <= np.asarray(rows)[:, None], s, -math.inf)


def naive(q, k, v, scale, rows=None, causal=False):
    """Standard attention. Returns (out [n_q, d_v], lse [n_q]).

    ``rows`` restricts the evaluation to those query rows (each output row depends
    only on its own query), for sampling large configurations.
    ``causal``: query i attends keys j <= i only (see ``causal_mask``).
    """
    q, k, v = _check(q, k, v)
    row_ids = np.arange(q.shape[0]) if rows is None else np.asarray(rows)
    if causal and q.shape[0] != k.shape[0]:
        raise ValueError("causal attention needs n_q == n_k")
    if rows is not None:
        q = q[row_ids]
    s = scores(q, k, scale)                      # s_i = dot(q, k_i)
    if causal:
        s = causal_mask(s, row_ids)
    m = s.max(axis=1, keepdims=True)             # maximum score per query
    p = np.exp(s - m)                            # e^{s_i - m}
    l = p.sum(axis=1, keepdims=True)             # sum_j e^{s_j - m}
    out = (p @ v) / l                            # sum_i v_i s'_i
    lse = (m + np.log(l))[:, 0]
    return out, lse


# ----------------------------------------------------------------------------------
# O2: Eq. (1) lazy softmax WITHOUT max subtraction. Numerically unstable
#     by design: the negative control. dtype selects the arithmetic.
# ----------------------------------------------------------------------------------
def lazy_unstable(q, k, v, scale, dtype=np.float64):
    q, k, v = (np.asarray(x, dtype=dtype) for x in _check(q, k, v))
    s = dtype(scale) * (q @ k.T)                 # s_i = dot(q, k_i)
    with np.errstate(over="ignore", invalid="ignore", divide="ignore"):
        e = np.exp(s)                            # s'_i = e^{s_i}
        return (e @ v) / e.sum(axis=1, keepdims=True)   # sum_i v_i s'_i / sum_j s'_j


# ----------------------------------------------------------------------------------
# O3: the paper's sequential algorithm with the running max, built on
#     the stream state (v*, s*, m*) initialised to (0, 0, -inf).
# ----------------------------------------------------------------------------------
def stream_init(d):
    """v* = 0 in R^d, s* = 0, m* = -inf."""
    return np.zeros(d, dtype=np.float64), 0.0, -math.inf


def stream_update(state, s_i, v_i):
    """One key/value pair:
    m_i = max(m*, s_i);  v* <- v* e^{m*-m_i} + v_i e^{s_i-m_i};
    s* <- s* e^{m*-m_i} + e^{s_i-m_i};  m* <- m_i.
    At m* = -inf (no update yet) e^{m*-m_i} is taken as 0 (reading 3).
    """
    v_star, s_star, m_star = state
    m_i = max(m_star, s_i)
    a = 0.0 if m_star == -math.inf else math.exp(m_star - m_i)
    b = math.exp(s_i - m_i)
    return v_star * a + _f64(v_i) * b, s_star * a + b, m_i


def stream_finalize(state):
    """v* / s*  (P:90). An empty stream is an error, not NaN (reading 3)."""
    v_star, s_star, m_star = state
    if m_star == -math.inf:
        raise EmptyKeysError("empty attention stream")
    return v_star / s_star


def single_query(q_row, k, v, scale):
    """Single-query attention by the stream (P:59-63 with P:85-90): keys in order."""
    q_row, k, v = _f64(q_row), _f64(k), _f64(v)
    if k.shape[0] == 0:
        raise EmptyKeysError("attention over an empty key list")
    st = stream_init(v.shape[1])
    for i in range(k.shape[0]):
        st = stream_update(st, scale * float(np.dot(q_row, k[i])), v[i])
    return st


def sequential(q, k, v, scale):
    """Self-attention by running the stream for every query.

    The stream of each query row is independent; for speed the key loop is shared
    by all rows (the per-row arithmetic is exactly stream_update's). Returns
    (out, (v*, s*, m*)) with v* [n_q, d_v], s* [n_q], m* [n_q].
    """
    q, k, v = _check(q, k, v)
    n_q = q.shape[0]
    v_star = np.zeros((n_q, v.shape[1]))
    s_star = np.zeros(n_q)
    m_star = np.full(n_q, -math.inf)
    for i in range(k.shape[0]):
        s_i = scale * (q @ k[i])                           # s_i = dot(q, k_i)
        m_i = np.maximum(m_star, s_i)                      # m_i = max(m*, s_i)
        a = np.where(m_star == -math.inf, 0.0, np.exp(m_star - m_i))
        b = np.exp(s_i - m_i)
        v_star = v_star * a[:, None] + v[i][None, :] * b[:, None]
        s_star = s_star * a + b
        m_star = m_i
    return v_star / s_star[:, None], (v_star, s_star, m_star)


# ----------------------------------------------------------------------------------
# O4: Figure 1 literally, except that ragged last chunks cover exactly
#     the remaining keys/queries (reading 2) instead of dynamic_slice's
#     clamped start.
# ----------------------------------------------------------------------------------
def summarize_chunk(query, key, value):
    """Figure 1 lines 12-19; ``query`` is already scaled (line 9)."""
    attn_weights = query @ key.T                                  # einsum qhd,khd->qhk
    max_score = attn_weights.max(axis=-1, keepdims=True)          # stop_gradient'ed max
    exp_weights = np.exp(attn_weights - max_score)
    exp_values = exp_weights @ value                              # einsum vhf,qhv->qhf
    return exp_values, exp_weights.sum(axis=-1), max_score[:, 0]


def query_chunk_attention(query, key, value, scale, key_chunk_size=4096):
    """Figure 1 lines 4-40 for one query chunk."""
    num_kv = key.shape[0]
    key_chunk_size = min(key_chunk_size, num_kv)                  # line 8
    query = query * scale                                         # line 9 (scale = 1/sqrt(d))
    chunks = [summarize_chunk(query, key[c:c + key_chunk_size], value[c:c + key_chunk_size])
              for c in range(0, num_kv, key_chunk_size)]          # lines 30-31 (lax.map)
    chunk_values = np.stack([c[0] for c in chunks])
    chunk_weights = np.stack([c[1] for c in chunks])
    chunk_max = np.stack([c[2] for c in chunks])
    global_max = chunk_max.max(axis=0, keepdims=True)             # line 33
    max_diffs = np.exp(chunk_max - global_max)                    # line 34
    chunk_values = chunk_values * max_diffs[..., None]            # line 35
    chunk_weights = chunk_weights * max_diffs                     # line 36
    all_values = chunk_values.sum(axis=0)                         # line 38
    all_weights = chunk_weights.sum(axis=0)[:, None]              # line 39
    return all_values / all_weights                               # line 40


def chunked(q, k, v, scale, query_chunk_size=1024, key_chunk_size=4096):
    """Figure 1 lines 42-56: scan over query chunks, write each result."""
    q, k, v = _check(q, k, v)
    res = np.empty((q.shape[0], v.shape[1]))
    for c in range(0, q.shape[0], query_chunk_size):
        res[c:c + query_chunk_size] = query_chunk_attention(
            q[c:c + query_chunk_size], k, v, scale, key_chunk_size)
    return res


# ----------------------------------------------------------------------------------
# O5: merge of P partial triples (m*, s*, v*) over disjoint key ranges — Figure 1's
#     global-max rescale (lines 33-40) applied to stream states.
#     m is in natural-log units of the scaled score. An empty range has
#     (m, s, v) = (-inf, 0, 0) and contributes nothing.
# ----------------------------------------------------------------------------------
def merge(m, s, vstar):
    m, s, vstar = _f64(m), _f64(s), _f64(vstar)     # [P, ...], [P, ...], [P, ..., d]
    global_max = m.max(axis=0, keepdims=True)
    if np.any(global_max == -math.inf):
        raise EmptyKeysError("all partials empty")
    max_diffs = np.where(m == -math.inf, 0.0, np.exp(m - global_max))
    all_values = (vstar * max_diffs[..., None]).sum(axis=0)
    all_weights = (s * max_diffs).sum(axis=0)
    return all_values / all_weights[..., None]


def partial_triple(q, k, v, scale):
    """(m*, s*, v*) of the stable stream for each query row over these keys,
    in closed form: m* = max_j s_j, s* = sum_j e^{s_j-m*}, v* = sum_j v_j e^{s_j-m*}.
    Empty key range -> (-inf, 0, 0)."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    if k.shape[0] == 0:
        n = q.shape[0]
        return np.full(n, -math.inf), np.zeros(n), np.zeros((n, v.shape[1]))
    s = scores(q, k, scale)
    m = s.max(axis=1)
    p = np.exp(s - m[:, None])
    return m, p.sum(axis=1), p @ v


# ----------------------------------------------------------------------------------
# O5t: multi-stage summarisation ("A multi-stage summarization approach could
#      achieve O(log n)"). The key chunks of a query chunk are summarised one
#      after another (partial_triple = Figure 1 lines 12-19's summary) and
#      combined like a binary counter: level l holds the summary of 2^l consecutive
#      chunks; a new summary carries upward while its level is occupied, merging two
#      summaries with Figure 1's rescale (lines 33-36, via merge2). The
#      occupied levels are merged at the end and v*/s* returned (line 40).
#      Returns (out, lse, max_alive): max_alive = most summaries alive at once.
#      Reading (reading 18): the paper gives no algorithm for this stage, only
#      the remark; the binary counter is the plainest schedule with O(log n) summaries.
# ----------------------------------------------------------------------------------
def merge2(a, b):
    """Two summaries (m, s, v*) of the same rows over disjoint key ranges -> one."""
    (ma, sa, va), (mb, sb, vb) = a, b
    m = np.maximum(ma, mb)
    wa = np.where(ma == -math.inf, 0.0, np.exp(ma - m))
    wb = np.where(mb == -math.inf, 0.0, np.exp(mb - m))
    return m, sa * wa + sb * wb, va * wa[:, None] + vb * wb[:, None]


def tree_summarize(q, k, v, scale, key_chunk_size):
    q, k, v = _check(q, k, v)
    levels = []            # levels[l] = summary of 2^l chunks, or None
    max_alive = 0
    for c in range(0, k.shape[0], key_chunk_size):
        cur = partial_triple(q, k[c:c + key_chunk_size], v[c:c + key_chunk_size], scale)
        max_alive = max(max_alive, 1 + sum(x is not None for x in levels))
        lvl = 0
        while lvl < len(levels) and levels[lvl] is not None:
            cur = merge2(levels[lvl], cur)
            levels[lvl] = None
            lvl += 1
        if lvl == len(levels):
            levels.append(None)
        levels[lvl] = cur
    acc = None
    for x in levels:
        if x is not None:
            acc = x if acc is None else merge2(x, acc)
    m, s_, vstar = acc
    return vstar / s_[:, None], m + np.log(s_), max_alive


# ----------------------------------------------------------------------------------
# O6: analytic backward of out = softmax(scale q k^T) v. The paper delegates the
#     derivative to jax.grad with checkpointing; the formulas are the
#     standard softmax calculus. The max carries no gradient
#     (stop_gradient): the result does not depend on it.
# ----------------------------------------------------------------------------------
def backward(q, k, v, dout, scale, causal=False):
    q, k, v = _check(q, k, v)
    dout = _f64(dout)
    s = scores(q, k, scale)
    if causal:
        s = causal_mask(s, np.arange(q.shape[0]))      # masked entries: P = 0, so dS = 0
    p = np.exp(s - s.max(axis=1, keepdims=True))
    p /= p.sum(axis=1, keepdims=True)                 # P = softmax(scale q k^T)
    dv = p.T @ dout                                   # dV = P^T dO
    dp = dout @ v.T                                   # dP = dO V^T
    delta = (p * dp).sum(axis=1, keepdims=True)       # delta_i = sum_j P_ij dP_ij
    ds = p * (dp - delta)                             # dS = P o (dP - delta)
    dq = scale * (ds @ k)                             # dQ = scale dS K
    dk = scale * (ds.T @ q)                           # dK = scale dS^T Q
    return dq, dk, dv


def backward_rows(q, k, v, dout, scale, q_rows, k_rows, block=2048, causal=False):
    """O6 restricted to some outputs, for checking large configurations: dq for the query
    rows ``q_rows`` and dk, dv for the key rows ``k_rows``, each exactly as in ``backward``
    (same formulas; the full softmax statistics lse_i and delta_i = dO_i . O_i of every query
    row are computed block by block of query rows, since each row's are independent)."""
    q, k, v = _check(q, k, v)
    dout = _f64(dout)
    n_q = q.shape[0]
    lse = np.empty(n_q)
    delta = np.empty(n_q)
    for a in range(0, n_q, block):
        o, l = naive(q, k, v, scale, rows=np.arange(a, min(a + block, n_q)), causal=causal)
        lse[a:a + block] = l
        delta[a:a + block] = delta_rowsum(o, dout[a:a + block])
    qr = np.asarray(q_rows)
    s = scores(q[qr], k, scale)
    if causal:
        s = causal_mask(s, qr)
    p = np.exp(s - lse[qr, None])                                # P rows of the sampled queries
    ds = p * (dout[qr] @ v.T - delta[qr, None])
    dq = scale * (ds @ k)
    kr = np.asarray(k_rows)
    sc = scores(q, k[kr], scale)
    if causal:                                                   # key kr[c] is seen by queries >= kr[c]
        sc = np.where(np.arange(n_q)[:, None] >= kr[None, :], sc, -math.inf)
    pc = np.exp(sc - lse[:, None])                               # P columns of the sampled keys
    dv = pc.T @ dout
    dsc = pc * (dout @ v[kr].T - delta[:, None])
    dk = scale * (dsc.T @ q)
    return dq, dk, dv


def delta_rowsum(out, dout):
    """delta_i = dot(dO_i, O_i) (equals sum_j P_ij dP_ij)."""
    return (_f64(out) * _f64(dout)).sum(axis=1)


# ----------------------------------------------------------------------------------
# O7: central finite differences of L = sum(dO o attention(q, k, v)), step h.
# ----------------------------------------------------------------------------------
def fd_grad(q, k, v, dout, scale, h=1e-6, causal=False):
    q, k, v = (np.array(x, dtype=np.float64) for x in _check(q, k, v))
    dout = _f64(dout)

    def loss():
        return float((naive(q, k, v, scale, causal=causal)[0] * dout).sum())

    grads = []
    for x in (q, k, v):
        g = np.zeros_like(x)
        for idx in np.ndindex(*x.shape):
            old = x[idx]
            x[idx] = old + h
            lp = loss()
            x[idx] = old - h
            lm = loss()
            x[idx] = old
            g[idx] = (lp - lm) / (2 * h)
        grads.append(g)
    return tuple(grads)


# ----------------------------------------------------------------------------------
# Multi-head wrappers over the library layout [B, n, H, d].
# ----------------------------------------------------------------------------------
def mha_forward(q, k, v, scale, rows=None, heads=None, causal=False):
    """O1 per (b, h). Returns out [B, n_q(or len(rows)), H, d_v] and lse [B, H, n_q]."""
    B, n_q, H, _ = q.shape
    nr = n_q if rows is None else len(rows)
    out = np.zeros((B, nr, H, v.shape[3]))
    lse = np.zeros((B, H, nr))
    for b in range(B):
        for h in (range(H) if heads is None else heads):
            o, l = naive(q[b, :, h], k[b, :, h], v[b, :, h], scale, rows=rows, causal=causal)
            out[b, :, h] = o
            lse[b, h] = l
    return out, lse


def mha_backward(q, k, v, dout, scale, causal=False):
    dq, dk, dv = (np.zeros(x.shape) for x in (q, k, v))
    for b in range(q.shape[0]):
        for h in range(q.shape[2]):
            dq[b, :, h], dk[b, :, h], dv[b, :, h] = backward(
                q[b, :, h], k[b, :, h], v[b, :, h], dout[b, :, h], scale, causal=causal)
    return dq, dk, dv
