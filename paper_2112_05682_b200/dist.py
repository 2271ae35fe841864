"""Multi-GPU plumbing (one process per GPU, torch.distributed over NCCL).

How the hot path shards:

* Self-attention: query rows are independent, so the work units (b, h, query
  row) are split across ranks with NO collective on the data path. ``shard_plan`` picks the
  split: whole batch elements when B divides evenly, else contiguous head blocks of the
  flattened (b, h) pairs, else (B*H < world, or no even split) query-row chunks of every
  (b, h) — the paper's query chunks spread over GPUs, K/V replicated.
* Very long single-query attention: the keys are split into ranges (MNNFast-style KV
  sharding). Each rank computes the stream triple (m*, s*, v*) of its range with
  ``mea_single_query_partial_packed``, which writes packed records {v*, m, s, pad, pad} straight
  into the buffer ONE ``all_gather_into_tensor`` sends; every rank then merges the P records per
  (b, h) with Figure 1's global-max rescale in ``mea_merge_triples``.
* Long-context self-attention beyond one GPU: the same with one record per
  query row (``mea_attention_partial_fwd_packed``, ``sharded_self_attention``).

The compute steps default to libmea.so; the exchange logic is covered on CPU (gloo, world
size 2) in tests/test_dist.py by passing the oracle's partial/merge instead.
"""
import torch
import torch.distributed as dist


def shard_range(total, world, rank):
    """[lo, hi) of an even split of `total` units over `world` ranks (first ranks get the
    remainder). Ranges are disjoint, ordered, and cover [0, total)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def shard_bh(B, H, world, rank):
    """The (b, h) pairs this rank owns for self-attention sharding (no collective)."""
    lo, hi = shard_range(B * H, world, rank)
    return [(i // H, i % H) for i in range(lo, hi)]


def shard_plan(B, H, n_q, world, rank, row_block=256):
    """This rank's share of a self-attention problem [B, n_q, H] (no collective):
    {"mode": "batch" | "heads" | "query", "b": (lo, hi), "h": (lo, hi), "q": (lo, hi)}.

    batch  - B % world == 0: whole batch elements (contiguous [B/world, n, H, d] slices).
    heads  - (B * H) % world == 0 and each rank's block stays inside one batch element: a
             contiguous range of heads of one b (the rank holds its [1, n, H/..., d] tensors).
    query  - otherwise (B * H < world, or no even split): every (b, h), a contiguous range of
             query rows in multiples of `row_block` (the kernel's CTA rows); K/V replicated.
    Every (b, h, query row) unit belongs to exactly one rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if B % world == 0:
        lo, hi = shard_range(B, world, rank)
        return {"mode": "batch", "b": (lo, hi), "h": (0, H), "q": (0, n_q)}
    if (B * H) % world == 0 and H % ((B * H) // world) == 0:
        per = (B * H) // world
        lo = rank * per
        b = lo // H
        return {"mode": "heads", "b": (b, b + 1), "h": (lo % H, lo % H + per), "q": (0, n_q)}
    blocks = -(-n_q // row_block)
    lo, hi = shard_range(blocks, world, rank)
    return {"mode": "query", "b": (0, B), "h": (0, H), "q": (min(n_q, lo * row_block), min(n_q, hi * row_block))}


def _world(group):
    return dist.get_world_size(group) if dist.is_initialized() else 1


def allgather_records(local, group=None):
    """One collective: every rank's packed records [rows, d + 4] -> [P, rows, d + 4] (rank order),
    NCCL all_gather_into_tensor into one preallocated buffer (no per-rank list, no cat/stack)."""
    world = _world(group)
    if world == 1:
        return local.unsqueeze(0)
    rows = local.shape[0]
    out = torch.empty((world * rows,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local.contiguous(), group=group)   # rank r's rows at [r*rows, (r+1)*rows)
    return out.view((world, rows) + tuple(local.shape[1:]))


def sharded_single_query(q, k_local, v_local, scale=None, out_dtype=torch.bfloat16, group=None,
                         partial_fn=None, merge_fn=None, workspace=None):
    """Single-query attention with the keys sharded over the ranks of `group`.

    q [B, H, d] (replicated); k_local, v_local [B, n_k_local, H, d] (this rank's key range,
    may be empty). Returns out [B, H, d] on every rank.
    partial_fn(q, k, v, scale) -> records [B*H, d+4]; merge_fn(records [P, B*H, d+4], out_dtype)
    -> [B*H, d] (defaults: libmea.so)."""
    if partial_fn is None or merge_fn is None:
        from . import api
        partial_fn = partial_fn or (lambda q_, k_, v_, sc: api.mea_single_query_partial_packed(
            q_, k_, v_, scale=sc, workspace=workspace))
        merge_fn = merge_fn or (lambda r_, od: api.mea_merge_triples(r_, out_dtype=od))
    B, H, d = q.shape
    recs = allgather_records(partial_fn(q, k_local, v_local, scale), group)
    return merge_fn(recs, out_dtype).reshape(B, H, d)


def sharded_self_attention(q, k_local, v_local, scale=None, out_dtype=torch.bfloat16, group=None,
                           partial_fn=None, merge_fn=None):
    """Self-attention with the keys sharded over the ranks of `group`.

    q [B, n_q, H, d] (replicated); k_local, v_local [B, n_k_local, H, d] (this rank's key range,
    may be empty). Every query row's triple over the local keys is written as a
    packed record, exchanged in one all-gather of B*n_q*H*(d+4) floats per rank and merged with
    the global-max rescale. Returns out [B, n_q, H, d] on every rank."""
    if partial_fn is None or merge_fn is None:
        from . import api
        partial_fn = partial_fn or (lambda q_, k_, v_, sc: api.mea_attention_partial_fwd_packed(q_, k_, v_, scale=sc))
        merge_fn = merge_fn or (lambda r_, od: api.mea_merge_triples(r_, out_dtype=od))
    B, n_q, H, d = q.shape
    recs = allgather_records(partial_fn(q, k_local, v_local, scale), group)
    return merge_fn(recs, out_dtype).reshape(B, n_q, H, d)
