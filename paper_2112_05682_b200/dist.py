"""Multi-GPU plumbing (one process per GPU, torch.distributed over NCCL).

Two ways the hot path shards:

* Self-attention: query rows are independent, so (b, h) pairs — or query
  blocks — are split across ranks with NO collective on the data path
  (``shard_range`` / ``shard_bh``).
* Very long single-query attention: the keys are split into ranges (MNNFast-style KV
  sharding). Each rank computes the stream triple (m*, s*, v*) of its range
  with ``mea_single_query_partial``; ONE all-gather exchanges the (d + 2) floats per (b, h)
  and every rank merges them with Figure 1's global-max rescale in
  ``mea_merge_partials``.

* Long-context self-attention beyond one GPU: the keys are split into
  ranges; each rank computes the triple of every query row over its range with
  ``mea_attention_partial_fwd``, one all-gather exchanges them and every rank merges
  (``sharded_self_attention``).

The compute steps default to libmea.so; the exchange logic is covered on CPU (gloo,
world size 2) in tests/test_dist.py by passing the oracle's partial/merge instead.
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


def _world(group):
    return dist.get_world_size(group) if dist.is_initialized() else 1


def gather_triples(m, s, vstar, group=None):
    """All-gather per-rank triples m [BH], s [BH], vstar [BH, d] -> stacked [P, BH], [P, BH],
    [P, BH, d]. One collective: the triple is packed as [BH, d + 2]."""
    BH, d = vstar.shape
    packed = torch.cat([m.reshape(BH, 1), s.reshape(BH, 1), vstar.reshape(BH, d)], dim=1).contiguous()
    world = _world(group)
    if world == 1:
        g = packed.unsqueeze(0)
    else:
        parts = [torch.empty_like(packed) for _ in range(world)]
        dist.all_gather(parts, packed, group=group)
        g = torch.stack(parts)
    return g[..., 0].contiguous(), g[..., 1].contiguous(), g[..., 2:].contiguous()


def sharded_single_query(q, k_local, v_local, scale=None, out_dtype=torch.bfloat16, group=None,
                         partial_fn=None, merge_fn=None):
    """Single-query attention with the keys sharded over the ranks of `group`.

    q [B, H, d] (replicated); k_local, v_local [B, n_k_local, H, d] (this rank's key range,
    may be empty). Returns out [B, H, d] on every rank.
    """
    if partial_fn is None or merge_fn is None:
        from . import api
        partial_fn = partial_fn or (lambda q_, k_, v_, sc: api.mea_single_query_partial(q_, k_, v_, scale=sc))
        merge_fn = merge_fn or (lambda m_, s_, v_, B_, H_, od: api.mea_merge_partials(m_, s_, v_, B_, H_, od))
    B, H, _ = q.shape
    m, s, vs = partial_fn(q, k_local, v_local, scale)
    M, S, V = gather_triples(m, s, vs, group)
    return merge_fn(M, S, V, B, H, out_dtype)


def sharded_self_attention(q, k_local, v_local, scale=None, out_dtype=torch.bfloat16, group=None,
                           partial_fn=None, merge_fn=None):
    """Self-attention with the keys sharded over the ranks of `group`.

    q [B, n_q, H, d] (replicated); k_local, v_local [B, n_k_local, H, d] (this rank's key range,
    may be empty). Every query row's triple over the local keys is exchanged in
    one all-gather of B*n_q*H*(d+2) floats per rank and merged with the global-max rescale
    (PAPER.md:140-147). Returns out [B, n_q, H, d] on every rank.
    """
    if partial_fn is None or merge_fn is None:
        from . import api
        partial_fn = partial_fn or (lambda q_, k_, v_, sc: api.mea_attention_partial_fwd(q_, k_, v_, scale=sc))
        merge_fn = merge_fn or (lambda m_, s_, v_, B_, R_, od: api.mea_merge_partials(m_, s_, v_, B_, R_, od))
    B, n_q, H, d = q.shape
    m, s, vs = partial_fn(q, k_local, v_local, scale)
    M, S, V = gather_triples(m.reshape(-1), s.reshape(-1), vs.reshape(-1, d), group)
    return merge_fn(M, S, V, B, n_q * H, out_dtype).reshape(B, n_q, H, d)
