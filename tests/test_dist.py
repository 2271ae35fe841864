"""Multi-process (gloo, world size 2, CPU) checks of the sharding and exchange logic.

The GPU kernels are not involved: the per-rank partial and the merge are the oracle's
(O5), so these tests pin the host-side plumbing of paper_2112_05682_b200.dist — disjoint
covering ranges, the shard plan, one all_gather_into_tensor of the packed records
{v*, m, s, pad, pad}, merge — against the unsharded oracle. The same code runs over NCCL with
libmea.so on GPUs (bench.py --gpus N, tests/test_gpu_partial.py).
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2112_05682_b200 import dist as D


def test_shard_range_covers_disjointly():
    for total in (0, 1, 7, 128, 1000):
        for world in (1, 2, 3, 8):
            ranges = [D.shard_range(total, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == total
            for (a, b), (c, d) in zip(ranges[:-1], ranges[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    pairs = [p for r in range(4) for p in D.shard_bh(8, 16, 4, r)]
    assert pairs == [(b, h) for b in range(8) for h in range(16)]


@pytest.mark.parametrize("B,H,n_q", [(8, 16, 1 << 20), (1, 16, 16384), (2, 16, 1000), (1, 4, 5000), (1, 1, 700),
                                     (3, 5, 513), (16, 2, 64)])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shard_plan_assigns_every_unit_once(B, H, n_q, world):
    """Every (b, h, query-row block) unit of self-attention belongs to exactly one rank, and the
    mode is the one the docstring promises (batch > heads > query chunks)."""
    plans = [D.shard_plan(B, H, n_q, world, r) for r in range(world)]
    count = {}
    for p in plans:
        (b0, b1), (h0, h1), (q0, q1) = p["b"], p["h"], p["q"]
        assert 0 <= b0 <= b1 <= B and 0 <= h0 <= h1 <= H and 0 <= q0 <= q1 <= n_q
        for b in range(b0, b1):
            for h in range(h0, h1):
                count.setdefault((b, h), []).append((q0, q1))
    for b in range(B):
        for h in range(H):
            rs = sorted(r for r in count.get((b, h), []) if r[1] > r[0])
            assert rs and rs[0][0] == 0 and rs[-1][1] == n_q, (b, h, rs)
            for (a, c), (e, f) in zip(rs[:-1], rs[1:]):
                assert c == e
    modes = {p["mode"] for p in plans}
    assert len(modes) == 1
    mode = modes.pop()
    if B % world == 0:
        assert mode == "batch"
    elif B * H < world:
        assert mode == "query"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _pack(m, s, vs):
    """Packed records {v*[d], m, s, 0, 0} (mea.h MEA_TRIPLE_FLOATS) from separate arrays."""
    rows, d = vs.shape
    r = torch.zeros(rows, d + 4, dtype=torch.float64)
    r[:, :d] = torch.as_tensor(vs)
    r[:, d] = torch.as_tensor(m)
    r[:, d + 1] = torch.as_tensor(s)
    return r


def _oracle_partial(q, k, v, scale):
    import oracle as O
    B, H, d = q.shape
    ms, ss, vs = [], [], []
    for b in range(B):
        for h in range(H):
            m, s, vv = O.partial_triple(q[b, h][None].numpy(), k[b, :, h].numpy(), v[b, :, h].numpy(), scale)
            ms.append(m[0]); ss.append(s[0]); vs.append(vv[0])
    return _pack(np.array(ms), np.array(ss), np.stack(vs))


def _oracle_merge(recs, out_dtype):
    import oracle as O
    d = recs.shape[-1] - 4
    r = recs.numpy()
    return torch.from_numpy(O.merge(r[..., d], r[..., d + 1], r[..., :d]))


def _init(rank, world, port):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker(rank, world, port, q, k, v, scale, ret):
    _init(rank, world, port)
    lo, hi = D.shard_range(k.shape[1], world, rank)
    out = D.sharded_single_query(q, k[:, lo:hi], v[:, lo:hi], scale=scale, out_dtype=torch.float64,
                                 partial_fn=_oracle_partial, merge_fn=_oracle_merge)
    ret[rank] = out.numpy()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_k", [1, 5, 300])
def test_key_sharded_single_query_gloo_world2(n_k):
    import oracle as O
    B, H, d, world = 2, 3, 8, 2
    g = torch.Generator().manual_seed(n_k)
    q = torch.randn(B, H, d, generator=g, dtype=torch.float64)
    k = torch.randn(B, n_k, H, d, generator=g, dtype=torch.float64)
    v = torch.randn(B, n_k, H, d, generator=g, dtype=torch.float64)
    scale = 1 / math.sqrt(d)
    ret = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), q, k, v, scale, ret), nprocs=world, join=True)
    for b in range(B):
        for h in range(H):
            ref = O.naive(q[b, h][None].numpy(), k[b, :, h].numpy(), v[b, :, h].numpy(), scale)[0][0]
            for r in range(world):    # every rank holds the merged result
                np.testing.assert_allclose(ret[r][b, h], ref, atol=1e-12)


def _oracle_partial_rows(q, k, v, scale):
    """Per query row packed record over these keys (O5), rows ordered (b, i, h) like
    mea_attention_partial_fwd_packed."""
    import oracle as O
    B, n_q, H, d = q.shape
    m = np.empty((B, n_q, H)); s = np.empty((B, n_q, H)); vs = np.empty((B, n_q, H, d))
    for b in range(B):
        for h in range(H):
            mm, ss, vv = O.partial_triple(q[b, :, h].numpy(), k[b, :, h].numpy(), v[b, :, h].numpy(), scale)
            m[b, :, h], s[b, :, h], vs[b, :, h] = mm, ss, vv
    return _pack(m.reshape(-1), s.reshape(-1), vs.reshape(-1, d))


def _worker_sa(rank, world, port, q, k, v, scale, ret):
    _init(rank, world, port)
    lo, hi = D.shard_range(k.shape[1], world, rank)
    out = D.sharded_self_attention(q, k[:, lo:hi], v[:, lo:hi], scale=scale, out_dtype=torch.float64,
                                   partial_fn=_oracle_partial_rows, merge_fn=_oracle_merge)
    ret[rank] = out.numpy()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_k", [1, 9, 200])
def test_key_sharded_self_attention_gloo_world2(n_k):
    """Long-context self-attention by key range: per-rank row records, one
    all-gather, merge == the unsharded definition (n_k = 1 leaves rank 1 with no keys)."""
    import oracle as O
    B, n_q, H, d, world = 2, 7, 3, 8, 2
    g = torch.Generator().manual_seed(100 + n_k)
    q = torch.randn(B, n_q, H, d, generator=g, dtype=torch.float64)
    k = torch.randn(B, n_k, H, d, generator=g, dtype=torch.float64)
    v = torch.randn(B, n_k, H, d, generator=g, dtype=torch.float64)
    scale = 1 / math.sqrt(d)
    ret = mp.Manager().dict()
    mp.spawn(_worker_sa, args=(world, _free_port(), q, k, v, scale, ret), nprocs=world, join=True)
    ref, _ = O.mha_forward(q.numpy(), k.numpy(), v.numpy(), scale)
    for r in range(world):
        np.testing.assert_allclose(ret[r], ref, atol=1e-12)


def _worker_qc(rank, world, port, q, k, v, scale, ret):
    """Query-chunk sharding (B*H < world): this rank computes its query rows only (oracle O1 as
    the per-rank compute), no collective; the result is gathered here only to check it."""
    import oracle as O
    _init(rank, world, port)
    B, n_q, H, d = q.shape
    plan = D.shard_plan(B, H, n_q, world, rank, row_block=4)
    assert plan["mode"] == "query"
    q0, q1 = plan["q"]
    out_local, _ = O.mha_forward(q[:, q0:q1].numpy(), k.numpy(), v.numpy(), scale)
    ret[rank] = (q0, q1, out_local)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_q", [3, 17])
def test_query_chunk_sharding_gloo_world2(n_q):
    """Self-attention with B*H = 1 < world: query rows split in row blocks across the ranks
    (PAPER.md:68-70 rows are independent; Figure 1's query chunks), K/V replicated, no
    data-path collective; the concatenated rank outputs equal the unsharded definition."""
    import oracle as O
    B, n_k, H, d, world = 1, 11, 1, 8, 2
    g = torch.Generator().manual_seed(300 + n_q)
    q = torch.randn(B, n_q, H, d, generator=g, dtype=torch.float64)
    k = torch.randn(B, n_k, H, d, generator=g, dtype=torch.float64)
    v = torch.randn(B, n_k, H, d, generator=g, dtype=torch.float64)
    scale = 1 / math.sqrt(d)
    ret = mp.Manager().dict()
    mp.spawn(_worker_qc, args=(world, _free_port(), q, k, v, scale, ret), nprocs=world, join=True)
    ref, _ = O.mha_forward(q.numpy(), k.numpy(), v.numpy(), scale)
    got = np.zeros_like(ref)
    covered = np.zeros(n_q, dtype=int)
    for r in range(world):
        q0, q1, o = ret[r]
        got[:, q0:q1] = o
        covered[q0:q1] += 1
    assert (covered == 1).all()
    np.testing.assert_allclose(got, ref, atol=1e-12)


def _worker_ag(rank, world, port, ret):
    _init(rank, world, port)
    local = torch.full((3, 12), float(rank)) + torch.arange(12.0)
    g = D.allgather_records(local)
    ret[rank] = g.numpy()
    dist.destroy_process_group()


def test_allgather_records_rank_order_gloo_world2():
    """The packed exchange is one all_gather_into_tensor in rank order: [P, rows, d + 4]."""
    ret = mp.Manager().dict()
    mp.spawn(_worker_ag, args=(2, _free_port(), ret), nprocs=2, join=True)
    for r in range(2):
        g = ret[r]
        assert g.shape == (2, 3, 12)
        for p in range(2):
            np.testing.assert_array_equal(g[p], np.full((3, 12), float(p)) + np.arange(12.0))
