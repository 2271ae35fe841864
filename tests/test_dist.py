"""Multi-process (gloo, world size 2, CPU) checks of the sharding and exchange logic.

The GPU kernels are not involved: the per-rank partial and the merge are the oracle's
(O5), so these tests pin the host-side plumbing of paper_2112_05682_b200.dist — disjoint
covering ranges, one all-gather of the packed triples, merge — against the unsharded
oracle. The same code runs over NCCL with libmea.so on GPUs (bench.py, test_gpu_*).
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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_partial(q, k, v, scale):
    import oracle as O
    B, H, d = q.shape
    ms, ss, vs = [], [], []
    for b in range(B):
        for h in range(H):
            m, s, vv = O.partial_triple(q[b, h][None].numpy(), k[b, :, h].numpy(), v[b, :, h].numpy(), scale)
            ms.append(m[0]); ss.append(s[0]); vs.append(vv[0])
    return torch.tensor(ms), torch.tensor(ss), torch.tensor(np.stack(vs))


def _oracle_merge(m, s, v, B, H, out_dtype):
    import oracle as O
    return torch.from_numpy(O.merge(m.numpy(), s.numpy(), v.numpy())).reshape(B, H, -1)


def _worker(rank, world, port, q, k, v, scale, ret):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
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
    """Per query row triple over these keys (O5), laid out like mea_attention_partial_fwd."""
    import oracle as O
    B, n_q, H, d = q.shape
    m = np.empty((B, n_q, H)); s = np.empty((B, n_q, H)); vs = np.empty((B, n_q, H, d))
    for b in range(B):
        for h in range(H):
            mm, ss, vv = O.partial_triple(q[b, :, h].numpy(), k[b, :, h].numpy(), v[b, :, h].numpy(), scale)
            m[b, :, h], s[b, :, h], vs[b, :, h] = mm, ss, vv
    return torch.from_numpy(m), torch.from_numpy(s), torch.from_numpy(vs)


def _oracle_merge_rows(m, s, v, B, R, out_dtype):
    import oracle as O
    return torch.from_numpy(O.merge(m.numpy(), s.numpy(), v.numpy())).reshape(B, R, -1)


def _worker_sa(rank, world, port, q, k, v, scale, ret):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = D.shard_range(k.shape[1], world, rank)
    out = D.sharded_self_attention(q, k[:, lo:hi], v[:, lo:hi], scale=scale, out_dtype=torch.float64,
                                   partial_fn=_oracle_partial_rows, merge_fn=_oracle_merge_rows)
    ret[rank] = out.numpy()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_k", [1, 9, 200])
def test_key_sharded_self_attention_gloo_world2(n_k):
    """Long-context self-attention by key range: per-rank row triples, one
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
