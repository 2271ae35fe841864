"""The library has no hidden per-call global state: calls on several CUDA streams at once, and
from several host threads at once, each with its own workspace, give the same results as the
same calls run one after another (bit for bit for the forward paths and the single query,
whose reductions have a fixed order; the fused backward's dq to its cross-CTA reduction order)."""
import math
import threading

import pytest
import torch

from paper_2112_05682_b200 import api

pytestmark = pytest.mark.gpu


def _inputs(seed, n=1000, H=4, d=64):
    q = torch.empty((1, n, H, d), dtype=torch.bfloat16, device="cuda")
    k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
    for t, tid in ((q, 1), (k, 2), (v, 3), (do, 4)):
        api.mea_fill_synthetic(t, seed, tid)
    return q, k, v, do


def _work(q, k, v, do):
    """Every workspace-using entry point once: online forward, key-split forward (arrival
    counters in the workspace), single query (tickets in the workspace), fused backward."""
    out, lse = api.mea_attention_fwd(q, k, v, want_lse=True)
    out_kc = api.mea_attention_fwd(q, k, v, q_chunk=256, k_chunk=256)
    sq = api.mea_single_query_fwd(q[:, 0].contiguous(), k, v, out_dtype=torch.float32)
    dq, dk, dv = api.mea_attention_bwd(q, k, v, out, do, lse=lse)
    return out, lse, out_kc, sq, dq, dk, dv


def _check(ref, got):
    out, lse, out_kc, sq, dq, dk, dv = got
    r_out, r_lse, r_kc, r_sq, r_dq, r_dk, r_dv = ref
    assert torch.equal(out, r_out) and torch.equal(lse, r_lse) and torch.equal(out_kc, r_kc)
    assert torch.equal(sq, r_sq)
    for a, b in ((dq, r_dq), (dk, r_dk), (dv, r_dv)):
        torch.testing.assert_close(a.float(), b.float(), rtol=0, atol=2e-2)


def test_concurrent_streams_match_sequential():
    sets = [_inputs(seed) for seed in range(4)]
    refs = [_work(*s) for s in sets]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in sets]
    for rep in range(3):
        outs = [None] * len(sets)
        for i, (s, st) in enumerate(zip(sets, streams)):
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                outs[i] = _work(*s)
        torch.cuda.synchronize()
        for ref, got in zip(refs, outs):
            _check(ref, got)


def test_host_threads_match_sequential():
    sets = [_inputs(seed + 10) for seed in range(3)]
    refs = [_work(*s) for s in sets]
    torch.cuda.synchronize()
    outs = [None] * len(sets)
    errors = []

    def run(i):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for _ in range(2):
                    outs[i] = _work(*sets[i])
            st.synchronize()
        except Exception as e:  # surfaced in the main thread
            errors.append(e)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(sets))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for ref, got in zip(refs, outs):
        _check(ref, got)
