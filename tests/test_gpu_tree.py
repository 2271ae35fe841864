"""GPU parity of the multi-stage (tree) summarisation schedule:
mea_attention_fwd_tree against the float64 oracle — the definition (O1) and O5t, the same binary
counter written out in numpy (pinned to O1 in tests/test_oracle.py) — on the same generated
inputs, bf16 tolerances. Shapes cover ragged key chunks, one chunk, the sqrt(n) default, query
chunks, d = 128 and a peak workspace that really is logarithmic.
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
from tests import helpers as Hh

pytestmark = pytest.mark.gpu


def _tree(q, k, v, scale, **kw):
    from paper_2112_05682_b200 import api
    out, lse = api.mea_attention_fwd_tree(Hh.to_dev(q, torch.bfloat16), Hh.to_dev(k, torch.bfloat16),
                                          Hh.to_dev(v, torch.bfloat16), scale=scale, want_lse=True,
                                          out_dtype=torch.float32, **kw)
    torch.cuda.synchronize()
    return out.double().cpu().numpy(), lse.double().cpu().numpy()


@pytest.mark.parametrize("B,n_q,n_k,H,d,q_chunk,k_chunk", [
    (1, 1, 1, 1, 64, 0, -1),            # one key, one chunk
    (1, 300, 1000, 2, 64, 0, 128),      # 8 chunks, ragged last
    (2, 257, 3000, 1, 64, 256, -1),     # sqrt(n) -> 128-key chunks (24), two query passes
    (1, 200, 1300, 2, 64, 0, 256),      # 6 chunks: levels 1 and 2 left at the end
    (1, 130, 1000, 2, 128, 100, 128),   # d = 128, 128-row query passes
])
def test_tree_schedule_matches_oracle(B, n_q, n_k, H, d, q_chunk, k_chunk):
    q, k, v = Hh.host_inputs(B, n_q, n_k, H, d, seed=41)
    scale = 1 / math.sqrt(d)
    ref, ref_lse = O.mha_forward(q, k, v, scale)
    got, lse = _tree(q, k, v, scale, q_chunk=q_chunk, k_chunk=k_chunk)
    Hh.assert_close_bf16(got, ref)
    assert np.abs(lse - ref_lse).max() < 1e-3
    # and O5t (the binary counter in float64) on one head, on the bf16-rounded inputs
    qb, kb, vb = (np.asarray(torch.tensor(x).bfloat16().double()) for x in (q, k, v))
    kc = 128 * math.ceil((math.ceil(math.sqrt(n_k)) if k_chunk < 0 else k_chunk) / 128)
    o5t, lse5t, _ = O.tree_summarize(qb[0, :, 0], kb[0, :, 0], vb[0, :, 0], scale, kc)
    Hh.assert_close_bf16(got[0, :, 0], o5t)
    assert np.abs(lse[0, 0] - lse5t).max() < 1e-3


def test_tree_equals_default_forward_and_workspace_is_small():
    """n = 16384 with sqrt(n) chunks (128 of them): same result as the online forward; peak
    allocation = the logarithmic workspace, far below Figure 1's flat summaries."""
    from paper_2112_05682_b200 import api
    from synth import gen
    B, n, H, d = 1, 16384, 2, 64
    q = torch.empty((B, n, H, d), dtype=torch.bfloat16, device="cuda")
    k, v = torch.empty_like(q), torch.empty_like(q)
    for t, tid in ((q, gen.TENSOR_Q), (k, gen.TENSOR_K), (v, gen.TENSOR_V)):
        api.mea_fill_synthetic(t, 0, tid)
    ref = api.mea_attention_fwd(q, k, v)
    ws_tree = api.mea_attention_fwd_tree_workspace_size(B, H, n, n, d, api.MEA_BF16, 1024, api.MEA_CHUNK_SQRT_N)
    ws_flat = api.mea_attention_fwd_workspace_size(B, H, n, n, d, api.MEA_BF16, 1024, api.MEA_CHUNK_SQRT_N)
    assert ws_tree == (7 + 2) * B * H * 1024 * (d + 2) * 4
    assert ws_flat == 128 * B * H * 1024 * (d + 2) * 4   # 128 splits: merged by merge_rows, no counters
    out = torch.empty_like(q)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    api.mea_attention_fwd_tree(q, k, v, out=out, q_chunk=1024)
    torch.cuda.synchronize()
    assert torch.cuda.max_memory_allocated() - base <= ws_tree + (1 << 20)
    assert (out.float() - ref.float()).abs().max().item() < 1e-2
    rows = np.array([0, 4095, 16383])
    kk = gen.normal_tensor((B, n, H, d), 0, gen.TENSOR_K, "bf16").astype(np.float64)
    vv = gen.normal_tensor((B, n, H, d), 0, gen.TENSOR_V, "bf16").astype(np.float64)
    qr = gen.rows_of((B, n, H, d), 0, gen.TENSOR_Q, 0, rows, 1)
    r, _ = O.naive(qr, kk[0, :, 1], vv[0, :, 1], 1 / math.sqrt(d))
    Hh.assert_close_bf16(out[0, rows, 1].double().cpu().numpy(), r)
