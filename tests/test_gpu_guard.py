"""Out-of-bounds write checks (compute-sanitizer is not available on this pool): every output
tensor is a view into a larger buffer whose guard regions before and after hold a sentinel;
after each call on ragged shapes (rows and keys not multiples of any tile) the guards must be
untouched and the outputs finite. Covers the epilogues of every entry point.
"""
import pytest
import torch

pytestmark = pytest.mark.gpu

GUARD = 4096   # elements on each side


def guarded(shape, dtype):
    n = 1
    for s in shape:
        n *= s
    buf = torch.full((n + 2 * GUARD,), 1234.5, dtype=dtype, device="cuda")
    # keep 16-byte alignment of the view: GUARD elements of >= 2 bytes is a multiple of 16 bytes
    return buf, buf[GUARD:GUARD + n].view(shape)


def check(buf, view):
    torch.cuda.synchronize()
    assert (buf[:GUARD] == 1234.5).all() and (buf[-GUARD:] == 1234.5).all(), "write outside the output"
    assert torch.isfinite(view.float()).all(), "output not fully written (or non-finite)"


def rnd(*shape, dtype=torch.bfloat16):
    return (torch.randn(*shape, device="cuda") * 0.5).to(dtype)


@pytest.mark.parametrize("d", [64, 128])
def test_no_out_of_bounds_writes(d):
    from paper_2112_05682_b200 import api
    torch.manual_seed(d)
    B, nq, nk, H = 2, 301, 333, 3
    q, k, v, do = rnd(B, nq, H, d), rnd(B, nk, H, d), rnd(B, nk, H, d), rnd(B, nq, H, d)
    for od in (torch.bfloat16, torch.float32):
        ob, o = guarded((B, nq, H, d), od)
        lb, lse = guarded((B, H, nq), torch.float32)
        api.mea_attention_fwd(q, k, v, out=o, lse=lse)
        check(ob, o); check(lb, lse)
        api.mea_attention_fwd(q, k, v, out=o, lse=lse, q_chunk=256, k_chunk=128)
        check(ob, o); check(lb, lse)
        api.mea_attention_fwd_tree(q, k, v, out=o, lse=lse, q_chunk=256, k_chunk=128)
        check(ob, o); check(lb, lse)
        api.mea_attention_fwd_padded(q, k, v, torch.tensor([5, 300], dtype=torch.int32, device="cuda"), out=o, lse=lse)
        check(ob, o); check(lb, lse)
    out, lse0 = api.mea_attention_fwd(q, k, v, want_lse=True)
    gb = [guarded(t.shape, torch.bfloat16) for t in (q, k, v)]
    api.mea_attention_bwd(q, k, v, out, do, lse=lse0, dq=gb[0][1], dk=gb[1][1], dv=gb[2][1])
    for b_, t in gb:
        check(b_, t)
    api.mea_attention_bwd_deterministic(q, k, v, out, do, lse=lse0, dq=gb[0][1], dk=gb[1][1], dv=gb[2][1])
    for b_, t in gb:
        check(b_, t)
    kl = torch.tensor([1, 200], dtype=torch.int32, device="cuda")
    op, lp = api.mea_attention_fwd_padded(q, k, v, kl, want_lse=True)
    api.mea_attention_bwd_padded(q, k, v, op, do, kl, lse=lp, dq=gb[0][1], dk=gb[1][1], dv=gb[2][1])
    for b_, t in gb:
        check(b_, t)
    # causal (n_q == n_k)
    qc, kc, vc, dc = rnd(B, nq, H, d), rnd(B, nq, H, d), rnd(B, nq, H, d), rnd(B, nq, H, d)
    ob, o = guarded((B, nq, H, d), torch.bfloat16)
    lb, lse = guarded((B, H, nq), torch.float32)
    api.mea_attention_fwd_causal(qc, kc, vc, out=o, lse=lse)
    check(ob, o); check(lb, lse)
    gc = [guarded(t.shape, torch.bfloat16) for t in (qc, kc, vc)]
    api.mea_attention_bwd_causal(qc, kc, vc, o, dc, lse=lse, dq=gc[0][1], dk=gc[1][1], dv=gc[2][1])
    for b_, t in gc:
        check(b_, t)
    # single query
    sb, so = guarded((B, H, d), torch.float32)
    api.mea_single_query_fwd(rnd(B, H, d), k, v, out=so)
    check(sb, so)
