"""The plain-C example (examples/mea_example.c) on the GPU: a C caller of the ABI gets the same
results as the Python binding for the same seeded inputs (forward and lse bit for bit, the fused
backward's dq to its reduction order, the single query bit for bit)."""
import math
import os
import subprocess

import pytest
import torch

from tests.test_abi import c_example_binary

pytestmark = pytest.mark.gpu


def test_c_example_matches_python_binding(tmp_path):
    from paper_2112_05682_b200 import _lib, api
    exe = c_example_binary(str(tmp_path))
    env = dict(os.environ, LD_LIBRARY_PATH=os.path.dirname(_lib.LIB_PATH) + ":" + os.environ.get("LD_LIBRARY_PATH", ""))
    r = subprocess.run([exe], capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    vals = {}
    for line in r.stdout.splitlines()[1:]:
        name, *xs = line.split()
        vals[name] = torch.tensor([float(x) for x in xs], dtype=torch.float32)  # %.8e round-trips f32

    B, H, n, d = 1, 2, 1000, 64
    q = torch.empty((B, n, H, d), dtype=torch.bfloat16, device="cuda")
    k, v, do = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
    for t, tid in ((q, 1), (k, 2), (v, 3), (do, 4)):
        api.mea_fill_synthetic(t, 0, tid)
    out, lse = api.mea_attention_fwd(q, k, v, want_lse=True, scale=1 / math.sqrt(d))
    dq, dk, dv = api.mea_attention_bwd(q, k, v, out, do, lse=lse, scale=1 / math.sqrt(d))
    sq = api.mea_single_query_fwd(q[:, 0].contiguous(), k, v, scale=1 / math.sqrt(d))
    torch.cuda.synchronize()
    flat = lambda t, m: t.reshape(-1)[:m].float().cpu()
    assert torch.equal(vals["out"], flat(out, 8))
    assert torch.allclose(vals["lse"], flat(lse, 4), rtol=0, atol=1e-6)
    assert torch.allclose(vals["dq"], flat(dq, 8), rtol=1e-2, atol=1e-3)
    assert torch.equal(vals["sq"], flat(sq, 8))
