"""Bring-up probes on the GPU: tcgen05 descriptors/TMEM layout, and the input generator."""
import numpy as np
import pytest
import torch

from synth import gen

pytestmark = pytest.mark.gpu


def test_umma_tile_descriptors():
    """S = A B^T (SS MMA) and O = bf16(S) V (TS MMA, P from TMEM) on one tile."""
    from paper_2112_05682_b200 import api
    g = torch.Generator().manual_seed(0)
    a = torch.randn(128, 64, generator=g).bfloat16()
    b = torch.randn(128, 64, generator=g).bfloat16()
    v = torch.randn(128, 64, generator=g).bfloat16()
    s, o = api.mea_debug_umma_tile(a.cuda(), b.cuda(), v.cuda())
    torch.cuda.synchronize()
    s_ref = a.double() @ b.double().T
    np.testing.assert_allclose(s.cpu().double().numpy(), s_ref.numpy(), atol=1e-3, rtol=1e-4)
    p = s.cpu().bfloat16().double()                 # what the kernel stores to TMEM
    o_ref = p @ v.double()
    np.testing.assert_allclose(o.cpu().double().numpy(), o_ref.numpy(), atol=2e-2, rtol=1e-3)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_device_generator_bit_identical(dtype):
    from paper_2112_05682_b200 import api
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    n = 100_003
    t = torch.empty(n, dtype=tdt, device="cuda")
    api.mea_fill_synthetic(t, 12345, gen.TENSOR_V, offset=7)
    host = gen.irwin_hall_values(12345, gen.TENSOR_V, np.arange(7, 7 + n, dtype=np.uint64))
    host = gen.round_to_bf16(host) if dtype == "bf16" else host.astype(np.float32)
    got = t.float().cpu().numpy()
    assert np.array_equal(got.view(np.uint32), np.asarray(host, dtype=np.float32).view(np.uint32))
