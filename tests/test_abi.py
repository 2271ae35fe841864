"""CPU-side checks of the boundary: the library builds, loads and exports every symbol
declared in include/*.h; the Python binding marshals exactly those names. No compute
calls (no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in ("mea.h", "mea_debug.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        names |= set(re.findall(r"MEA_API\s+[\w\s\*]+?\b(mea_\w+)\s*\(", src))
    return names


@pytest.fixture(scope="module")
def lib():
    from paper_2112_05682_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2112_05682_b200 import build
        build.build()
    return _lib.load()


def test_header_declares_north_star_entry_points():
    names = declared_symbols()
    for n in ("mea_attention_fwd", "mea_single_query_fwd", "mea_attention_bwd", "mea_merge_partials",
              "mea_single_query_partial"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), f"libmea.so does not export {name}"


def test_binding_signatures_cover_header():
    from paper_2112_05682_b200 import _lib
    assert declared_symbols() == set(_lib.SIGNATURES)


def test_host_only_calls(lib):
    from paper_2112_05682_b200 import api
    assert lib.mea_version().decode().startswith("mea")
    assert lib.mea_status_string(2) == b"MEA_ERR_EMPTY_KEYS"
    n = ctypes.c_size_t(123)
    # default schedule needs no workspace; key-chunk summaries do (paper's O(sqrt n) buffers)
    assert lib.mea_attention_fwd_workspace_size(1, 16, 16384, 16384, 64, 1, 0, 0, ctypes.byref(n)) == 0
    assert n.value == 0
    assert lib.mea_attention_fwd_workspace_size(1, 16, 16384, 16384, 64, 1, 1024, 4096, ctypes.byref(n)) == 0
    # one query chunk of summaries alive + the fused merge's arrival counters
    # (one per (b, h, 256-row query block of the window), after 16-byte alignment)
    assert n.value == 4 * 16 * 1024 * 66 * 4 + 16 * 4 * 4
    assert lib.mea_attention_fwd_workspace_size(1, 16, 16384, 16384, 64, 1, 0, 4096, ctypes.byref(n)) == 0
    assert n.value == 4 * 16 * 16384 * 66 * 4 + 16 * 64 * 4    # q_chunk 0: all rows in one launch
    assert lib.mea_attention_fwd_workspace_size(1, 16, 16384, 16384, 64, 1, 300, 4096, ctypes.byref(n)) == 0
    assert n.value == 4 * 16 * 512 * 66 * 4 + 16 * 2 * 4       # q_chunk rounded up to the 256-row CTA
    assert lib.mea_attention_fwd_workspace_size(1, 16, 16384, 16384, 64, 1, 1024, 16384, ctypes.byref(n)) == 0
    assert n.value == 0                          # k_chunk >= n_k: no key split, q_chunk has no effect
    # single-query workspace is independent of n_k once the split count saturates
    a, b = ctypes.c_size_t(), ctypes.c_size_t()
    lib.mea_single_query_workspace_size(1, 1, 1 << 20, 64, 1, ctypes.byref(a))
    lib.mea_single_query_workspace_size(1, 1, 1 << 24, 64, 1, ctypes.byref(b))
    assert a.value == b.value > 0
    # validation happens before any launch: these never touch the GPU
    assert api.mea_attention_fwd_workspace_size(1, 1, 8, 8, 64, 1) == 0
    assert lib.mea_attention_fwd(None, None, None, None, 1, 1, 4, 0, 64, 1, 1, 1.0, None, 0, 0, None, 0,
                                 None) == 2  # empty keys
    assert lib.mea_attention_fwd(None, None, None, None, 1, 1, 0, 5, 64, 1, 1, 1.0, None, 0, 0, None, 0,
                                 None) == 0  # n_q == 0 no-op
    assert lib.mea_attention_fwd(None, None, None, None, 0, 1, 4, 5, 64, 1, 1, 1.0, None, 0, 0, None, 0,
                                 None) == 1
    assert lib.mea_attention_fwd(None, None, None, None, 1, 1, 4, 5, 64, 2, 1, 1.0, None, 0, 0, None, 0,
                                 None) == 3  # MEA_F32_SPLIT needs float32 output
    assert lib.mea_attention_fwd(None, None, None, None, 1, 1, 4, 5, 64, 7, 1, 1.0, None, 0, 0, None, 0,
                                 None) == 1  # bad dtype
    assert lib.mea_attention_fwd(None, None, None, None, 1, 1, 4, 5, 64, 1, 1, float("nan"), None, 0, 0, None,
                                 0, None) == 1
    p = ctypes.c_void_p(16)
    assert lib.mea_attention_fwd(p, p, p, p, 1, 1, 4, 5, 32, 1, 1, 1.0, None, 0, 0, None, 0, None) == 3
    q = ctypes.c_void_p(8)  # misaligned
    assert lib.mea_attention_fwd(q, p, p, p, 1, 1, 4, 5, 64, 1, 1, 1.0, None, 0, 0, None, 0, None) == 4
    assert lib.mea_single_query_fwd(p, p, p, p, 1, 1, 0, 64, 1, 1, 1.0, None, 0, None) == 2
    assert lib.mea_merge_partials(p, p, p, 0, 1, 1, 64, p, 1, None) == 2
    assert b"no partials" in lib.mea_last_error_detail()


def test_host_only_validation_of_the_newer_entry_points(lib):
    """Causal, partial, d = 128 and backward argument checks all happen before any launch."""
    p = ctypes.c_void_p(16)
    # causal: bf16 only (status 3 = unsupported); n == 0 is a no-op; n_k == 0 impossible (n_q == n_k)
    assert lib.mea_attention_fwd_causal(p, p, p, p, 1, 1, 8, 64, 0, 0, 1.0, None, None) == 3
    assert lib.mea_attention_fwd_causal(p, p, p, p, 1, 1, 0, 64, 1, 1, 1.0, None, None) == 0
    assert lib.mea_attention_fwd_causal(p, p, p, p, 1, 1, 8, 32, 1, 1, 1.0, None, None) == 3  # d = 32
    assert lib.mea_attention_bwd_causal(p, p, p, p, p, p, p, p, 1, 1, 8, 64, 1, 0.0, None, None, 0, None) == 3
    # key chunks at d = 128 need their summaries' workspace (status 5); f32 key chunks: unsupported
    assert lib.mea_attention_fwd(p, p, p, p, 1, 1, 300, 300, 128, 1, 1, 1.0, None, 0, 128, None, 0, None) == 5
    n1 = ctypes.c_size_t(0)
    assert lib.mea_attention_fwd_workspace_size(1, 2, 300, 300, 128, 1, 0, 128, ctypes.byref(n1)) == 0
    assert n1.value == 3 * 2 * 300 * 130 * 4
    assert lib.mea_attention_fwd(p, p, p, p, 1, 1, 300, 300, 64, 0, 0, 1.0, None, 0, 128, None, 0, None) == 3
    # backward: d outside {64, 128}, f32 inputs
    assert lib.mea_attention_bwd(p, p, p, p, p, p, p, p, 1, 1, 8, 8, 32, 1, 1.0, None, None, 0, None) == 3
    assert lib.mea_attention_bwd(p, p, p, p, p, p, p, p, 1, 1, 8, 8, 64, 0, 1.0, None, None, 0, None) == 3
    # backward workspace too small (status 5) before any launch
    assert lib.mea_attention_bwd(p, p, p, p, p, p, p, p, 1, 1, 8, 8, 64, 1, 1.0, None, p, 16, None) == 5
    # partial forward: bf16 d in {64, 128}; n_q == 0 no-op
    assert lib.mea_attention_partial_fwd(p, p, p, p, p, p, 1, 1, 8, 8, 96, 1, 1.0, None) == 3
    assert lib.mea_attention_partial_fwd(p, p, p, p, p, p, 1, 1, 0, 8, 64, 1, 1.0, None) == 0
    # d = 128 workspace sizes: forward none; backward (fused kernel, bwd128_sm100a.cu) delta and
    # lse2 (each padded to 128 rows per (b, h), 256-byte aligned) + the f32 dQ accumulator
    n = ctypes.c_size_t(7)
    assert lib.mea_attention_fwd_workspace_size(1, 2, 300, 300, 128, 1, 0, 0, ctypes.byref(n)) == 0
    assert n.value == 0
    assert lib.mea_attention_bwd_workspace_size(1, 2, 300, 300, 128, 1, 1, ctypes.byref(n)) == 0
    assert n.value == 2 * (2 * 384 * 4) + 300 * 2 * 128 * 4
    assert lib.mea_attention_bwd_workspace_size(1, 2, 300, 300, 64, 1, 1, ctypes.byref(n)) == 0
    assert n.value > 300 * 2 * 64 * 4                       # d = 64 fused: + dq accumulator


def test_tree_schedule_workspace_is_logarithmic(lib):
    """mea_attention_fwd_tree_workspace_size: (floor(log2(chunks)) + 2) summaries per
    query row, against the flat schedule's `chunks`; MEA_CHUNK_SQRT_N = ceil(sqrt(n_k)) keys
    (rounded up to the 128-key tile) in both. Host-only argument checks."""
    import math
    p = ctypes.c_void_p(16)
    B, H, d = 1, 2, 64
    row = B * H * (d + 2) * 4
    for n_k in (128, 1000, 16384, 1 << 20):
        kc = math.ceil(math.sqrt(n_k))
        chunks = -(-n_k // (-(-kc // 128) * 128))
        t, f = ctypes.c_size_t(0), ctypes.c_size_t(0)
        assert lib.mea_attention_fwd_tree_workspace_size(B, H, 512, n_k, d, 1, 256, -1, ctypes.byref(t)) == 0
        assert t.value == (int(math.floor(math.log2(chunks))) + 2) * 256 * row
        assert lib.mea_attention_fwd_workspace_size(B, H, 512, n_k, d, 1, 256, -1, ctypes.byref(f)) == 0
        flat = chunks * 256 * row   # + merge arrival counters when the in-kernel merge applies (<= 16)
        assert f.value == ((flat + 15) // 16 * 16 + B * H * 4 if 1 < chunks <= 16 else flat if chunks > 16 else 0)
        if chunks >= 8:
            assert t.value < f.value
    # k_chunk 0 also means sqrt(n); explicit chunk, whole rows (q_chunk 0); d = 128 rows per pass
    t = ctypes.c_size_t(0)
    assert lib.mea_attention_fwd_tree_workspace_size(1, 1, 300, 16384, 64, 1, 0, 0, ctypes.byref(t)) == 0
    assert t.value == (7 + 2) * 300 * 66 * 4
    assert lib.mea_attention_fwd_tree_workspace_size(1, 1, 300, 16384, 64, 1, 0, 4096, ctypes.byref(t)) == 0
    assert t.value == (2 + 2) * 300 * 66 * 4
    assert lib.mea_attention_fwd_tree_workspace_size(1, 1, 300, 16384, 128, 1, 100, 4096, ctypes.byref(t)) == 0
    assert t.value == (2 + 2) * 128 * 130 * 4
    # invalid / unsupported: k_chunk -2, f32, d = 32, missing workspace (status 5)
    assert lib.mea_attention_fwd_tree_workspace_size(1, 1, 8, 8, 64, 1, 0, -2, ctypes.byref(t)) == 1
    assert lib.mea_attention_fwd_tree_workspace_size(1, 1, 8, 8, 64, 0, 0, 0, ctypes.byref(t)) == 3
    assert lib.mea_attention_fwd_tree(p, p, p, p, 1, 1, 8, 8, 32, 1, 1, 1.0, None, 0, 0, None, 0, None) == 3
    assert lib.mea_attention_fwd_tree(p, p, p, p, 1, 1, 8, 8, 64, 1, 1, 1.0, None, 0, 0, None, 0, None) == 5
    assert lib.mea_attention_fwd_tree(p, p, p, p, 1, 1, 8, 0, 64, 1, 1, 1.0, None, 0, 0, None, 0, None) == 2


def test_padded_entry_points_validate_on_the_host(lib):
    """Key padding: kv_lens NULL (1) / misaligned (4) / non-bf16 (3) rejected before any launch."""
    p = ctypes.c_void_p(16)
    assert lib.mea_attention_fwd_padded(p, p, p, p, 1, 1, 8, 8, 64, 1, 1, 1.0, None, None, None) == 1
    assert lib.mea_attention_fwd_padded(p, p, p, p, 1, 1, 8, 8, 64, 1, 1, 1.0, None, ctypes.c_void_p(18), None) == 4
    assert lib.mea_attention_fwd_padded(p, p, p, p, 1, 1, 8, 8, 64, 0, 0, 1.0, None, p, None) == 3
    assert lib.mea_attention_bwd_padded(p, p, p, p, p, p, p, p, 1, 1, 8, 8, 64, 1, 1.0, None, None, None, 0, None) == 1
    assert lib.mea_attention_bwd_padded(p, p, p, p, p, p, p, p, 1, 1, 8, 8, 64, 0, 1.0, None, p, None, 0, None) == 3
    assert lib.mea_attention_bwd_padded(p, p, p, p, p, p, p, p, 1, 1, 8, 8, 64, 1, 1.0, None, p, p, 16, None) == 5


def test_stats_pass_workspace_is_lse_only(lib):
    """B0 (lse not given): at d = 64 the statistics pass writes lse only, so the
    backward workspace grows by the lse buffer (4 B per query row) and no output-sized scratch;
    d = 128 still reruns the forward (output in scratch)."""
    B, H, n = 1, 16, 16384
    for fn in (lib.mea_attention_bwd_workspace_size, lib.mea_attention_bwd_deterministic_workspace_size):
        a, b = ctypes.c_size_t(0), ctypes.c_size_t(0)
        assert fn(B, H, n, n, 64, 1, 1, ctypes.byref(a)) == 0
        assert fn(B, H, n, n, 64, 1, 0, ctypes.byref(b)) == 0
        assert b.value - a.value == B * H * n * 4
        assert fn(B, H, n, n, 128, 1, 1, ctypes.byref(a)) == 0
        assert fn(B, H, n, n, 128, 1, 0, ctypes.byref(b)) == 0
        assert b.value - a.value == B * H * n * 4 + B * n * H * 128 * 2


def c_example_binary(out_dir):
    """Compile examples/mea_example.c (plain C99 against include/mea.h) and link libmea.so."""
    import shutil
    import subprocess
    from paper_2112_05682_b200 import _lib
    cc = shutil.which("gcc") or shutil.which("cc")
    cuda_inc = "/usr/local/cuda/include"
    if cc is None or not os.path.exists(os.path.join(cuda_inc, "cuda_runtime_api.h")):
        pytest.skip("no C compiler / CUDA headers")
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2112_05682_b200 import build
        build.build()
    exe = os.path.join(out_dir, "mea_example")
    cmd = [cc, "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", cuda_inc,
           os.path.join(ROOT, "examples", "mea_example.c"), "-L", os.path.dirname(_lib.LIB_PATH), "-lmea",
           "-L", "/usr/local/cuda/lib64", "-lcudart", "-lm", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_compiles_and_links(tmp_path):
    """The C ABI is usable from plain C99: the example builds warning-free and links libmea.so."""
    assert os.path.exists(c_example_binary(str(tmp_path)))
