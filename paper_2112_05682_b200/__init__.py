"""paper_2112_05682_b200 — memory-efficient exact attention (arXiv 2112.05682) on B200.

The product is the C-ABI library ``libmea.so`` (include/mea.h) built from ``csrc/``
for sm_100a; ``api`` is a thin ctypes binding with the same function names.
"""
from .api import (  # noqa: F401
    MEA_BF16, MEA_F32, EmptyKeysError, MeaError, mea_attention_bwd, mea_attention_bwd_deterministic,
    mea_attention_bwd_deterministic_workspace_size, mea_attention_bwd_workspace_size,
    mea_attention_bwd_causal, mea_attention_fwd_causal, mea_attention_partial_fwd,
    mea_attention_fwd, mea_attention_fwd_workspace_size, mea_debug_umma_tile, mea_fill_synthetic,
    MEA_CHUNK_SQRT_N, mea_attention_fwd_tree, mea_attention_fwd_tree_workspace_size,
    mea_attention_fwd_padded, mea_attention_bwd_padded,
    mea_merge_partials, mea_single_query_fwd, mea_single_query_partial, mea_single_query_workspace_size, version,
)
