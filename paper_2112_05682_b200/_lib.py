"""ctypes loader for the in-tree libmea.so (C ABI: include/mea.h).

Fails loudly when the library is missing: there is no CPU fallback anywhere in the
product path.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmea.so")

# symbol -> (restype, argtypes); mirrors include/mea.h and include/mea_debug.h
_c = ctypes
_i64, _f, _vp, _fp, _sz = _c.c_int64, _c.c_float, _c.c_void_p, _c.POINTER(_c.c_float), _c.c_size_t
_st = _c.c_int
SIGNATURES = {
    "mea_version": (_c.c_char_p, []),
    "mea_status_string": (_c.c_char_p, [_st]),
    "mea_last_error_detail": (_c.c_char_p, []),
    "mea_attention_fwd": (_st, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _st, _st, _f, _vp, _i64, _i64,
                                _vp, _sz, _vp]),
    "mea_attention_fwd_workspace_size": (_st, [_i64, _i64, _i64, _i64, _i64, _st, _i64, _i64, _c.POINTER(_sz)]),
    "mea_attention_fwd_padded": (_st, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _st, _st, _f, _vp, _vp,
                                       _vp]),
    "mea_attention_bwd_padded": (_st, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _st, _f,
                                       _vp, _vp, _vp, _sz, _vp]),
    "mea_attention_fwd_tree": (_st, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _st, _st, _f, _vp, _i64,
                                     _i64, _vp, _sz, _vp]),
    "mea_attention_fwd_tree_workspace_size": (_st, [_i64, _i64, _i64, _i64, _i64, _st, _i64, _i64,
                                                    _c.POINTER(_sz)]),
    "mea_attention_fwd_causal": (_st, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _st, _st, _f, _vp, _vp]),
    "mea_attention_bwd_causal": (_st, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _st, _f, _vp,
                                       _vp, _sz, _vp]),
    "mea_single_query_fwd": (_st, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _st, _st, _f, _vp, _sz, _vp]),
    "mea_single_query_workspace_size": (_st, [_i64, _i64, _i64, _i64, _st, _c.POINTER(_sz)]),
    "mea_attention_partial_fwd": (_st, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _st, _f,
                                        _vp]),
    "mea_single_query_partial": (_st, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _st, _f, _vp, _sz,
                                       _vp]),
    "mea_merge_partials": (_st, [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _st, _vp]),
    "mea_single_query_partial_packed": (_st, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _st, _f, _vp, _sz, _vp]),
    "mea_attention_partial_fwd_packed": (_st, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _st, _f, _vp]),
    "mea_merge_triples": (_st, [_vp, _i64, _i64, _i64, _vp, _st, _vp]),
    "mea_debug_set_option": (_st, [_c.c_char_p, _c.c_int]),
    "mea_debug_read_probe": (_st, [_vp, _sz, _c.c_int, _vp, _vp]),
    "mea_attention_bwd": (_st, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _st, _f, _vp,
                                _vp, _sz, _vp]),
    "mea_attention_bwd_workspace_size": (_st, [_i64, _i64, _i64, _i64, _i64, _st, _c.c_int, _c.POINTER(_sz)]),
    "mea_attention_bwd_deterministic": (_st, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64,
                                              _st, _f, _vp, _vp, _sz, _vp]),
    "mea_attention_bwd_deterministic_workspace_size": (_st, [_i64, _i64, _i64, _i64, _i64, _st, _c.c_int,
                                                             _c.POINTER(_sz)]),
    "mea_fill_synthetic": (_st, [_vp, _i64, _st, _c.c_uint64, _c.c_uint32, _i64, _vp]),
    "mea_debug_umma_tile": (_st, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "mea_profile_enable": (None, [_c.c_int]),
    "mea_profile_read": (_st, [_c.c_char_p, _sz]),
}

_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2112_05682_b200.build` "
                "(this package has no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
