"""ctypes binding of libpatchserve.so (the C ABI in include/patchserve.h).

The library is built in-tree by `__graft_entry__.build()` / `make -C
paper_2501_09253_b200/csrc`.  There is no fallback: if the library is missing or
fails to load, every op raises.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import InputError, IntegrityError

LIB_PATH = os.environ.get("PS_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                         "libpatchserve.so")  # override: experiments only

ABI_VERSION = 3  # include/patchserve.h PS_ABI_VERSION
PS_OK, PS_ERR_INPUT, PS_ERR_INTEGRITY, PS_ERR_CUDA = 0, 1, 2, 3
DTYPE_F32, DTYPE_BF16, DTYPE_F64 = 0, 1, 2

p = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
f32 = C.c_float
f64 = C.c_double


class GemmArgs(C.Structure):
    _fields_ = [
        ("a", p), ("lda", C.c_int), ("M", C.c_int),
        ("a_mode", C.c_int), ("P", C.c_int), ("ps", C.c_int), ("Cp", C.c_int),
        ("b", p), ("N", C.c_int), ("K", C.c_int),
        ("bias", p),
        ("epi", C.c_int), ("out", p), ("ldo", C.c_int), ("out2", p), ("ldo2", C.c_int), ("n_split", C.c_int),
        ("resid", p), ("c_real", C.c_int),
        ("bn", C.c_int), ("out_tiled", C.c_int), ("dbg", p), ("m_map", p), ("m_count", C.c_int),
        ("cta_pair", C.c_int), ("m_count_dev", p),
    ]


_SIGS = {
    "ps_abi_version": ([], C.c_int),
    "ps_last_error": ([], C.c_char_p),
    "ps_launch_count": ([], C.c_uint64),
    "ps_device_check": ([C.c_int], C.c_int),
    "ps_csp_count": ([C.c_int, p, i32, p, p], C.c_int),
    "ps_csp_build": ([C.c_int, p, i32] + [p] * 9, C.c_int),
    "ps_csp_split": ([p, p, p, p, C.c_int, C.c_int, C.c_int, C.c_int, p, C.c_int], C.c_int),
    "ps_csp_split_bias": ([p, p, p, p, C.c_int, C.c_int, C.c_int, p, C.c_int, p, p, p], C.c_int),
    "ps_blend_reassemble": ([p, p, p, p, p, p, C.c_int, C.c_int, C.c_int, p, C.c_int, p], C.c_int),
    "ps_csp_reassemble": ([p, p, p, p, p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int], C.c_int),
    "ps_halo_frames_nchw": ([p, p, C.c_int, p, C.c_int, C.c_int, C.c_int, p], C.c_int),
    "ps_gn_partials": ([p, p, C.c_int, C.c_int, C.c_int, C.c_int, p], C.c_int),
    "ps_gn_partials_sub": ([p, p, C.c_int, C.c_int, C.c_int, C.c_int, p, C.c_int, p, p], C.c_int),
    "ps_gn_finalize": ([p, p, p, C.c_int, C.c_int, C.c_int, f32, p], C.c_int),
    "ps_to_cl": ([p, p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, p, p, C.c_int, p, p, f32, p], C.c_int),
    "ps_frames_cl": ([p, p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, p, p, p, C.c_int, p, p, p], C.c_int),
    "ps_frames_cl_sub": ([p, p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, p, p, p, C.c_int, p, p, p, C.c_int, p,
                          p], C.c_int),
    "ps_halo_strips": ([p, p, C.c_int, C.c_int, C.c_int, p, p, C.c_int], C.c_int),
    "ps_copy_segments": ([p, p, p, C.c_int, p, p, i64], C.c_int),
    "ps_copy_segments_var": ([p, p, p, C.c_int, p, p, p], C.c_int),
    "ps_from_cl": ([p, p, C.c_int, C.c_int, C.c_int, C.c_int, p, p], C.c_int),
    "ps_gemm": ([p, C.POINTER(GemmArgs)], C.c_int),
    "ps_feed_forward": ([p, p, C.c_int, C.c_int, p, p, p, p, C.c_int, C.c_int, C.c_int, p, p, p, C.c_int, p],
                        C.c_int),
    "ps_attention": ([p, p, p, C.c_int, C.c_int, C.c_int, C.c_int, p, p, p, C.c_int, p], C.c_int),
    "ps_attention_pairs": ([p, p, p, C.c_int, C.c_int, C.c_int, C.c_int, p, p, p, C.c_int, p, p], C.c_int),
    "ps_attention_splitkv": ([p, p, p, C.c_int, C.c_int, C.c_int, C.c_int, p, p, p, p, p, p, C.c_int, p, p, p],
                             C.c_int),
    "ps_attention_pairs_splitkv": ([p, p, p, C.c_int, C.c_int, C.c_int, C.c_int, p, p, p, p, p, p, p, C.c_int, p, p,
                                    p], C.c_int),
    "ps_attention_combine": ([p, p, p, p, p, p, p, p, C.c_int, C.c_int, p], C.c_int),
    "ps_kv_peer_maps": ([p, C.c_int, p, p, p, p, C.c_int], C.c_int),
    "ps_attention_peer": ([p, p, p, C.c_int, C.c_int, C.c_int, C.c_int, p, p, p, p, p, p, C.c_int, p, p, p, p, p, p],
                          C.c_int),
    "ps_attention_debug": ([p], C.c_int),
    "ps_attention_trace": ([p], C.c_int),
    "ps_feed_forward_debug": ([p], C.c_int),
    "ps_pairwise_plan": ([i64, p, p, p, p, p, p], C.c_int),
    "ps_cache_predict": ([p, p, C.c_int, C.c_int, i64, p, p, p, p, f64, C.c_int, p, C.c_int, p, C.c_int, p, C.c_int, p, p, p],
                         C.c_int),
    "ps_compact": ([p, p, C.c_int, p, p, p, p], C.c_int),
    "ps_compact_lists": ([p, p, C.c_int, p, C.c_int, p, C.c_int, C.c_int, C.c_int, C.c_int] + [p] * 9, C.c_int),
    "ps_cache_gather": ([p, p, p, p, C.c_int, i64, C.c_int, p, p, p, p, p], C.c_int),
    "ps_cache_fill": ([p, p, p, p, p, C.c_int, i64, C.c_int, p, p, p], C.c_int),
    "ps_cache_update": ([p, p, p, p, p, C.c_int, i64, C.c_int, p, p, p, p, p], C.c_int),
    "ps_cache_evict": ([p, p, p, p, C.c_int], C.c_int),
    "ps_cache_substitute": ([p, p, p, C.c_int, i64, C.c_int, p, p, p, p, C.c_int, p], C.c_int),
    "ps_cache_finish": ([p, p, p, p, p, C.c_int, i64, C.c_int, p, p, p, p, p], C.c_int),
    "ps_select_patches": ([p, p, C.c_int, i64, C.c_int, p, p, p], C.c_int),
    "ps_prompt_bias": ([p, p, p, p, C.c_int, C.c_int, C.c_int, p], C.c_int),
    "ps_blend": ([p, p, p, p, p, C.c_int, C.c_int, C.c_int, p], C.c_int),
    "ps_convert": ([p, p, C.c_int, p, C.c_int, i64], C.c_int),
    "ps_checksum": ([p, p, i64, p], C.c_int),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load():
    """Load and type the library (raises OSError if it is absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if lib.ps_abi_version() != ABI_VERSION:
            raise OSError(f"{LIB_PATH}: ABI version {lib.ps_abi_version()} != {ABI_VERSION} expected by the facade "
                          "(stale build? run `make -C paper_2501_09253_b200/csrc`)")
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == PS_OK:
        return
    msg = load().ps_last_error().decode(errors="replace")
    if rc == PS_ERR_INPUT:
        raise InputError(msg)
    if rc == PS_ERR_INTEGRITY:
        raise IntegrityError(msg)
    raise RuntimeError(f"CUDA error in libpatchserve: {msg}")


# measurement hook (bench.py / tools): when set to an object with .wants(name), .before(name)
# and .after(name), calls of those entry points are bracketed by it (CUDA events on the
# launching stream); None on the product path
TIMER = None


def call(name: str, *args) -> None:
    t = TIMER
    if t is not None and t.wants(name):
        t.before(name)
        check(getattr(load(), name)(*args))
        t.after(name)
        return
    check(getattr(load(), name)(*args))


def launches() -> int:
    return int(load().ps_launch_count())
