"""ctypes binding of the C ABI in include/fic_b200.h (libfic_b200.so).

The library is built in-tree (``make`` / ``__graft_entry__.build()``).  There
is no fallback: if it is missing or no CUDA device is present, every entry
point raises.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FIC_B200_LIB selects another build of the same library (kernel experiments)
LIB_PATH = os.environ.get("FIC_B200_LIB") or os.path.join(HERE, "libfic_b200.so")

FIC_OK, FIC_EINVAL, FIC_ECUDA, FIC_ENOMEM = 0, 1, 2, 3


class FicParams(ctypes.Structure):
    _fields_ = [
        ("range_size", ctypes.c_int32),
        ("domain_size", ctypes.c_int32),
        ("stride", ctypes.c_int32),
        ("isometries", ctypes.c_int32),
        ("strategy", ctypes.c_int32),
        ("fd_source", ctypes.c_int32),
        ("has_delta", ctypes.c_int32),
        ("matcher", ctypes.c_int32),
        ("delta", ctypes.c_double),
        ("h_ln_table", ctypes.POINTER(ctypes.c_double)),
        ("ln_len", ctypes.c_int32),
        ("shard_index", ctypes.c_int32),
        ("shard_count", ctypes.c_int32),
        ("max_segment", ctypes.c_int32),
        ("small_pool", ctypes.c_int32),
        ("h_fd_weights_dom", ctypes.POINTER(ctypes.c_double)),
        ("h_fd_weights_rng", ctypes.POINTER(ctypes.c_double)),
        ("n_fd_weights_dom", ctypes.c_int32),
        ("n_fd_weights_rng", ctypes.c_int32),
    ]


class FicStats(ctypes.Structure):
    _fields_ = [
        ("n_ranges", ctypes.c_int64),
        ("n_domains", ctypes.c_int64),
        ("comparisons", ctypes.c_int64),
        ("mean_pool_size", ctypes.c_double),
        ("fd_min", ctypes.c_double),
        ("fd_max", ctypes.c_double),
        ("half_width", ctypes.c_double),
        ("ms_fd", ctypes.c_double),
        ("ms_pool", ctypes.c_double),
        ("ms_match", ctypes.c_double),
        ("ms_tensor", ctypes.c_double),
        ("ms_exact", ctypes.c_double),
        ("ms_total", ctypes.c_double),
        ("exact_evals", ctypes.c_int64),
        ("tensor_candidates", ctypes.c_int64),
        ("tensor_comparisons", ctypes.c_int64),
        ("tensor_tiles", ctypes.c_int32),
        ("exact_tiles", ctypes.c_int32),
        ("work_items", ctypes.c_int32),
        ("kernel_launches", ctypes.c_int32),
        ("ms_pool_main", ctypes.c_double),
        ("graph", ctypes.c_int64),
        ("ms_sl", ctypes.c_double),
        ("sl_entries", ctypes.c_int64),
        ("hl_entries", ctypes.c_int64),
        ("hl_tests", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


# every symbol include/fic_b200.h declares
EXPORTS = ("fic_encode_v1", "fic_plan_v1", "fic_pool_v1", "fic_dbc_v1", "fic_dbc_v2", "fic_decode_v1",
           "fic_decode_step_v1", "fic_shard_pack_v1", "fic_shard_unpack_v1",
           "fic_guard_selftest_v1", "fic_last_error", "fic_abi_version", "fic_release")

_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the library; raise loudly when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"CUDA library {path} is missing: build it with `make` or "
            "`python -c 'import __graft_entry__; __graft_entry__.build()'`; "
            "there is no CPU fallback")
    lib = ctypes.CDLL(path)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    P = ctypes.POINTER
    lib.fic_encode_v1.argtypes = [vp, i32, i32, P(FicParams), vp, vp, vp, vp, P(FicStats), vp]
    lib.fic_plan_v1.argtypes = [vp, i32, i32, P(FicParams), vp, vp, vp, vp, vp, P(FicStats), vp]
    lib.fic_dbc_v1.argtypes = [vp, i64, i32, i32, P(ctypes.c_double), i32,
                               P(ctypes.c_double), i32, vp, vp]
    lib.fic_dbc_v2.argtypes = [vp, i64, i32, i32, i32, P(ctypes.c_double), i32,
                               P(ctypes.c_double), i32, vp, vp]
    lib.fic_dbc_v2.restype = ctypes.c_int
    lib.fic_decode_v1.argtypes = [vp, i32, i32, i32, i32, i32, i32, ctypes.c_double, vp, vp, vp]
    lib.fic_pool_v1.argtypes = [vp, i32, i32, P(FicParams), vp, vp, vp, vp, vp, vp]
    lib.fic_decode_step_v1.argtypes = [vp, i32, i32, i32, i32, i32, vp, vp, vp, vp]
    lib.fic_shard_pack_v1.argtypes = [vp, vp, vp, i64, vp, vp]
    lib.fic_shard_unpack_v1.argtypes = [vp, i64, vp, vp, vp, vp, vp]
    for name in ("fic_encode_v1", "fic_plan_v1", "fic_pool_v1", "fic_dbc_v1", "fic_decode_v1",
                 "fic_decode_step_v1", "fic_shard_pack_v1", "fic_shard_unpack_v1"):
        getattr(lib, name).restype = ctypes.c_int
    lib.fic_guard_selftest_v1.argtypes = [i32]
    lib.fic_guard_selftest_v1.restype = ctypes.c_int
    lib.fic_last_error.restype = ctypes.c_char_p
    lib.fic_last_error.argtypes = []
    lib.fic_abi_version.restype = ctypes.c_int
    lib.fic_release.restype = None
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a status code to the reference's exception types."""
    if rc == FIC_OK:
        return
    msg = load().fic_last_error().decode()
    if rc == FIC_EINVAL:
        raise ValueError(msg)
    if rc == FIC_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"CUDA error in libfic_b200: {msg}")
