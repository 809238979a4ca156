"""ctypes binding of libkrpg.so (the C ABI declared in include/krpg.h).

The shared library is built in-tree (``lib/libkrpg.so``) by :func:`build`.
There is no fallback: if the library or a CUDA device is missing, every call
fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
# KRPG_LIB_VARIANT=checked selects the bounds-checked build (make CHECKED=1, tests only)
LIB_PATH = os.path.join(PKG, "lib", "libkrpg_checked.so" if os.environ.get("KRPG_LIB_VARIANT") == "checked"
                        else "libkrpg.so")
HEADER = os.path.join(ROOT, "include", "krpg.h")

KRPG_OK = 0
KRPG_INVALID_ARGUMENT = 1
KRPG_RUNTIME_ERROR = 2
KRPG_CUDA_ERROR = 3
EXCLUDED = 0xFFFFFFFF
STORE_F64, STORE_F32 = 0, 1
MODE_TWO_STAGE, MODE_ONE_STAGE = 0, 1


class KrpgError(RuntimeError):
    """std::runtime_error analogue (reference: degenerate draws, zero KRP)."""


class KrpgInvalidArgument(KrpgError, ValueError):
    """std::invalid_argument analogue (bad shapes, indices, values)."""


class KrpgCudaError(KrpgError):
    pass


def build(force: bool = False, quiet: bool = True) -> str:
    """Compile libkrpg.so for sm_100a (nvcc cross-compiles without a GPU)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-C", os.path.join(PKG, "csrc"), "-j8"], check=True,
                       stdout=subprocess.DEVNULL if quiet else None)
    else:
        subprocess.run(["make", "-C", os.path.join(PKG, "csrc"), "-j8"], check=True,
                       stdout=subprocess.DEVNULL if quiet else None)
    return LIB_PATH


_u32, _u64, _i64, _int = C.c_uint32, C.c_uint64, C.c_int64, C.c_int
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p

_SIGS = {
    "krpg_last_error": ([], C.c_char_p),
    "krpg_device_count": ([], _int),
    "krpg_create": ([C.POINTER(_dp), C.POINTER(_u64), _u32, _u32, _u32, _int, C.POINTER(_vp)], _int),
    "krpg_create_device": ([C.POINTER(_vp), C.POINTER(_u64), _u32, _u32, _u32, _int, C.POINTER(_vp)], _int),
    "krpg_destroy": ([_vp], _int),
    "krpg_info": ([_vp, C.POINTER(_u32), C.POINTER(_u32), C.POINTER(_u64)], _int),
    "krpg_factor_gram": ([_vp, _u32, _dp], _int),
    "krpg_factor": ([_vp, _u32, _dp], _int),
    "krpg_tree_shape": ([_vp, _u32, C.POINTER(_u64), C.POINTER(_u64)], _int),
    "krpg_node_gram": ([_vp, _u32, _u64, _dp], _int),
    "krpg_tree_grams": ([_vp, _u32, _dp], _int),
    "krpg_sample": ([_vp, _i64, _u64, _u64, _u64, _u32, C.POINTER(_u32), _dp, _dp, _dp], _int),
    "krpg_sample_device": ([_vp, _i64, _u64, _u64, _u64, _u32, _vp, _vp, _vp, _vp], _int),
    "krpg_sync": ([_vp], _int),
    "krpg_stream": ([_vp], _vp),
    "krpg_conditional": ([_vp, _i64, _u32, _dp, _dp, _dp], _int),
    "krpg_update_factor": ([_vp, _u32, _dp, _u64], _int),
    "krpg_update_entries": ([_vp, _u32, C.POINTER(_u64), C.POINTER(_u32), _dp, _u64], _int),
    "krpg_validate": ([_vp, C.c_double], _int),
    "krpg_gather_sa_device": ([_vp, _u64, _vp, _vp, _vp, _vp], _int),
    "krpg_last_build_ms": ([_vp, C.POINTER(C.c_float)], _int),
    "krpg_update_factor_device": ([_vp, _u32, _vp, _u64], _int),
    "krpg_rebuild": ([_vp, _u32], _int),
    "krpg_profile_enable": ([_vp, _int], _int),
    "krpg_profile_read": ([_vp, _dp, C.POINTER(_u64), _int], _int),
    "krpg_topology_node_rows": ([_u64, _u64, _u64, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64),
                                 C.POINTER(_u64)], _int),
    "krpg_host_eigh": ([_dp, _u32, _dp, _dp], _int),
    "krpg_is_checked_build": ([], _int),
    "krpg_set_option": ([_vp, _int, _i64], _int),
    "krpg_tree_device": ([_vp, _u32, C.POINTER(_vp), C.POINTER(_u64)], _int),
    "krpg_factor_device": ([_vp, _u32, C.POINTER(_vp)], _int),
    "krpg_build_partition": ([_vp, _u32, _u32, _u32, _vp], _int),
    "krpg_finish_partitions": ([_vp, _u32, _u32, _vp], _int),
    "krpg_partition_rows": ([_u64, _u32, _u32, _u32, C.POINTER(_u64), C.POINTER(_u64)], _int),
    "krpg_tensor_create": ([C.POINTER(_u64), _u32, C.POINTER(_u32), _dp, _u64, _int, C.POINTER(_vp)], _int),
    "krpg_tensor_create_device": ([C.POINTER(_u64), _u32, _vp, _vp, _u64, _int, C.POINTER(_vp)], _int),
    "krpg_tensor_destroy": ([_vp], _int),
    "krpg_tensor_info": ([_vp, C.POINTER(_u64), C.POINTER(C.c_double)], _int),
    "krpg_tensor_entries": ([_vp, C.POINTER(_u32), _dp], _int),
    "krpg_sts_solve": ([_vp, _vp, _u32, _u64, _u64, _dp], _int),
    "krpg_sts_last_stats": ([_vp, C.POINTER(_u64)], _int),
    "krpg_product_lev_sample": ([_vp, C.c_int64, _u64, _u64, _u64, C.POINTER(_u32), _dp, _dp, _dp], _int),
    "krpg_product_lev_sample_factors": ([C.POINTER(_dp), C.POINTER(_u64), _u32, _u32, C.c_int64, _u64, _u64, _int,
                                         C.POINTER(_u32), _dp, _dp, _dp], _int),
    "krpg_leverage_scores": ([_vp, _u32, _dp], _int),
    "krpg_segtree_create": ([_dp, _u64, _u32, _u64, _dp, _dp, _int, C.POINTER(_vp)], _int),
    "krpg_segtree_create_segments": ([_dp, _u64, _u32, C.POINTER(_u64), _u64, _dp, _dp, _int, C.POINTER(_vp)], _int),
    "krpg_segtree_leaf_offsets": ([_vp, C.POINTER(_u64)], _int),
    "krpg_segtree_node_rows": ([_vp, _u64, C.POINTER(_u64), C.POINTER(_u64)], _int),
    "krpg_segtree_destroy": ([_vp], _int),
    "krpg_segtree_clone": ([_vp, C.POINTER(_vp)], _int),
    "krpg_segtree_shape": ([_vp, C.POINTER(_u64), C.POINTER(_u64)], _int),
    "krpg_segtree_node_gram": ([_vp, _u64, _dp], _int),
    "krpg_segtree_sample": ([_vp, _dp, _u64, _u64, _u64, _u64, C.POINTER(_u64), _dp], _int),
    "krpg_segtree_sample_keyed": ([_vp, _dp, _u64, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64), _dp], _int),
    "krpg_segtree_probabilities": ([_vp, _dp, _dp], _int),
    "krpg_segtree_update_entry": ([_vp, _u64, _u32, C.c_double], _int),
}
OPT_GROUPED_DESCENT = 1

PROF_NAMES = ["tree_leaf", "tree_levels", "etree", "draws", "prob", "update", "other", "sts",
              "d_root", "d_level_cta", "d_level_warp", "d_regroup", "d_leaf", "d_misc", "sts_scatter", "spare3"]
OPT_PROFILE_DETAIL = 2
OPT_FUSED_DEEP = 3
OPT_ASYNC = 4
OPT_SLICES = 5
OPT_HOST_TRACE = 6
# kernel-variant / tuning options (include/krpg.h)
TUNING = {"eval_reg": 16, "pos0_tables": 17, "deep_threshold": 18, "deep_chunk": 19, "eval_split": 20,
          "deep_dmma_min": 21, "leaf_par": 22, "out_slices": 23, "sts_deterministic": 25, "eval_ml": 26}

_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    """Load libkrpg.so (raises if it was never built — no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: the CUDA extension is not built "
                "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
        l = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(l, name)
            f.argtypes = args
            f.restype = res
        _lib = l
    return _lib


def check(rc: int) -> None:
    if rc == KRPG_OK:
        return
    msg = lib().krpg_last_error().decode()
    if rc == KRPG_INVALID_ARGUMENT:
        raise KrpgInvalidArgument(msg)
    if rc == KRPG_CUDA_ERROR:
        raise KrpgCudaError(msg)
    raise KrpgError(msg)


def declared_symbols() -> list[str]:
    """Entry points declared in include/krpg.h (for the ABI export test)."""
    import re
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(krpg_[a-z_0-9]+)\s*\(", text)))
