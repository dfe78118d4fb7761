"""ctypes binding of libbsrprune.so (include/bsrprune.h) -- argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels.  There is no
CPU or PyTorch fallback: if the shared library is missing or was built for
another architecture the import / first call raises.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BSRP_LIB") or os.path.join(_PKG, "libbsrprune.so")  # BSRP_LIB: dev builds only

BSR_OK = 0
STATUS_NAMES = {0: "BSR_OK", 1: "BSR_ERR_INVALID_ARG", 2: "BSR_ERR_SHAPE", 3: "BSR_ERR_UNSUPPORTED",
                4: "BSR_ERR_ALIGNMENT", 5: "BSR_ERR_WORKSPACE", 6: "BSR_ERR_CUDA"}
DT_F32, DT_BF16 = 0, 1
PREC = {"fp32": 0, "tf32": 1, "bf16": 2}
ALGO = {"auto": 0, "runs": 1, "span": 2, "simt": 3, "dense": 4}

EXPORTED = ["bsr_num_blocks", "bsr_keep_count", "bsr_storage_bytes", "bsr_prune_workspace_bytes",
            "bsr_wgrad_workspace_bytes", "bsr_wgrad_algo_workspace_bytes", "bsr_prune", "bsr_prune_k", "bsr_validate", "bsr_prune_stochastic_workspace_bytes", "bsr_prune_stochastic", "bsr_block_sumsq", "bsr_decompress",
            "bsr_wgrad", "bsr_wgrad_algo", "bsr_wgrad_nk_workspace_bytes", "bsr_wgrad_nk", "bsr_wgrad_multicast", "bsr_wgrad_multicast_unicast_test", "bsr_set_pdl", "bsr_affine_wgrad_workspace_bytes", "bsr_affine_wgrad", "bsr_select_hist", "bsr_select_counts", "bsr_prune_threshold", "bsr_gselect_state_bytes", "bsr_gselect_init",
            "bsr_gselect_hist", "bsr_gselect_update", "bsr_gselect_counts", "bsr_gselect_take", "bsr_prune_gselect", "bsr_rows_keep_per_sample", "bsr_prune_rows_workspace_bytes", "bsr_prune_rows",
            "bsr_decompress_rows", "bsr_wgrad_rows_workspace_bytes", "bsr_wgrad_rows", "bsr_wgrad_rows_tc_workspace_bytes", "bsr_wgrad_rows_tc", "bsr_act_block_sumsq", "bsr_prune_presummed", "bsr_status_string", "bsr_last_error", "bsr_kernel_launches", "bsr_version"]


class BsrT(ctypes.Structure):
    """Mirror of bsr_t."""
    _fields_ = [("M", ctypes.c_int64), ("K", ctypes.c_int64), ("b", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("nnzb", ctypes.c_int64), ("rowptr", ctypes.c_void_p), ("colidx", ctypes.c_void_p),
                ("values", ctypes.c_void_p)]


class BsrError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {detail}")
        self.status = status
        self.detail = detail


_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                           "(there is no fallback implementation)")
    lib = ctypes.CDLL(path)
    i64, i32, vp, sz, dbl = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_double
    P = ctypes.POINTER(BsrT)
    sig = {
        "bsr_num_blocks": (i64, [i64, i64, i32]),
        "bsr_keep_count": (i64, [i64, dbl]),
        "bsr_storage_bytes": (sz, [i64, i32, i64, i32]),
        "bsr_prune_workspace_bytes": (sz, [i64, i64, i32]),
        "bsr_wgrad_workspace_bytes": (sz, [i64, i64, i32, i64, i32]),
        "bsr_wgrad_algo_workspace_bytes": (sz, [i64, i64, i32, i64, i32, i32]),
        "bsr_prune": (i32, [vp, i64, i64, i32, dbl, i32, P, vp, sz, vp]),
        "bsr_prune_k": (i32, [vp, i64, i64, i32, i64, i32, P, vp, sz, vp]),
        "bsr_validate": (i32, [P, vp, vp]),
        "bsr_prune_stochastic_workspace_bytes": (sz, [i64, i64, i32]),
        "bsr_prune_stochastic": (i32, [vp, i64, i64, i32, i64, i64, ctypes.c_double, ctypes.c_uint64, i32, P, vp, sz, vp]),
        "bsr_block_sumsq": (i32, [vp, i64, i64, i32, i32, vp, vp]),
        "bsr_decompress": (i32, [P, vp, vp]),
        "bsr_wgrad": (i32, [P, vp, i32, i64, vp, i32, i32, vp, sz, vp]),
        "bsr_wgrad_algo": (i32, [P, vp, i32, i64, vp, i32, i32, i32, vp, sz, vp]),
        "bsr_wgrad_nk_workspace_bytes": (sz, [i64, i64, i32, i64, i32, i32]),
        "bsr_wgrad_nk": (i32, [P, vp, i32, i64, vp, i32, i32, i32, vp, sz, vp]),
        "bsr_wgrad_multicast": (i32, [P, vp, i32, i64, vp, i32, i32, vp, sz, vp]),
        "bsr_wgrad_multicast_unicast_test": (i32, [P, vp, i32, i64, vp, i32, i32, vp, sz, vp]),
        "bsr_set_pdl": (ctypes.c_uint32, [ctypes.c_uint32]),
        "bsr_affine_wgrad_workspace_bytes": (sz, [i64, i64, i32]),
        "bsr_affine_wgrad": (i32, [P, vp, i32, vp, i32, vp, sz, vp]),
        "bsr_select_hist": (i32, [vp, i64, i64, i32, i32, i32, ctypes.c_uint32, vp, vp, sz, vp]),
        "bsr_select_counts": (i32, [i64, i64, i32, ctypes.c_uint32, i32, vp, vp, sz, vp]),
        "bsr_prune_threshold": (i32, [vp, i64, i64, i32, i32, ctypes.c_uint32, i32, i64, i64, P, vp, sz, vp]),
        "bsr_gselect_state_bytes": (sz, []),
        "bsr_gselect_init": (i32, [i64, vp, vp]),
        "bsr_gselect_hist": (i32, [vp, i64, i64, i32, i32, i32, vp, vp, vp, sz, vp]),
        "bsr_gselect_update": (i32, [vp, i32, vp, vp]),
        "bsr_gselect_counts": (i32, [i64, i64, i32, vp, vp, vp, sz, vp]),
        "bsr_gselect_take": (i32, [vp, i32, i32, vp, vp]),
        "bsr_prune_gselect": (i32, [vp, i64, i64, i32, i32, vp, i64, P, vp, sz, vp]),
        "bsr_rows_keep_per_sample": (i64, [i64, i64, i32, dbl]),
        "bsr_prune_rows_workspace_bytes": (sz, [i64, i64, i32]),
        "bsr_prune_rows": (i32, [vp, i64, i64, i32, i64, dbl, i32, vp, vp, vp, vp, sz, vp]),
        "bsr_decompress_rows": (i32, [vp, vp, vp, i64, i64, i32, i32, vp, vp]),
        "bsr_wgrad_rows_workspace_bytes": (sz, [i64, i64, i32, i64]),
        "bsr_wgrad_rows": (i32, [vp, vp, vp, i64, i64, i64, i32, i32, vp, i32, i64, vp, i32, vp, sz, vp]),
        "bsr_wgrad_rows_tc_workspace_bytes": (sz, [i64, i64, i32, i64, i32]),
        "bsr_wgrad_rows_tc": (i32, [vp, vp, vp, i64, i64, i64, i32, i32, vp, i32, i64, vp, i32, vp, sz, vp]),
        "bsr_act_block_sumsq": (i32, [vp, vp, i64, i64, i32, i32, i32, vp, sz, vp]),
        "bsr_prune_presummed": (i32, [vp, i64, i64, i32, i64, i32, P, vp, sz, vp]),
        "bsr_status_string": (ctypes.c_char_p, [i32]),
        "bsr_last_error": (ctypes.c_char_p, []),
        "bsr_kernel_launches": (ctypes.c_uint64, []),
        "bsr_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int):
    if status != BSR_OK:
        raise BsrError(status, load().bsr_last_error().decode())
