"""ctypes mirror of include/ga.h and loader for the in-tree libga.so.

There is no fallback: if libga.so is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# GA_LIB overrides the library path (A/B timing of two builds); default: the in-tree build
LIB_PATH = os.environ.get("GA_LIB") or os.path.join(_PKG, "libga.so")

GA_EXCHANGE_ALLGATHER, GA_EXCHANGE_RING = 0, 1
GA_OK, GA_ERR_INVALID_ARG, GA_ERR_UNSUPPORTED, GA_ERR_CUDA, GA_ERR_COMM, GA_ERR_OOM, GA_ERR_MASK = 0, -1, -2, -3, -4, -5, -6
GA_COMM_ID_BYTES = 128
GA_F32, GA_BF16, GA_F16 = 0, 1, 2
GA_MASK_CSR, GA_MASK_WINDOW, GA_MASK_LONGNET, GA_MASK_BIGBIRD, GA_MASK_BLOCK_DILATED = 0, 1, 2, 3, 4
GA_KERNEL_AUTO, GA_KERNEL_EDGE, GA_KERNEL_TILED, GA_KERNEL_TC = 0, 1, 2, 3
GA_BB_WINDOW, GA_BB_GLOBAL, GA_BB_RANDOM = 1, 2, 4
GA_LONGNET_MULTISET, GA_LONGNET_HEAD_OFFSETS = 1, 2

STATUS_NAMES = {0: "GA_OK", -1: "GA_ERR_INVALID_ARG", -2: "GA_ERR_UNSUPPORTED", -3: "GA_ERR_CUDA",
                -4: "GA_ERR_COMM", -5: "GA_ERR_OOM", -6: "GA_ERR_MASK"}


class GaMask(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("parts", ctypes.c_int32), ("L", ctypes.c_int64),
        ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p), ("nnz", ctypes.c_int64),
        ("w", ctypes.c_int64), ("r", ctypes.c_int64),
        ("w0", ctypes.c_int64), ("alpha", ctypes.c_int64),
        ("seg", ctypes.c_int64),
        ("global_idx", ctypes.c_void_p), ("n_global", ctypes.c_int64),
        ("n_random", ctypes.c_int64), ("seed", ctypes.c_uint64),
    ]


class GaState(ctypes.Structure):
    _fields_ = [("m", ctypes.c_void_p), ("l", ctypes.c_void_p), ("o", ctypes.c_void_p)]


GA_STATE_WRITE, GA_STATE_ACCUMULATE = 0, 1


class GaOpts(ctypes.Structure):
    _fields_ = [
        ("q_begin", ctypes.c_int64), ("q_rows", ctypes.c_int64),
        ("kv_begin", ctypes.c_int64), ("kv_rows", ctypes.c_int64),
        ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
        ("edge_counter", ctypes.c_void_p), ("row_fingerprint", ctypes.c_void_p),
        ("kernel", ctypes.c_int32), ("heavy_threshold", ctypes.c_int32),
        ("state", GaState), ("state_mode", ctypes.c_int32), ("exchange", ctypes.c_int32),
        ("tensor_counter", ctypes.c_void_p),
    ]


# (name, restype, argtypes) for every symbol include/ga.h declares
_V, _I64, _I32, _U64, _SZ, _F = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_float
_PM, _PO = ctypes.POINTER(GaMask), ctypes.POINTER(GaOpts)
SIGNATURES = [
    ("ga_attention", ctypes.c_int, [_V, _V, _V, _PM, _V, _I64, _I32, _I32, ctypes.c_int, _V]),
    ("ga_attention_ex", ctypes.c_int, [_V, _V, _V, _PM, _V, _I64, _I32, _I32, ctypes.c_int, _PO, _V]),
    ("ga_attention_host", ctypes.c_int, [_V, _V, _V, _PM, _V, _I64, _I32, _I32, ctypes.c_int, _V]),
    ("ga_workspace_size", ctypes.c_int, [_PM, _I64, _I32, _I32, ctypes.c_int, _PO, ctypes.POINTER(_SZ)]),
    ("ga_mask_count", ctypes.c_int, [_PM, ctypes.POINTER(_I64)]),
    ("ga_query_alignment", ctypes.c_int, [_PM, _I32, ctypes.c_int, ctypes.POINTER(_I64)]),
    ("ga_mask_to_csr", ctypes.c_int, [_PM, _V, _V, _V]),
    ("ga_coo_to_csr", ctypes.c_int, [ctypes.c_int64, _V, _V, ctypes.c_int64, _V, _V, ctypes.POINTER(ctypes.c_int64), _V]),
    ("ga_mask_validate", ctypes.c_int, [_PM, _V, ctypes.POINTER(ctypes.c_int)]),
    ("ga_fill_inputs", ctypes.c_int, [_V, ctypes.c_int, _I64, _U64, _I32, _I64, _F, _V]),
    ("ga_state_finalize", ctypes.c_int, [ctypes.POINTER(GaState), _I64, _I32, _I32, ctypes.c_int, _V, _V]),
    ("ga_attention_backward", ctypes.c_int, [_V, _V, _V, _V, _V, ctypes.POINTER(GaMask), _V, _V, _V, _V, _I64, _I32,
                                             _I32, ctypes.c_int, _V]),
    ("ga_comm_get_unique_id", ctypes.c_int, [_V]),
    ("ga_comm_create", ctypes.c_int, [_I32, _I32, _V, _I32, ctypes.POINTER(_V)]),
    ("ga_comm_alloc", ctypes.c_int, [_V, _SZ, ctypes.POINTER(_V)]),
    ("ga_comm_free", ctypes.c_int, [_V, _V]),
    ("ga_comm_barrier", ctypes.c_int, [_V, _V]),
    ("ga_comm_host_allgather", ctypes.c_int, [_V, _V, _SZ, _V]),
    ("ga_comm_status", ctypes.c_int, [_V, ctypes.POINTER(ctypes.c_int)]),
    ("ga_attention_sharded", ctypes.c_int, [_V, _V, _V, _PM, _V, _I64, _I64, _I64, _I32, _I32, ctypes.c_int, _PO, _V,
                                            _V]),
    ("ga_comm_destroy", ctypes.c_int, [_V]),
    ("ga_last_error", ctypes.c_char_p, []),
    ("ga_launch_count", ctypes.c_ulonglong, []),
    ("ga_version", ctypes.c_char_p, []),
]

_lib = None


class GaError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def lib():
    """Load libga.so (raises if it is missing: there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libga.so not found at {LIB_PATH}; run `python -m paper_2502_01659_b200.build` "
                               "(the CUDA extension is required; there is no fallback path)")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != GA_OK:
        raise GaError(status, lib().ga_last_error().decode())
