"""ctypes binding of include/tilefabric_b200/tf_abi.h (the C-ABI boundary).

This is exactly the stub a Python host of the reference would add (see
INTEGRATION.md).  The shared library is built in-tree by
``paper_2511_02168_b200/csrc/Makefile``; there is no fallback: if it is
missing or the device is not sm_100 every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TFB_LIB") or os.path.join(HERE, "libtilefabric_b200.so")

# tf_status -> the reference's exception classes (common.hpp:39-94).


class Error(RuntimeError):
    """tilefabric::Error"""


class ConfigError(Error):
    pass


class BoundsError(Error):
    pass


class ShapeError(Error):
    pass


class DeadlockError(Error):
    pass


class WorldError(Error):
    pass


class EmptyAttentionError(Error):
    pass


class NumericError(Error):
    pass


class CudaError(Error):
    pass


_STATUS = {1: ConfigError, 2: BoundsError, 3: ShapeError, 4: DeadlockError, 5: WorldError,
           6: EmptyAttentionError, 7: NumericError, 8: CudaError}

TF_AG_BASELINE, TF_AG_PULL, TF_AG_PUSH = 0, 1, 2
TF_FD_BSP, TF_FD_INDEPENDENT_AG, TF_FD_FINE_WAITS, TF_FD_FUSED, TF_FD_FUSED_BY_ARRIVAL = 0, 1, 2, 3, 4
TF_FD_FUSED_OWNER = 5
TF_F32, TF_BF16 = 0, 1
TF_PAGED_NHD, TF_PAGED_HND = 0, 1
TF_SHARD_K, TF_SHARD_M = 0, 1
TF_OK, TF_ERR_CONFIG, TF_ERR_BOUNDS, TF_ERR_SHAPE, TF_ERR_DEADLOCK, TF_ERR_WORLD = 0, 1, 2, 3, 4, 5
TF_ERR_EMPTY_ATTENTION, TF_ERR_NUMERIC, TF_ERR_CUDA = 6, 7, 8
IPC_HANDLE_BYTES = 64


class AgShape(C.Structure):
    _fields_ = [("m", C.c_size_t), ("n", C.c_size_t), ("k", C.c_size_t),
                ("bm", C.c_size_t), ("bn", C.c_size_t), ("bk", C.c_size_t), ("dtype", C.c_int),
                ("shard", C.c_int)]  # tf_ag_shard: 0 K (the reference), 1 M


class FdShape(C.Structure):
    _fields_ = [("batch", C.c_int), ("q_heads", C.c_int), ("kv_heads", C.c_int),
                ("head_dim", C.c_int), ("kv_len", C.c_size_t), ("scale", C.c_float),
                ("kv_dtype", C.c_int), ("out_dtype", C.c_int)]


class Taxes(C.Structure):
    """tf_taxes: the Three Taxes measured on the device (taxmeter.hpp:45-63)."""
    _fields_ = [("launches", C.c_uint64), ("signal_waits", C.c_uint64), ("wait_idle_ns", C.c_uint64),
                ("barrier_waits", C.c_uint64), ("bulk_sync_ns", C.c_uint64), ("staged_bytes", C.c_uint64)]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


class FdPaged(C.Structure):
    """tf_fd_paged: page pools NHD [num_pages][page_size][kv_heads][d] (layout 0) or
    HND [num_pages][kv_heads][page_size][d] (layout 1) + block tables."""
    _fields_ = [("page_size", C.c_int), ("pages_per_seq", C.c_int), ("num_pages", C.c_int), ("layout", C.c_int)]


# name -> (restype, argtypes); every symbol tf_abi.h declares.
_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)
SIGNATURES = {
    "tf_last_error": (C.c_char_p, []),
    "tf_abi_version": (C.c_int, []),
    "tf_world_create": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.c_size_t, C.c_double, _PP]),
    "tf_world_create_ipc": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_size_t, C.c_double, _PP]),
    "tf_world_ipc_export": (C.c_int, [_P, _P]),
    "tf_world_ipc_import": (C.c_int, [_P, _P]),
    "tf_world_destroy": (C.c_int, [_P]),
    "tf_world_size": (C.c_int, [_P]),
    "tf_world_local_ranks": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "tf_world_stream": (_P, [_P, C.c_int]),
    "tf_world_reset_heap": (C.c_int, [_P]),
    "tf_heap_alloc": (C.c_int, [_P, C.c_char_p, C.c_size_t, _PP]),
    "tf_board_alloc": (C.c_int, [_P, C.c_char_p, C.c_int, C.c_int, _PP]),
    "tf_signal": (C.c_int, [_P, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int]),
    "tf_wait_signal": (C.c_int, [_P, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_uint64]),
    "tf_read_signal": (C.c_int, [_P, C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint64)]),
    "tf_signal_soak": (C.c_int, [_P, C.c_uint64, C.c_int, C.POINTER(C.c_uint64)]),
    "tf_world_barrier": (C.c_int, [_P, C.c_int]),
    "tf_ag_gemm": (C.c_int, [_P, C.c_int, C.POINTER(AgShape), _PP, _PP, _PP, _PP, _PP]),
    "tf_ag_gemm_async": (C.c_int, [_P, C.c_int, C.POINTER(AgShape), _PP, _PP, _PP, _PP, _PP]),
    "tf_ag_gemm_host": (C.c_int, [_P, C.c_int, C.POINTER(AgShape), _PP, _PP, _PP, _PP]),
    "tf_world_set_events": (C.c_int, [_P, C.c_int]),
    "tf_ag_events": (C.c_int, [_P, C.c_int, C.POINTER(C.c_uint64), C.c_size_t, C.POINTER(C.c_size_t)]),
    "tf_fd_events": (C.c_int, [_P, C.c_int, C.POINTER(C.c_uint64), C.c_size_t, C.POINTER(C.c_size_t)]),
    "tf_ag_gemm_host_async": (C.c_int, [_P, C.c_int, C.POINTER(AgShape), _PP, _PP, _PP, _PP]),
    "tf_ag_gathered": (C.c_int, [_P, C.c_int, _P, C.c_size_t]),
    "tf_ag_flag_counts": (C.c_int, [_P, C.c_int, C.POINTER(C.c_uint64), C.c_size_t,
                                    C.POINTER(C.c_size_t)]),
    "tf_flash_decode": (C.c_int, [_P, C.c_int, C.POINTER(FdShape), _PP, _PP, _PP, _PP, _PP, _PP]),
    "tf_flash_decode_async": (C.c_int, [_P, C.c_int, C.POINTER(FdShape), _PP, _PP, _PP, _PP,
                                        _PP, _PP]),
    "tf_flash_decode_paged": (C.c_int, [_P, C.c_int, C.POINTER(FdShape), C.POINTER(FdPaged), _PP, _PP, _PP, _PP,
                                        _PP, _PP, _PP]),
    "tf_flash_decode_paged_async": (C.c_int, [_P, C.c_int, C.POINTER(FdShape), C.POINTER(FdPaged), _PP, _PP, _PP,
                                              _PP, _PP, _PP, _PP]),
    "tf_fd_partial_async": (C.c_int, [_P, C.POINTER(FdShape), _PP, _PP, _PP, _PP, _PP]),
    "tf_fd_combine_async": (C.c_int, [_P, C.POINTER(FdShape), _PP, _PP, _PP]),
    "tf_fd_flag_counts": (C.c_int, [_P, C.c_int, C.POINTER(C.c_uint64), C.c_size_t,
                                    C.POINTER(C.c_size_t)]),
    "tf_memcpy": (C.c_int, [_P, _P, _P, C.c_size_t]),
    "tf_memcpy_async": (C.c_int, [_P, _P, _P, C.c_size_t, _P]),
    "tf_device_alloc": (C.c_int, [_P, C.c_int, C.c_size_t, _PP]),
    "tf_device_free": (C.c_int, [_P, C.c_int, _P]),
    "tf_uniform_reals": (C.c_int, [C.c_uint64, C.c_size_t, C.POINTER(C.c_float)]),
    "tf_world_sync": (C.c_int, [_P]),
    "tf_launch_count": (C.c_uint64, [_P]),
    "tf_tax_report": (C.c_int, [_P, C.c_int, C.POINTER(Taxes)]),
    "tf_tax_reset": (C.c_int, [_P]),
    "tf_world_set_skew": (C.c_int, [_P, C.c_int, C.c_uint64]),
    "tf_device_count": (C.c_int, []),
}

_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-j8", "-C", os.path.join(HERE, "csrc")], check=True)


def lib() -> C.CDLL:
    """Load the in-tree library (building it if this is a source checkout)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status:
        msg = lib().tf_last_error().decode(errors="replace")
        raise _STATUS.get(status, Error)(msg)


def ptr_array(ptrs) -> C.Array:
    arr = (C.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p if p else None
    return arr
