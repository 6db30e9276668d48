"""ctypes binding of the C-ABI in include/sparsedrop_b200.h.

This is the only place Python touches libsparsedrop_b200.so. Every compute entry
point runs the sm_100a kernels; there is no CPU fallback: if the library is
missing or no B200 is visible, calls raise instead of computing elsewhere.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "lib" / "libsparsedrop_b200.so"
HEADER_PATH = _PKG.parent / "include" / "sparsedrop_b200.h"

SD_OK, SD_EINVAL, SD_ERANGE, SD_ERUNTIME = 0, 1, 2, 3
SD_DTYPE_F32, SD_DTYPE_BF16 = 0, 1


class SdBlockMask(ctypes.Structure):
    """Mirror of ``sd_block_mask`` (include/sparsedrop_b200.h)."""

    _fields_ = [
        ("block_rows", ctypes.c_int32),
        ("block_cols", ctypes.c_int32),
        ("m_blk", ctypes.c_int32),
        ("k_blk", ctypes.c_int32),
        ("row_block_offset", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("words", ctypes.c_void_p),
        ("keep_count", ctypes.c_void_p),
        ("row_cnt", ctypes.c_void_p),
        ("row_idx", ctypes.c_void_p),
        ("col_cnt", ctypes.c_void_p),
        ("col_idx", ctypes.c_void_p),
        ("row_order", ctypes.c_void_p),
        ("col_order", ctypes.c_void_p),
        ("ticket", ctypes.c_void_p),
    ]


_P = ctypes.c_void_p
_I = ctypes.c_int32
_MASKP = ctypes.POINTER(SdBlockMask)

# name -> (restype, argtypes)
PROTOTYPES = {
    "sd_abi_version": (ctypes.c_int, []),
    "sd_last_error": (ctypes.c_char_p, []),
    "sd_device_count": (ctypes.c_int, []),
    "sd_launch_count": (ctypes.c_uint64, []),
    "sd_set_tuning": (ctypes.c_int, [_I]),
    "sd_device_alloc": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_size_t]),
    "sd_device_free": (ctypes.c_int, [_P]),
    "sd_memcpy": (ctypes.c_int, [_P, _P, ctypes.c_size_t, _I, _P]),
    "sd_memset": (ctypes.c_int, [_P, _I, ctypes.c_size_t, _P]),
    "sd_stream_synchronize": (ctypes.c_int, [_P]),
    "sd_mask_workspace_bytes": (ctypes.c_size_t, [_I, _I]),
    "sd_mask_bind": (ctypes.c_int, [_MASKP, _P, _I, _I, _I, _I, _I]),
    "sd_mask_sample": (ctypes.c_int, [_MASKP, ctypes.c_uint64, ctypes.c_double, _I, _I, _P]),
    "sd_mask_compact": (ctypes.c_int, [_MASKP, _P]),
    "sd_mask_transpose": (ctypes.c_int, [_MASKP, _MASKP, _P]),
    "sd_mask_retile": (ctypes.c_int, [_MASKP, _I, _I, _MASKP, _P]),
    "sd_dense_gemm": (ctypes.c_int, [_P, _P, _P, _I, _I, _I, _I, _P]),
    "sd_dense_gemm_nt": (ctypes.c_int, [_P, _P, _P, _I, _I, _I, _I, _P]),
    "sd_dense_gemm_tn": (ctypes.c_int, [_P, _P, _P, _I, _I, _I, _I, _P]),
    "sd_dsd_matmul": (ctypes.c_int, [_P, _MASKP, _P, ctypes.c_float, _P, _I, _I, _I, _I, _P, _P]),
    "sd_sdd_matmul": (ctypes.c_int, [_P, _P, _MASKP, ctypes.c_float, _P, _I, _I, _I, _I, _P, _P]),
    "sd_linear_forward": (ctypes.c_int, [_P, _MASKP, _P, ctypes.c_float, _P, _I, _I, _I, _I, _P]),
    "sd_linear_backward_dx": (ctypes.c_int, [_P, _P, _MASKP, ctypes.c_float, _P, _I, _I, _I, _I, _P]),
    "sd_linear_backward_dw": (ctypes.c_int, [_P, _MASKP, _P, ctypes.c_float, _P, _I, _I, _I, _I, _P]),
    "sd_layer_plan_create": (ctypes.c_int, [ctypes.POINTER(_P), _P, _P, _P, _P, _I, _P, _I, _P, _I, _I, _I, _I,
                                            ctypes.c_double, _MASKP]),
    "sd_layer_plan_forward": (ctypes.c_int, [_P, ctypes.c_uint64, _P]),
    "sd_layer_plan_backward": (ctypes.c_int, [_P, _P]),
    "sd_layer_plan_backward_dw": (ctypes.c_int, [_P, _P]),
    "sd_layer_plan_backward_dx": (ctypes.c_int, [_P, _P]),
    "sd_layer_plan_backward_dw_part": (ctypes.c_int, [_P, _I, _I, _P]),
    "sd_dev_mask_counter_waits": (ctypes.c_uint64, []),
    "sd_dev_dsd_pairs": (ctypes.c_int, [_P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _P, _I, ctypes.c_float, _P]),
    "sd_layer_plan_dense_forward": (ctypes.c_int, [_P, _P]),
    "sd_layer_plan_dense_backward": (ctypes.c_int, [_P, _P]),
    "sd_layer_plan_set_options": (ctypes.c_int, [_P, _I]),
    "sd_layer_plan_graph_step": (ctypes.c_int, [_P, ctypes.c_uint64, _I, _P]),
    "sd_layer_plan_destroy": (ctypes.c_int, [_P]),
    "sd_comm_unique_id": (ctypes.c_int, [_P]),
    "sd_comm_init": (ctypes.c_int, [ctypes.POINTER(_P), _I, _I, _P]),
    "sd_comm_destroy": (ctypes.c_int, [_P]),
    "sd_comm_nccl_version": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int32)]),
    "sd_comm_allreduce_sum": (ctypes.c_int, [_P, _P, ctypes.c_size_t, _I, _P]),
    "sd_layer_plan_backward_allreduce": (ctypes.c_int, [_P, _P, _I, _P, _P]),
    "sd_gelu_forward": (ctypes.c_int, [_P, _P, ctypes.c_int64, _P]),
    "sd_gelu_backward": (ctypes.c_int, [_P, _P, _P, ctypes.c_int64, _P]),
    "sd_gemm_ex": (ctypes.c_int, [_P, _I, _P, _I, _P, _I, _I, _I, _I, ctypes.c_float, _P]),
    "sd_dropout_apply": (ctypes.c_int, [_P, _P, _I, _I, ctypes.c_uint64, ctypes.c_double, ctypes.c_float, _MASKP, _P]),
    "sd_flops_dense": (ctypes.c_uint64, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]),
    "sd_flops_effective": (
        ctypes.c_uint64,
        [ctypes.c_int64, ctypes.c_int64, _I, _I, _I, ctypes.c_int64, _I],
    ),
}

_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


def load() -> ctypes.CDLL:
    """Load libsparsedrop_b200.so (built by __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("SPARSEDROP_B200_LIB", LIB_PATH))
    if not path.exists():
        raise NativeLibraryMissing(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)"
        )
    lib = ctypes.CDLL(str(path))
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    """Raise the Python analogue of the reference's exception for a status code:
    std::invalid_argument -> ValueError, std::out_of_range -> IndexError,
    std::runtime_error -> RuntimeError."""
    if status == SD_OK:
        return
    msg = load().sd_last_error().decode(errors="replace")
    if status == SD_EINVAL:
        raise ValueError(msg)
    if status == SD_ERANGE:
        raise IndexError(msg)
    raise RuntimeError(msg)
