"""ctypes binding of libsbnet.so (include/sbnet.h).

The product path has no CPU fallback: if the extension is missing or no CUDA device is
visible, every op raises ``RuntimeError`` naming the problem.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import (BlockConvError, GeometryError, ShapeMismatchError, UnsupportedConfigError)

_HERE = os.path.dirname(os.path.abspath(__file__))
# SBN_LIB_PATH: load an alternative build (A/B experiments of compile-time variants, tools/)
LIB_PATH = os.environ.get("SBN_LIB_PATH") or os.path.join(_HERE, "libsbnet.so")

SBN_F32, SBN_F64, SBN_BF16 = 0, 1, 2
SBN_POOL_MAX, SBN_POOL_AVG = 0, 1
SBN_ALGO_AUTO, SBN_ALGO_SIMT, SBN_ALGO_TCGEN05 = 0, 1, 2

SBN_OK = 0
SBN_ERR_INVALID = -1
SBN_ERR_SHAPE = -2
SBN_ERR_UNSUPPORTED = -3
SBN_ERR_WORKSPACE = -4
SBN_ERR_CUDA = -5


class Geometry(C.Structure):
    _fields_ = [(name, C.c_int32) for name in (
        "n", "h", "w", "bh", "bw", "sy", "sx", "oy", "ox", "gy", "gx", "obh", "obw", "oh", "ow")]


class UnitParams(C.Structure):
    _fields_ = [(name, C.c_void_p) for name in (
        "w1", "b1", "w2", "b2", "w3", "b3", "bn1_scale", "bn1_shift", "bn2_scale",
        "bn2_shift", "bn3_scale", "bn3_shift", "tc_packed")] + [("tc_packed_bytes", C.c_size_t), ("tc_packed_variant", C.c_int)]


_P = C.c_void_p
_I = C.c_int
_G = C.POINTER(Geometry)

# name -> (restype, argtypes); mirrors include/sbnet.h
_PROTOS = {
    "sbn_version": (C.c_char_p, []),
    "sbn_last_error": (C.c_char_p, []),
    "sbn_device_sm_count": (_I, [_I]),
    "sbn_launch_count": (C.c_uint64, []),
    "sbn_reduce_mask_workspace": (C.c_size_t, [_G]),
    "sbn_reduce_mask": (_I, [_P, _G, _I, C.c_double, _P, _P, _P, C.c_size_t, _P]),
    "sbn_downsample_mask": (_I, [_P, _I, _I, _I, _I, _P, _P]),
    "sbn_gather": (_I, [_P, _I, _I, _G, _P, _P, _I, _I, _P, _P]),
    "sbn_in_bounds": (_I, [_G, _P, _P, _I, _P, _P]),
    "sbn_scatter": (_I, [_P, _I, _I, _G, _P, _P, _I, _I, _I, _P, _P]),
    "sbn_copy_block_regions": (_I, [_P, _P, _I, _I, _G, _P, _P, _I, _I, _P]),
    "sbn_copy_block_regions_t": (_I, [_P, _P, _I, _I, _G, _P, _P, _I, _I, _I, _P]),
    "sbn_gather_grad_workspace": (C.c_size_t, [_G]),
    "sbn_dense_conv_supported": (_I, [_I, _I, _I, _I, _I, _I, _I]),
    "sbn_dense_conv_packed_bytes": (C.c_size_t, [_I, _I, _I]),
    "sbn_dense_conv_pack": (_I, [_P, _I, _I, _I, _P, _P]),
    "sbn_dense_conv": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P]),
    "sbn_gather_grad": (_I, [_P, _I, _I, _G, _P, _P, _I, _P, _P, C.c_size_t, _P]),
    "sbn_sparse_conv": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _G, _P, _P, _P, _P, _P, _I, _P, _P,
                             C.c_size_t, _I, _P]),
    "sbn_sparse_conv_masked_sync_bytes": (C.c_size_t, [_G]),
    "sbn_sparse_conv_masked_workspace": (C.c_size_t, [_I, _I, _I, _I, _I, _I, _I, _G]),
    "sbn_sparse_conv_masked": (_I, [_P, _P, _I, _I, _I, _I, _I, _I, _I, _G, _P, _P, _P, _P, _P, C.c_size_t,
                                    _P, C.c_size_t, _I, _P]),
    "sbn_sparse_conv_packed_bytes": (C.c_size_t, [_I, _I, _I, _I, _I, _I, _I, _G]),
    "sbn_sparse_conv_pack": (_I, [_P, _I, _I, _I, _I, _I, _I, _I, _G, _P, _P]),
    "sbn_sparse_conv_algo": (_I, [_I, _I, _I, _I, _I, _I, _I, _G]),
    "sbn_residual_unit_workspace": (C.c_size_t, [_I, _I, _I, _G, _I, _I]),
    "sbn_residual_unit": (_I, [_P, _I, _I, _I, _G, _I, _I, C.POINTER(UnitParams), _P, _P, _I,
                               _P, _P, C.c_size_t, _I, _P]),
    "sbn_residual_unit_algo": (_I, [_I, _I, _I, _G, _I, _I]),
    "sbn_selftest_umma": (_I, [_P, _P, _I, _I, _I, _P, _P]),
    "sbn_debug_set_trace": (_I, [_P]),
    "sbn_debug_set_flags": (_I, [_I]),
    "sbn_debug_last_occupancy": (_I, [_I]),
    "sbn_sparse_residual_unit_sync_bytes": (C.c_size_t, [_G]),
    "sbn_sparse_residual_unit_workspace": (C.c_size_t, [_I, _I, _I, _G, _I, _I]),
    "sbn_sparse_residual_unit": (_I, [_P, _P, _I, _I, _I, _G, _I, _I, C.POINTER(UnitParams), _P, _P,
                                      C.c_size_t, _P, C.c_size_t, _I, _P]),
    "sbn_residual_unit_packed_bytes": (C.c_size_t, [_I, _I, _I, _G, _I, _I]),
    "sbn_residual_unit_packed_variant": (_I, [_I, _I, _I, _G, _I, _I]),
    "sbn_conv_grad_input": (_I, [_P, _I] + [_I] * 7 + [_P] + [_I] * 6 + [_P, _P]),
    "sbn_conv_grad_weight_workspace": (C.c_size_t, [_I] * 8),
    "sbn_conv_grad_weight": (_I, [_P, _P, _I] + [_I] * 13 + [_P, _P, _P, C.c_size_t, _P]),
    "sbn_residual_unit_pack": (_I, [C.POINTER(UnitParams), _I, _I, _I, _G, _I, _I, _P, _P]),
    "sbn_conv_forward": (_I, [_P, _I] + [_I] * 7 + [_P] + [_I] * 6 + [_P, _P, _P]),
    "sbn_bn_relu": (_I, [_P, _I, C.c_long, _I, _P, _P, _P, _P, _P, _P]),
    "sbn_bn_relu_grad": (_I, [_P, _P, _I, C.c_long, _I, _P, _P, _P, _P]),
    "sbn_add": (_I, [_P, _P, _I, C.c_long, _P, _P]),
    "sbn_bn_train_workspace": (C.c_size_t, [_I, C.c_long, _I]),
    "sbn_bn_train": (_I, [_P, _I, C.c_long, _I, _P, _P, C.c_double, _P, _P, _P, _P, C.c_size_t, _P]),
}

_lib = None
_lock = threading.Lock()


def exported_symbols():
    return sorted(_PROTOS)


def load(require_cuda: bool = True):
    """Load (once) and return the ctypes handle.  Raises RuntimeError when the
    extension is not built, or (require_cuda) when no CUDA device is present."""
    global _lib
    if require_cuda:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("sbnet: no CUDA device visible; this package has no CPU fallback")
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"sbnet: CUDA extension not built ({LIB_PATH} missing); run "
                        "`python -m paper_1801_02108_b200.build` or __graft_entry__.build()")
                lib = C.CDLL(LIB_PATH)
                for name, (res, args) in _PROTOS.items():
                    fn = getattr(lib, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = lib
    return _lib


def check(status: int, what: str) -> None:
    if status == SBN_OK:
        return
    msg = f"{what}: {load(False).sbn_last_error().decode(errors='replace')}"
    if status == SBN_ERR_SHAPE:
        raise ShapeMismatchError(msg)
    if status == SBN_ERR_INVALID:
        raise GeometryError(msg)
    if status == SBN_ERR_UNSUPPORTED:
        raise UnsupportedConfigError(msg)
    raise BlockConvError(f"[status {status}] {msg}")


def stream_handle(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def launch_count() -> int:
    return int(load(False).sbn_launch_count()) if _lib is not None or os.path.exists(LIB_PATH) else 0
