"""Activation container over torch tensors (reference `tensor.py:16-74`).

``Tensor4D`` keeps the reference's contract — logical dims are always (n, h, w, c)
whatever the storage layout — but holds a ``torch.Tensor`` (normally CUDA-resident) and
adds bfloat16.  numpy arrays and CPU tensors are accepted and stay where they are; the
ops move them to the current CUDA device on first use (a host->device copy, counted by
the e2e benchmark).
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from .errors import ShapeMismatchError

_FLOATS = (torch.float32, torch.float64, torch.bfloat16)


class Layout(Enum):
    CHANNELS_LAST = 0   # storage (n, h, w, c)
    CHANNELS_FIRST = 1  # storage (n, c, h, w)


def as_torch(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a
    return torch.from_numpy(np.ascontiguousarray(a))


def cuda(t: torch.Tensor, device=None) -> torch.Tensor:
    """Move to CUDA (non_blocking when the source is pinned) and make contiguous."""
    if not t.is_cuda:
        if not torch.cuda.is_available():
            raise RuntimeError("sbnet: no CUDA device visible; this package has no CPU fallback")
        t = t.to(device or torch.device("cuda", torch.cuda.current_device()),
                 non_blocking=t.is_pinned())
    return t.contiguous()


@dataclass(frozen=True)
class Tensor4D:
    """Contiguous 4-d activation tensor; immutable by convention."""

    data: torch.Tensor
    layout: Layout = Layout.CHANNELS_LAST

    def __post_init__(self):
        t = as_torch(self.data)
        if t.dim() != 4:
            raise ShapeMismatchError(f"Tensor4D requires 4 dims, got {t.dim()}")
        if t.dtype not in _FLOATS:
            raise ShapeMismatchError(f"Tensor4D dtype must be float32/float64/bfloat16, got {t.dtype}")
        object.__setattr__(self, "data", t.contiguous())

    @classmethod
    def from_nhwc(cls, arr, layout: Layout = Layout.CHANNELS_LAST) -> "Tensor4D":
        t = as_torch(arr)
        if layout is Layout.CHANNELS_FIRST:
            t = t.permute(0, 3, 1, 2)
        return cls(t.contiguous(), layout)

    @property
    def dims(self) -> tuple[int, int, int, int]:
        s = tuple(self.data.shape)
        if self.layout is Layout.CHANNELS_LAST:
            return s
        return (s[0], s[2], s[3], s[1])

    @property
    def dtype(self) -> torch.dtype:
        return self.data.dtype

    @property
    def device(self) -> torch.device:
        return self.data.device

    def nhwc(self) -> torch.Tensor:
        """(n, h, w, c)-ordered view (non-contiguous for CHANNELS_FIRST storage)."""
        if self.layout is Layout.CHANNELS_LAST:
            return self.data
        return self.data.permute(0, 2, 3, 1)

    def at(self, i: int, y: int, x: int, k: int) -> float:
        if self.layout is Layout.CHANNELS_LAST:
            return float(self.data[i, y, x, k])
        return float(self.data[i, k, y, x])

    def astype(self, dtype) -> "Tensor4D":
        return Tensor4D(self.data.to(dtype), self.layout)

    def cuda(self, device=None) -> "Tensor4D":
        return Tensor4D(cuda(self.data, device), self.layout)

    def numpy(self) -> np.ndarray:
        """Host copy in storage order (bf16 widened to float32)."""
        t = self.data.detach()
        if t.dtype == torch.bfloat16:
            t = t.float()
        return t.cpu().numpy()


def transpose_layout(x: Tensor4D) -> Tensor4D:
    """Switch between CHANNELS_LAST and CHANNELS_FIRST; logical contents unchanged."""
    if x.layout is Layout.CHANNELS_LAST:
        return Tensor4D(x.data.permute(0, 3, 1, 2).contiguous(), Layout.CHANNELS_FIRST)
    return Tensor4D(x.data.permute(0, 2, 3, 1).contiguous(), Layout.CHANNELS_LAST)


def dtype_code(dt: torch.dtype) -> int:
    from . import _lib
    if dt == torch.float32:
        return _lib.SBN_F32
    if dt == torch.float64:
        return _lib.SBN_F64
    if dt == torch.bfloat16:
        return _lib.SBN_BF16
    raise ShapeMismatchError(f"unsupported dtype {dt}")


def compute_dtype(dt: torch.dtype) -> torch.dtype:
    """Accumulate/BN dtype of the kernels: float64 for float64 data, float32 otherwise."""
    return torch.float64 if dt == torch.float64 else torch.float32
