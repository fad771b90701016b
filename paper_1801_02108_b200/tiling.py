"""Block geometry, masks and the reduce_mask operator (reference `tiling.py`).

Geometry (`compute_block_spec`) is host integer arithmetic; `reduce_mask` and
`downsample_mask` run on the GPU through libsbnet (`sbn_reduce_mask`,
`sbn_downsample_mask`).  A `BlockIndexList` lives on the device: (cap, 3) int32 rows
plus a device-resident count, so consumers never wait for the host; `count`,
`entries` and `len()` synchronise on first use only.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import CoverageError, GeometryError, ShapeMismatchError
from .ops import ConvParams, Padding, PoolMode
from .tensor import as_torch, cuda


# ----------------------------------------------------------------------------- masks

class BinaryMask:
    """Per-frame {0,1} computation mask (n, h, w) shared across channels
    (reference `tiling.py:16-44`).  Backed by a uint8 torch tensor."""

    __slots__ = ("data",)

    def __init__(self, data, validate: bool = True):
        t = as_torch(data)
        if t.dtype != torch.uint8:
            t = t.to(torch.uint8)
        if t.dim() != 3:
            raise ShapeMismatchError(f"mask must be 3-d (n, h, w), got {t.dim()}-d")
        t = t.contiguous()
        if validate and t.numel() and int(t.max()) > 1:
            raise ShapeMismatchError("mask values must be 0 or 1")
        self.data = t

    @property
    def dims(self) -> tuple[int, int, int]:
        return tuple(self.data.shape)

    @property
    def active_fraction(self) -> float:
        return float(self.data.float().mean()) if self.data.numel() else 0.0

    @classmethod
    def full(cls, n: int, h: int, w: int, device=None) -> "BinaryMask":
        return cls(torch.ones((n, h, w), dtype=torch.uint8, device=device), validate=False)

    @classmethod
    def empty(cls, n: int, h: int, w: int, device=None) -> "BinaryMask":
        return cls(torch.zeros((n, h, w), dtype=torch.uint8, device=device), validate=False)

    def cuda(self) -> "BinaryMask":
        return BinaryMask(cuda(self.data), validate=False)

    def numpy(self) -> np.ndarray:
        return self.data.cpu().numpy()


# ----------------------------------------------------------------------------- geometry

@dataclass(frozen=True)
class BlockSpec:
    """Tiling geometry of one conv layer (field meanings as reference `tiling.py:47-61`)."""

    block_size: tuple[int, int]
    overlap: tuple[int, int]
    in_stride: tuple[int, int]
    out_block_size: tuple[int, int]
    grid_origin: tuple[int, int]
    grid_count: tuple[int, int]
    kernel: tuple[int, int]
    conv_stride: tuple[int, int]
    padding: Padding
    input_size: tuple[int, int]
    out_size: tuple[int, int]

    def c_geometry(self, n: int) -> _lib.Geometry:
        g = _lib.Geometry()
        g.n, (g.h, g.w) = n, self.input_size
        g.bh, g.bw = self.block_size
        g.sy, g.sx = self.in_stride
        g.oy, g.ox = self.grid_origin
        g.gy, g.gx = self.grid_count
        g.obh, g.obw = self.out_block_size
        g.oh, g.ow = self.out_size
        return g


def compute_block_spec(input_dims, conv: ConvParams, block_size) -> BlockSpec:
    """Overlap-save geometry for one layer (reference `tiling.py:64-99`).

    Per axis: overlap = k - s; in_stride = block - overlap; out block = (block - k)//s + 1
    (also the output stride, so output windows abut exactly); origin = -pad; grid =
    ceil((padded extent - overlap) / in_stride), at least 1.
    """
    h, w = int(input_dims[1]), int(input_dims[2])
    block = (int(block_size[0]), int(block_size[1]))
    k, s, pad = tuple(conv.kernel), tuple(conv.stride), conv.pad
    if block[0] < k[0] or block[1] < k[1]:
        raise GeometryError(f"block size {block} smaller than kernel {k}")
    if (block[0] - k[0]) % s[0] or (block[1] - k[1]) % s[1]:
        raise GeometryError(
            f"block size {block} incompatible with kernel {k} stride {s}: stride must divide "
            "block_size - kernel for gap-free output tiling")
    ov = (k[0] - s[0], k[1] - s[1])
    ins = (block[0] - ov[0], block[1] - ov[1])
    ob = ((block[0] - k[0]) // s[0] + 1, (block[1] - k[1]) // s[1] + 1)
    ext = (h + 2 * pad[0], w + 2 * pad[1])
    grid = tuple(max(1, -(-(ext[a] - ov[a]) // ins[a])) for a in range(2))
    out = conv.out_size(h, w)
    assert ins[0] // s[0] == ob[0] and ins[1] // s[1] == ob[1]
    assert grid[0] * ob[0] >= out[0] and grid[1] * ob[1] >= out[1]
    return BlockSpec(block_size=block, overlap=ov, in_stride=ins, out_block_size=ob,
                     grid_origin=(-pad[0], -pad[1]), grid_count=grid, kernel=k, conv_stride=s,
                     padding=conv.padding, input_size=(h, w), out_size=out)


# ----------------------------------------------------------------------------- index lists

class BlockIndexList:
    """Active blocks as (frame, block_y, block_x) rows in ascending order
    (reference `tiling.py:102-117`).

    Device form: ``rows`` int32 (cap, 3) CUDA tensor whose first ``count`` rows are
    valid, and ``count_dev`` int32 (1,).  Also constructible from host entries.
    """

    def __init__(self, entries=None, *, rows: torch.Tensor | None = None,
                 count_dev: torch.Tensor | None = None):
        if rows is None:
            e = np.ascontiguousarray(np.asarray(entries if entries is not None else np.zeros((0, 3)),
                                                dtype=np.int64).reshape(-1, 3))
            self._host = e
            self._count = int(e.shape[0])
            self.rows = None
            self.count_dev = None
        else:
            self._host = None
            self._count = None
            self.rows = rows
            self.count_dev = count_dev

    def to_device(self, device=None) -> "BlockIndexList":
        if self.rows is None:
            dev = device or torch.device("cuda", torch.cuda.current_device())
            cap = max(1, self._count)
            rows = torch.zeros((cap, 3), dtype=torch.int32, device=dev)
            if self._count:
                rows[: self._count] = torch.from_numpy(self._host.astype(np.int32)).to(dev)
            self.rows = rows
            self.count_dev = torch.tensor([self._count], dtype=torch.int32, device=dev)
        return self

    @property
    def capacity(self) -> int:
        return int(self.rows.shape[0]) if self.rows is not None else self._count

    @property
    def count(self) -> int:
        if self._count is None:
            self._count = int(self.count_dev.item())
        return self._count

    def __len__(self) -> int:
        return self.count

    @property
    def entries(self) -> np.ndarray:
        if self._host is None:
            n = self.count
            self._host = self.rows[:n].to(torch.int64).cpu().numpy().reshape(-1, 3)
        return self._host


class _WorkspacePool(threading.local):
    """Per-thread, per-(device, stream) cached workspaces for reduce_mask.  The kernel
    leaves its workspace zeroed, so a buffer is zeroed once and reused forever."""

    def __init__(self):
        self.bufs = {}

    def get(self, nbytes: int, device) -> torch.Tensor:
        key = (str(device), torch.cuda.current_stream(device).cuda_stream)
        buf = self.bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.zeros(max(nbytes, 4096), dtype=torch.uint8, device=device)
            self.bufs[key] = buf
        return buf


_WS = _WorkspacePool()


def reduce_mask(mask: BinaryMask, spec: BlockSpec, pool: PoolMode = PoolMode.MAX,
                threshold: float | None = None) -> BlockIndexList:
    """Pool the mask over each block's input window and threshold into an ordered active
    block list (reference `tiling.py:138-160`).  One kernel launch; no host sync."""
    n, h, w = mask.dims
    if (h, w) != tuple(spec.input_size):
        raise ShapeMismatchError(f"mask spatial dims {(h, w)} != spec input size {spec.input_size}")
    area = spec.block_size[0] * spec.block_size[1]
    if threshold is None:
        threshold = 1.0 / area
    if not 0.0 < threshold <= 1.0:
        raise ValueError(f"threshold must be in (0, 1], got {threshold}")
    lib = _lib.load()
    m = cuda(mask.data)
    dev = m.device
    g = spec.c_geometry(n)
    cap = max(1, n * spec.grid_count[0] * spec.grid_count[1])
    rows = torch.empty((cap, 3), dtype=torch.int32, device=dev)
    count = torch.empty((1,), dtype=torch.int32, device=dev)
    nbytes = lib.sbn_reduce_mask_workspace(C.byref(g))
    ws = _WS.get(nbytes, dev)
    st = lib.sbn_reduce_mask(m.data_ptr(), C.byref(g),
                             _lib.SBN_POOL_MAX if pool is PoolMode.MAX else _lib.SBN_POOL_AVG,
                             float(threshold), rows.data_ptr(), count.data_ptr(), ws.data_ptr(),
                             ws.numel(), _lib.stream_handle(dev))
    _lib.check(st, "reduce_mask")
    return BlockIndexList(rows=rows, count_dev=count)


def downsample_mask(mask: BinaryMask, factor: int) -> BinaryMask:
    """Max-pool with window = stride = factor, ceil dims (reference `tiling.py:163-174`)."""
    if factor < 1:
        raise ValueError(f"factor must be >= 1, got {factor}")
    if factor == 1:
        return mask
    n, h, w = mask.dims
    lib = _lib.load()
    m = cuda(mask.data)
    out = torch.empty((n, -(-h // factor), -(-w // factor)), dtype=torch.uint8, device=m.device)
    _lib.check(lib.sbn_downsample_mask(m.data_ptr(), n, h, w, factor, out.data_ptr(),
                                       _lib.stream_handle(m.device)), "downsample_mask")
    return BinaryMask(out, validate=False)


# ----------------------------------------------------------------------------- coverage

@dataclass(frozen=True)
class CoverageReport:
    covered_pixels: int
    total_active_pixels: int
    total_block_area: int
    block_count: int

    @property
    def covered_fraction(self) -> float:
        return 1.0 if self.total_active_pixels == 0 else self.covered_pixels / self.total_active_pixels


def coverage_check(mask: BinaryMask, spec: BlockSpec, idx: BlockIndexList) -> CoverageReport:
    """Disjoint-write and coverage verification (reference `tiling.py:191-234`); a host
    diagnostic used by tests, vectorised over the write-count map."""
    m = mask.numpy()
    n, h, w = m.shape
    oh, ow = spec.out_size
    obh, obw = spec.out_block_size
    (kh, kw), (sh, sw) = spec.kernel, spec.conv_stride
    ph, pw = -spec.grid_origin[0], -spec.grid_origin[1]
    wc = np.zeros((n, oh, ow), np.int32)
    for i, by, bx in idx.entries:
        wc[i, by * obh:min(by * obh + obh, oh), bx * obw:min(bx * obw + obw, ow)] += 1
    if wc.size and wc.max() > 1:
        i, y, x = np.unravel_index(int(wc.argmax()), wc.shape)
        raise CoverageError(f"overlapping scatter writes at output pixel (batch {i}, y {y}, x {x})")
    # prefix sums of the written map: any write in the output window reached by a pixel
    pre = np.zeros((n, oh + 1, ow + 1), np.int64)
    pre[:, 1:, 1:] = (wc > 0).cumsum(1).cumsum(2)
    covered = 0
    for i, y, x in np.argwhere(m):
        lo_y = max(0, -(-(y + ph - kh + 1) // sh))
        hi_y = min(oh - 1, (y + ph) // sh)
        lo_x = max(0, -(-(x + pw - kw + 1) // sw))
        hi_x = min(ow - 1, (x + pw) // sw)
        if lo_y > hi_y or lo_x > hi_x:
            covered += 1
            continue
        s = (pre[i, hi_y + 1, hi_x + 1] - pre[i, lo_y, hi_x + 1] - pre[i, hi_y + 1, lo_x]
             + pre[i, lo_y, lo_x])
        if s == 0:
            raise CoverageError(f"active mask pixel (batch {i}, y {y}, x {x}) not covered by any active block")
        covered += 1
    return CoverageReport(covered, int(m.sum()), idx.count * spec.block_size[0] * spec.block_size[1],
                          idx.count)
