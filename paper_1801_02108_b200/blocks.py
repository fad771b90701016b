"""gather / scatter between dense NHWC tensors and block stacks (reference `blocks.py`).

Every op is one libsbnet launch on the current CUDA stream (`sbn_gather`,
`sbn_scatter`, `sbn_in_bounds`).  Results are bit-exact with the reference: copies
move raw bytes, the add mode does one add per element in the tensor dtype.
`sparse_gather` / `sparse_scatter(add=, transpose=)` are the north-star spellings of
the same operators (the uber/sbnet TF op names).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import GeometryError, ShapeMismatchError
from .tensor import Layout, Tensor4D, cuda, dtype_code
from .tiling import BlockIndexList, BlockSpec


@dataclass(frozen=True)
class GatheredBlocks:
    """Stacked active blocks plus the geometry they came from (reference `blocks.py:18-37`)."""

    tensor: Tensor4D          # logical (B, bh, bw, c)
    spec: BlockSpec
    indices: BlockIndexList

    def __post_init__(self):
        if self.tensor.dims[0] != self.indices.count:
            raise ShapeMismatchError(
                f"block tensor batch {self.tensor.dims[0]} != index count {self.indices.count}")

    @property
    def count(self) -> int:
        return self.indices.count

    def with_tensor(self, tensor: Tensor4D) -> "GatheredBlocks":
        return GatheredBlocks(tensor, self.spec, self.indices)


def _check_indices(idx: BlockIndexList, spec: BlockSpec, n: int) -> None:
    """Host-side range check for host-constructed lists (reference `blocks.py:40-48`);
    device lists from reduce_mask are in range by construction."""
    if idx.rows is not None or idx.count == 0:
        return
    e = idx.entries
    gy, gx = spec.grid_count
    if e[:, 0].min() < 0 or e[:, 0].max() >= n:
        raise GeometryError(f"block batch index out of range [0, {n})")
    if e[:, 1].min() < 0 or e[:, 1].max() >= gy or e[:, 2].min() < 0 or e[:, 2].max() >= gx:
        raise GeometryError(f"block index outside grid {spec.grid_count}")


def _check_source(x: Tensor4D, spec: BlockSpec) -> None:
    _, h, w, _ = x.dims
    if (h, w) != tuple(spec.input_size):
        raise ShapeMismatchError(f"tensor spatial dims {(h, w)} != spec input size {spec.input_size}")


def _nhwc_cuda(x: Tensor4D) -> torch.Tensor:
    return cuda(x.nhwc())


def _gather(x: Tensor4D, idx: BlockIndexList, spec: BlockSpec, transpose: bool) -> GatheredBlocks:
    _check_source(x, spec)
    n, h, w, c = x.dims
    _check_indices(idx, spec, n)
    lib = _lib.load()
    xt = _nhwc_cuda(x)
    idx.to_device(xt.device)
    B = idx.count
    bh, bw = spec.block_size
    shape = (B, c, bh, bw) if transpose else (B, bh, bw, c)
    out = torch.empty(shape, dtype=xt.dtype, device=xt.device)
    if B:
        g = spec.c_geometry(n)
        st = lib.sbn_gather(xt.data_ptr(), dtype_code(xt.dtype), c, C.byref(g), idx.rows.data_ptr(),
                            idx.count_dev.data_ptr(), B, int(transpose), out.data_ptr(),
                            _lib.stream_handle(xt.device))
        _lib.check(st, "gather")
    return GatheredBlocks(Tensor4D(out, Layout.CHANNELS_FIRST if transpose else Layout.CHANNELS_LAST),
                          spec, idx)


def gather(x: Tensor4D, idx: BlockIndexList, spec: BlockSpec) -> GatheredBlocks:
    """Copy each indexed input window into a (B, bh, bw, c) stack, zero-filling the
    out-of-image halo (reference `blocks.py:57-74`)."""
    return _gather(x, idx, spec, False)


def gather_transpose(x: Tensor4D, idx: BlockIndexList, spec: BlockSpec) -> GatheredBlocks:
    """Fused gather + NHWC->(B, c, bh, bw) transpose (reference `blocks.py:77-94`)."""
    return _gather(x, idx, spec, True)


def in_bounds_map(idx: BlockIndexList, spec: BlockSpec, n: int | None = None) -> torch.Tensor:
    """(B, bh, bw) bool map of window positions that read real pixels (reference
    `blocks.py:97-112`)."""
    lib = _lib.load()
    idx.to_device()
    B = idx.count
    out = torch.zeros((B,) + tuple(spec.block_size), dtype=torch.uint8, device=idx.rows.device)
    if B:
        g = spec.c_geometry(n if n is not None else 1)
        _lib.check(lib.sbn_in_bounds(C.byref(g), idx.rows.data_ptr(), idx.count_dev.data_ptr(), B,
                                     out.data_ptr(), _lib.stream_handle(out.device)), "in_bounds_map")
    return out.bool()


def _check_scatter(blocks: GatheredBlocks, out_spec: BlockSpec) -> None:
    if blocks.spec != out_spec:
        raise GeometryError("block source geometry does not match scatter geometry")
    d = blocks.tensor.dims
    if (d[1], d[2]) != tuple(out_spec.out_block_size):
        raise ShapeMismatchError(
            f"block spatial dims {(d[1], d[2])} != output block size {out_spec.out_block_size}")


def _scatter(blocks: GatheredBlocks, out_spec: BlockSpec, dst: Tensor4D, add: bool,
             inplace: bool = False) -> Tensor4D:
    _check_scatter(blocks, out_spec)
    n, oh, ow, c = dst.dims
    if (oh, ow) != tuple(out_spec.out_size):
        raise ShapeMismatchError(f"destination spatial dims {(oh, ow)} != conv output {out_spec.out_size}")
    if c != blocks.tensor.dims[3]:
        raise ShapeMismatchError(f"destination channels {c} != block channels {blocks.tensor.dims[3]}")
    lib = _lib.load()
    d = _nhwc_cuda(dst)
    out = d if (inplace and d.data_ptr() == dst.nhwc().data_ptr()) else d.clone()
    blk = cuda(blocks.tensor.data)
    if blk.dtype != out.dtype:
        raise ShapeMismatchError(f"block dtype {blk.dtype} != destination dtype {out.dtype}")
    idx = blocks.indices.to_device(out.device)
    B = blocks.count
    if B:
        transpose = blocks.tensor.layout is Layout.CHANNELS_FIRST
        g = out_spec.c_geometry(n)
        st = lib.sbn_scatter(blk.data_ptr(), dtype_code(out.dtype), c, C.byref(g), idx.rows.data_ptr(),
                             idx.count_dev.data_ptr(), B, int(add), int(transpose), out.data_ptr(),
                             _lib.stream_handle(out.device))
        _lib.check(st, "scatter")
    return Tensor4D.from_nhwc(out, dst.layout)


def scatter(blocks: GatheredBlocks, out_spec: BlockSpec, dst: Tensor4D) -> Tensor4D:
    """Write each block into its disjoint output window; other pixels keep dst's values.
    Returns a new tensor (reference `blocks.py:145-147`)."""
    if blocks.tensor.layout is Layout.CHANNELS_FIRST:
        raise GeometryError("scatter expects ChannelsLast blocks; use scatter_transpose")
    return _scatter(blocks, out_spec, dst, add=False)


def scatter_add(blocks: GatheredBlocks, out_spec: BlockSpec, dst: Tensor4D) -> Tensor4D:
    """As scatter, accumulating into dst (reference `blocks.py:150-152`)."""
    if blocks.tensor.layout is Layout.CHANNELS_FIRST:
        raise GeometryError("scatter_add expects ChannelsLast blocks")
    return _scatter(blocks, out_spec, dst, add=True)


def scatter_transpose(blocks: GatheredBlocks, out_spec: BlockSpec, dst: Tensor4D) -> Tensor4D:
    """Scatter ChannelsFirst (B, c, obh, obw) blocks into an NHWC destination in one pass
    (reference `blocks.py:155-159`)."""
    if blocks.tensor.layout is not Layout.CHANNELS_FIRST:
        raise GeometryError("scatter_transpose expects ChannelsFirst blocks")
    return _scatter(blocks, out_spec, dst, add=False)


# ---- training path (adjoints) ---------------------------------------------------------

def gather_grad(g_blocks: GatheredBlocks, spec: BlockSpec, dst_dims, dtype=None) -> Tensor4D:
    """Adjoint of gather: block gradients summed over their (overlapping) input windows
    (reference `blocks.py:162-188`).  One pixel-centric launch (`sbn_gather_grad`): every
    element is the covering blocks' values added in index order from zero — the
    reference's canonical order, so f32/f64 results are bit-exact, with no atomics."""
    if g_blocks.spec != spec:
        raise GeometryError("gradient block geometry does not match spec")
    n, h, w, c = (int(v) for v in dst_dims)
    if (h, w) != tuple(spec.input_size):
        raise ShapeMismatchError(f"destination spatial dims {(h, w)} != spec input size {spec.input_size}")
    bd = g_blocks.tensor.dims
    if (bd[1], bd[2]) != tuple(spec.block_size):
        raise ShapeMismatchError(f"gradient block dims {(bd[1], bd[2])} != block size {spec.block_size}")
    if g_blocks.tensor.layout is Layout.CHANNELS_FIRST:
        raise GeometryError("gather_grad expects ChannelsLast block gradients")
    lib = _lib.load()
    blk = cuda(g_blocks.tensor.data)
    if dtype is not None:
        blk = blk.to(dtype if isinstance(dtype, torch.dtype) else torch.from_numpy(np.zeros(1, dtype)).dtype)
    out = torch.empty((n, h, w, c), dtype=blk.dtype, device=blk.device)
    idx = g_blocks.indices.to_device(blk.device)
    g = spec.c_geometry(n)
    ws = torch.empty(max(1, int(lib.sbn_gather_grad_workspace(C.byref(g)))), dtype=torch.uint8, device=blk.device)
    B = g_blocks.count
    st = lib.sbn_gather_grad(blk.data_ptr() if B else None, dtype_code(blk.dtype), c, C.byref(g),
                             idx.rows.data_ptr(), idx.count_dev.data_ptr(), B, out.data_ptr(), ws.data_ptr(),
                             ws.numel(), _lib.stream_handle(blk.device))
    _lib.check(st, "gather_grad")
    return Tensor4D(out)


def _out_grid_spec_geometry(spec: BlockSpec, n: int) -> _lib.Geometry:
    """Geometry of a gather over the disjoint OUTPUT grid: image = out size, block =
    stride = out block, origin 0 (windows never overlap; the tail is zero-filled)."""
    g = spec.c_geometry(n)
    g.h, g.w = spec.out_size
    g.bh, g.bw = spec.out_block_size
    g.sy, g.sx = spec.out_block_size
    g.oy = g.ox = 0
    return g


def scatter_grad(g_out: Tensor4D, idx: BlockIndexList, out_spec: BlockSpec) -> GatheredBlocks:
    """Adjoint of scatter: the upstream gradient over each block's disjoint, clipped write
    window (reference `blocks.py:191-204`) — `sbn_gather` over the output grid."""
    n, oh, ow, c = g_out.dims
    if (oh, ow) != tuple(out_spec.out_size):
        raise ShapeMismatchError(f"gradient spatial dims {(oh, ow)} != conv output {out_spec.out_size}")
    _check_indices(idx, out_spec, n)
    lib = _lib.load()
    t = _nhwc_cuda(g_out)
    idx.to_device(t.device)
    B = idx.count
    obh, obw = out_spec.out_block_size
    out = torch.empty((B, obh, obw, c), dtype=t.dtype, device=t.device)
    if B:
        g = _out_grid_spec_geometry(out_spec, n)
        st = lib.sbn_gather(t.data_ptr(), dtype_code(t.dtype), c, C.byref(g), idx.rows.data_ptr(),
                            idx.count_dev.data_ptr(), B, 0, out.data_ptr(), _lib.stream_handle(t.device))
        _lib.check(st, "scatter_grad")
    return GatheredBlocks(Tensor4D(out), out_spec, idx)


# ---- north-star (uber/sbnet op) spellings -------------------------------------------

def sparse_gather(x: Tensor4D, idx: BlockIndexList, spec: BlockSpec,
                  transpose: bool = False) -> GatheredBlocks:
    return _gather(x, idx, spec, transpose)


def sparse_scatter(blocks: GatheredBlocks, out_spec: BlockSpec, dst: Tensor4D, add: bool = False,
                   transpose: bool | None = None, inplace: bool = False) -> Tensor4D:
    if transpose is not None and transpose != (blocks.tensor.layout is Layout.CHANNELS_FIRST):
        raise GeometryError("transpose flag does not match the block stack layout")
    if add and blocks.tensor.layout is Layout.CHANNELS_FIRST:
        raise GeometryError("add mode expects ChannelsLast blocks")
    return _scatter(blocks, out_spec, dst, add=add, inplace=inplace)
