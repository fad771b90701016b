"""Composite sparse layers (reference `layers.py`): sparse_conv2d, the sparse residual
unit, stages and the backbone.

Hot path per layer = two libsbnet launches on the current stream, no host sync:
``sbn_reduce_mask`` (mask -> ordered device index list) and one fused kernel
(``sbn_sparse_conv`` / ``sbn_residual_unit``) that gathers, computes and scatters
without materialising the block stack.  Dense comparators (`conv2d_direct`,
`dense_residual_unit`) and stage projections use cuDNN.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.nn.functional as F

from . import _lib
from .blocks import GatheredBlocks, gather, gather_grad, in_bounds_map, scatter_grad
from .errors import EmptyBlockListError, GeometryError, ShapeMismatchError, UnsupportedConfigError
from .ops import (BnMode, BnParams, ConvParams, FilterBank, Padding, PoolMode, add_nhwc, bn_inference, bn_relu_grad_nhwc,
                  bn_relu_nhwc, conv_forward_nhwc, conv_grads_nhwc, dense_conv_nhwc, exact_fp32, projection_conv)
from .tensor import Layout, Tensor4D, cuda, dtype_code
from .tiling import (BinaryMask, BlockIndexList, BlockSpec, compute_block_spec, downsample_mask,
                     reduce_mask)

_ALGOS = {"auto": _lib.SBN_ALGO_AUTO, "simt": _lib.SBN_ALGO_SIMT, "tcgen05": _lib.SBN_ALGO_TCGEN05}


def _algo(a) -> int:
    if isinstance(a, int):
        return a
    try:
        return _ALGOS[a]
    except KeyError:
        raise ValueError(f"unknown algo {a!r}; expected one of {sorted(_ALGOS)}") from None


def _check_mask(x: Tensor4D, mask: BinaryMask) -> None:
    n, h, w, _ = x.dims
    if mask.dims != (n, h, w):
        raise ShapeMismatchError(f"mask dims {mask.dims} != tensor (n, h, w) {(n, h, w)}")


class _Scratch(threading.local):
    def __init__(self):
        self.bufs = {}

    def get(self, nbytes: int, device, kind: str = "unit") -> torch.Tensor:
        """Zero-initialised, cached per (device, stream, kind); grows by reallocating (zeroed).
        Kinds never share a buffer.  "*sync" kinds hold only self-resetting words (always
        zero between calls), so reuse across geometries is safe; other kinds keep their
        barrier words at offset 0 and free-form data after them."""
        key = (str(device), torch.cuda.current_stream(device).cuda_stream, kind)
        b = self.bufs.get(key)
        if b is None or b.numel() < nbytes:
            b = torch.zeros(max(nbytes, 1 << 16), dtype=torch.uint8, device=device)  # barrier words must start at 0
            self.bufs[key] = b
        return b

    def frame(self, shape, dtype, device, tag: str = "frame") -> torch.Tensor:
        """Device staging frame (host-frame unit path, CHANNELS_FIRST windows), cached per
        (device, stream, tag, shape, dtype); its content outside the copied regions is
        never read."""
        key = (str(device), torch.cuda.current_stream(device).cuda_stream, tag, tuple(shape), dtype)
        b = self.bufs.get(key)
        if b is None:
            b = torch.empty(shape, dtype=dtype, device=device)
            self.bufs[key] = b
        return b


_SCRATCH = _Scratch()


# ----------------------------------------------------------------------------- sparse conv

def sparse_conv2d(x: Tensor4D, mask: BinaryMask, f: FilterBank, p: ConvParams,
                  block_size: tuple[int, int], pool: PoolMode = PoolMode.MAX,
                  threshold: float | None = None, dst: Tensor4D | None = None,
                  algo="auto") -> Tensor4D:
    """Mask-guided convolution (reference `layers.py:27-47`): reduce_mask, then one fused
    gather -> valid conv -> scatter kernel.  Output pixels in active write regions equal
    the dense convolution; others keep `dst` (zeros by default)."""
    _check_mask(x, mask)
    if f.kernel != tuple(p.kernel) or f.c_in != x.dims[3] or f.c_out != p.filter_count:
        raise ShapeMismatchError("filter bank does not match the conv params / input channels")
    spec = compute_block_spec(x.dims, p, block_size)
    out_layout = x.layout if dst is None else dst.layout  # the result takes dst's layout (blocks.py:141)
    if (x.layout is Layout.CHANNELS_FIRST and out_layout is Layout.CHANNELS_FIRST
            and _cf_windows_ok(x.dtype, (x.dims[3], spec.block_size[1]), (f.c_out, spec.out_block_size[1]))):
        return _sparse_conv2d_channels_first(x, mask, f, p, spec, pool, threshold, dst, algo)
    xt = cuda(x.nhwc())
    n = x.dims[0]
    if dst is None:
        out = torch.zeros((n, spec.out_size[0], spec.out_size[1], f.c_out), dtype=xt.dtype,
                          device=xt.device)
    else:
        if dst.dims != (n, spec.out_size[0], spec.out_size[1], f.c_out):
            raise ShapeMismatchError(f"destination dims {dst.dims} != conv output")
        out = cuda(dst.nhwc()).clone()
    if pool == PoolMode.MAX and threshold is None:
        # default pooling: the mask reduction runs inside the conv kernel (one launch)
        sparse_conv_masked_into(xt, out, cuda(mask.data), f, p, spec, algo)
    else:
        sparse_conv_into(xt, out, f, p, spec, reduce_mask(mask, spec, pool, threshold), algo)
    return Tensor4D.from_nhwc(out, out_layout)


def _cf_windows_ok(dtype: torch.dtype, *regions: tuple[int, int]) -> bool:
    """Whether sbn_copy_block_regions_t can move these (channels, row width) windows: it
    copies 16-byte pixel vectors (c * element size % 16 == 0) through a shared-memory row
    tile of c * (width + 1) elements (<= 96 KB, gather_scatter.cu).  Otherwise the caller
    takes the full-layout NHWC path."""
    es = torch.empty((), dtype=dtype).element_size()
    return all(ch * es % 16 == 0 and ch * (wd + 1) * es <= 96 * 1024 for ch, wd in regions)


def _copy_windows_t(src: torch.Tensor, dst: torch.Tensor, c: int, spec: BlockSpec, idx: BlockIndexList,
                    region: int, to_channels_last: bool) -> None:
    """Active window regions between a CHANNELS_FIRST tensor and an NHWC staging tensor
    (sbn_copy_block_regions_t; region 0 input windows, 1 output windows)."""
    lib = _lib.load()
    g = spec.c_geometry(src.shape[0])
    _lib.check(lib.sbn_copy_block_regions_t(src.data_ptr(), dst.data_ptr(), dtype_code(src.dtype), c, C.byref(g),
                                            idx.rows.data_ptr(), idx.count_dev.data_ptr(), idx.capacity, region,
                                            0 if to_channels_last else 1, _lib.stream_handle(src.device)),
               "copy_block_regions_t")


def _sparse_conv2d_channels_first(x: Tensor4D, mask: BinaryMask, f: FilterBank, p: ConvParams,
                                  spec: BlockSpec, pool, threshold, dst, algo) -> Tensor4D:
    """sparse_conv2d for CHANNELS_FIRST storage at sparse cost: the active input windows
    are transposed into an NHWC staging frame, the NHWC conv runs there, and only the
    active output windows are transposed back (no full-tensor layout conversion)."""
    xc = cuda(x.data)  # (n, c, h, w)
    n, h, w, c = x.dims
    oh, ow = spec.out_size
    idx = reduce_mask(mask, spec, pool, threshold)
    idx.to_device(xc.device)
    stage_in = _SCRATCH.frame((n, h, w, c), xc.dtype, xc.device, tag="cf_conv_in")
    stage_out = _SCRATCH.frame((n, oh, ow, f.c_out), xc.dtype, xc.device, tag="cf_conv_out")
    _copy_windows_t(xc, stage_in, c, spec, idx, 0, True)
    sparse_conv_into(stage_in, stage_out, f, p, spec, idx, algo)
    if dst is None:
        out = torch.zeros((n, f.c_out, oh, ow), dtype=xc.dtype, device=xc.device)
    else:
        if dst.dims != (n, oh, ow, f.c_out):
            raise ShapeMismatchError(f"destination dims {dst.dims} != conv output")
        out = cuda(dst.data).clone()
    _copy_windows_t(stage_out, out, f.c_out, spec, idx, 1, False)
    return Tensor4D(out, Layout.CHANNELS_FIRST)


def _conv_packed(lib, f: FilterBank, w: torch.Tensor, dc: int, p: ConvParams, g, device) -> torch.Tensor | None:
    """Tensor-core weight image for (filter bank, kernel variant), packed once and cached."""
    kh, kw = p.kernel
    sh, sw = p.stride
    nb = lib.sbn_sparse_conv_packed_bytes(dc, f.c_in, f.c_out, kh, kw, sh, sw, C.byref(g))
    if not nb:
        return None
    key = ("tc_pack", w.dtype, str(device), kh, kw, sh, sw, g.bh, g.bw)  # layout depends on the kernel variant
    packed = f._cache.get(key)
    if packed is None:
        packed = torch.empty(nb, dtype=torch.uint8, device=device)
        _lib.check(lib.sbn_sparse_conv_pack(w.data_ptr(), dc, f.c_in, f.c_out, kh, kw, sh, sw, C.byref(g),
                                            packed.data_ptr(), _lib.stream_handle(device)), "sparse_conv_pack")
        f._cache[key] = packed
    return packed


def sparse_conv_masked_into(xt: torch.Tensor, out: torch.Tensor, mask: torch.Tensor, f: FilterBank,
                            p: ConvParams, spec: BlockSpec, algo="auto") -> None:
    """sparse_conv2d from the (device) mask with the default MAX pooling, stream-ordered, no
    sync: on the tcgen05 path one kernel reduces the mask and convolves the active blocks
    (sbn_sparse_conv_masked); otherwise reduce_mask + the fused conv."""
    lib = _lib.load()
    w, b = f.device_tensors(xt.dtype, xt.device)
    g = spec.c_geometry(xt.shape[0])
    kh, kw = p.kernel
    sh, sw = p.stride
    a = _algo(algo)
    dc = dtype_code(xt.dtype)
    packed = _conv_packed(lib, f, w, dc, p, g, xt.device) if a != _lib.SBN_ALGO_SIMT else None
    gb = C.byref(g)
    sync = _SCRATCH.get(int(lib.sbn_sparse_conv_masked_sync_bytes(gb)), xt.device, "conv_sync")
    ws = _SCRATCH.get(int(lib.sbn_sparse_conv_masked_workspace(dc, f.c_in, f.c_out, kh, kw, sh, sw, gb)),
                      xt.device, "conv_scratch")
    st = lib.sbn_sparse_conv_masked(xt.data_ptr(), mask.data_ptr(), dc, f.c_in, f.c_out, kh, kw, sh, sw, gb,
                                    w.data_ptr(), None if b is None else b.data_ptr(),
                                    None if packed is None else packed.data_ptr(), out.data_ptr(),
                                    sync.data_ptr(), sync.numel(), ws.data_ptr(), ws.numel(), a,
                                    _lib.stream_handle(xt.device))
    _lib.check(st, "sparse_conv2d")


def sparse_conv_into(xt: torch.Tensor, out: torch.Tensor, f: FilterBank, p: ConvParams,
                     spec: BlockSpec, idx: BlockIndexList, algo="auto") -> None:
    """Fused gather -> conv -> scatter of the active blocks of `xt` into `out` (NHWC CUDA
    tensors), stream-ordered, no sync."""
    lib = _lib.load()
    w, b = f.device_tensors(xt.dtype, xt.device)
    idx.to_device(xt.device)
    g = spec.c_geometry(xt.shape[0])
    kh, kw = p.kernel
    sh, sw = p.stride
    a = _algo(algo)
    dc = dtype_code(xt.dtype)
    packed = None
    if a != _lib.SBN_ALGO_SIMT:
        nb = lib.sbn_sparse_conv_packed_bytes(dc, f.c_in, f.c_out, kh, kw, sh, sw, C.byref(g))
        if nb:
            key = ("tc_pack", xt.dtype, str(xt.device), kh, kw, sh, sw, g.bh, g.bw)  # layout depends on the kernel variant
            packed = f._cache.get(key)
            if packed is None:
                packed = torch.empty(nb, dtype=torch.uint8, device=xt.device)
                _lib.check(lib.sbn_sparse_conv_pack(w.data_ptr(), dc, f.c_in, f.c_out, kh, kw, sh, sw,
                                                    C.byref(g), packed.data_ptr(),
                                                    _lib.stream_handle(xt.device)), "sparse_conv_pack")
                f._cache[key] = packed
    st = lib.sbn_sparse_conv(xt.data_ptr(), dc, f.c_in, f.c_out, kh, kw, sh, sw,
                             C.byref(g), w.data_ptr(), None if b is None else b.data_ptr(),
                             None if packed is None else packed.data_ptr(),
                             idx.rows.data_ptr(), idx.count_dev.data_ptr(), idx.capacity,
                             out.data_ptr(), None, 0, a, _lib.stream_handle(xt.device))
    _lib.check(st, "sparse_conv2d")


def sparse_conv_algo(dtype: torch.dtype, f: FilterBank, p: ConvParams, spec: BlockSpec) -> str:
    g = spec.c_geometry(1)
    a = _lib.load(False).sbn_sparse_conv_algo(dtype_code(dtype), f.c_in, f.c_out, *p.kernel,
                                              *p.stride, C.byref(g))
    return "tcgen05" if a == _lib.SBN_ALGO_TCGEN05 else "simt"


def sparse_conv2d_grads(x: Tensor4D, mask: BinaryMask, f: FilterBank, p: ConvParams,
                        block_size: tuple[int, int], g_out: Tensor4D, pool: PoolMode = PoolMode.MAX,
                        threshold: float | None = None):
    """Input / weight / bias gradients of sparse_conv2d for upstream gradient g_out
    (reference `layers.py:50-65`): gather (sbn_gather) -> scatter_grad (sbn_gather over the
    output grid) -> per-block conv gradients on the stack -> gather_grad
    (sbn_gather_grad).  Returns (dx Tensor4D, dw HWIO tensor, db tensor) on the device."""
    _check_mask(x, mask)
    spec = compute_block_spec(x.dims, p, block_size)
    idx = reduce_mask(mask, spec, pool, threshold)
    xt = cuda(x.nhwc())
    w, _ = f.device_tensors(xt.dtype, xt.device)
    if idx.count == 0:
        return (Tensor4D.from_nhwc(torch.zeros_like(xt), x.layout), torch.zeros_like(w),
                torch.zeros(f.c_out, dtype=xt.dtype, device=xt.device))
    g = gather(Tensor4D(xt), idx, spec)
    gb = scatter_grad(g_out, idx, spec)
    dxb, dw, db = conv_grads_nhwc(g.tensor.data, w, p.stride, (0, 0), cuda(gb.tensor.data))
    dx = gather_grad(g.with_tensor(Tensor4D(dxb)), spec, x.dims)
    return Tensor4D.from_nhwc(dx.nhwc(), x.layout), dw, db


def sparse_residual_unit_grads(x: Tensor4D, mask: BinaryMask, u: "ResidualUnitParams",
                               block_size: tuple[int, int], g_out: Tensor4D, halo: int = 1):
    """Input and conv-weight gradients of the pre-activation, inference-BN sparse unit
    (reference `layers.py:232-270`).  The branch is recomputed on the gathered stack with
    its intermediates, differentiated back through 1x1 / ReLU / BN scale / crop / 3x3 /
    in-bounds map / 1x1 / ReLU / BN1 scale, and gather_grad'ed onto g_out — every step on
    the native kernels (direct convs `sbn_conv_forward`, `sbn_bn_relu` / `sbn_bn_relu_grad`,
    `sbn_conv_grad_*`, `sbn_gather_grad`, `sbn_add`).
    Returns (dx, {"conv1": (dw, db), "conv2": ..., "conv3": ...}) on the device."""
    if not u.pre_activation:
        raise UnsupportedConfigError("gradients implemented for the pre-activation chain only")
    _check_mask(x, mask)
    if u.channels != x.dims[3]:
        raise ShapeMismatchError(f"unit channels {u.channels} != input channels {x.dims[3]}")
    spec = unit_spec(x.dims, block_size, halo)
    idx = reduce_mask(mask, spec, PoolMode.MAX)
    xt = cuda(x.nhwc())
    dt, dev = xt.dtype, xt.device
    if dt not in (torch.float32, torch.float64):
        raise UnsupportedConfigError("residual-unit gradients are float32/float64 (as the reference)")
    ws = {}
    for nm in ("conv1", "conv2", "conv3"):
        fb = getattr(u, nm)
        wt, bt = fb.device_tensors(dt, dev)
        ws[nm] = (wt, bt if bt is not None else torch.zeros(fb.c_out, dtype=dt, device=dev))
    if idx.count == 0:
        return g_out, {nm: (torch.zeros_like(ws[nm][0]), torch.zeros_like(ws[nm][1])) for nm in ws}
    a = gather(Tensor4D(xt), idx, spec).tensor.data
    conv2_pad = (0, 0) if halo >= 1 else (1, 1)
    crop = halo - 1 if halo >= 1 else 0
    valid = in_bounds_map(idx, spec, x.dims[0]).to(dt)[..., None]
    s1, t1 = u.bn1.folded(dt, dev)
    s2, t2 = u.bn2.folded(dt, dev)
    s3, t3 = u.bn3.folded(dt, dev)

    def conv(t, nm, pad=(0, 0)):
        return conv_forward_nhwc(t, ws[nm][0], ws[nm][1], (1, 1), pad)

    # every step native: direct convs, BN + ReLU (+ in-bounds map) and their adjoints
    b1, r1 = bn_relu_nhwc(a, s1, t1)
    b2, r2 = bn_relu_nhwc(conv(r1, "conv1"), s2, t2, valid)
    c2 = conv(r2, "conv2", conv2_pad)
    c2c = c2[:, crop:c2.shape[1] - crop, crop:c2.shape[2] - crop].contiguous() if crop else c2
    b3, r3 = bn_relu_nhwc(c2c, s3, t3)
    gb = cuda(scatter_grad(g_out, idx, spec).tensor.data)
    d_r3, dw3, db3 = conv_grads_nhwc(r3, ws["conv3"][0], (1, 1), (0, 0), gb)
    d_c2c = bn_relu_grad_nhwc(d_r3, b3, s3)
    if crop:
        d_c2 = torch.zeros(c2.shape, dtype=dt, device=dev)
        d_c2[:, crop:-crop, crop:-crop] = d_c2c
        d_c2c = d_c2
    d_r2, dw2, db2 = conv_grads_nhwc(r2, ws["conv2"][0], (1, 1), conv2_pad, d_c2c)
    d_c1 = bn_relu_grad_nhwc(d_r2, b2, s2, valid)
    d_r1, dw1, db1 = conv_grads_nhwc(r1, ws["conv1"][0], (1, 1), (0, 0), d_c1)
    d_a0 = bn_relu_grad_nhwc(d_r1, b1, s1)
    d_branch = gather_grad(GatheredBlocks(Tensor4D(d_a0.contiguous()), spec, idx), spec, x.dims)
    dx = add_nhwc(cuda(g_out.nhwc()), d_branch.data)
    return Tensor4D.from_nhwc(dx, x.layout), {"conv1": (dw1, db1), "conv2": (dw2, db2), "conv3": (dw3, db3)}


def sparse_batch_norm(blocks: GatheredBlocks, bn: BnParams, mode: BnMode = BnMode.INFERENCE):
    """Batch norm over gathered blocks only (reference `layers.py:68-82`)."""
    t = cuda(blocks.tensor.nhwc())
    if bn.channels != t.shape[3]:
        raise ShapeMismatchError(f"bn channels {bn.channels} != block channels {t.shape[3]}")
    if mode is BnMode.INFERENCE:
        return blocks.with_tensor(Tensor4D.from_nhwc(bn_inference(t, bn), blocks.tensor.layout))
    if blocks.count == 0:
        raise EmptyBlockListError("train-mode statistics are undefined for an empty block list")
    if t.dtype not in (torch.float32, torch.float64):
        raise UnsupportedConfigError("train-mode batch norm is float32 / float64 (as the reference)")
    # native: deterministic per-channel mean / population variance + normalisation (sbn_bn_train)
    lib = _lib.load()
    t = t.contiguous()
    c = t.shape[3]
    rows = t.numel() // c
    g = torch.as_tensor(np.asarray(bn.gamma), device=t.device, dtype=t.dtype)
    be = torch.as_tensor(np.asarray(bn.beta), device=t.device, dtype=t.dtype)
    out = torch.empty_like(t)
    mean = torch.empty(c, dtype=t.dtype, device=t.device)
    var = torch.empty(c, dtype=t.dtype, device=t.device)
    dt = dtype_code(t.dtype)
    ws = torch.empty(int(lib.sbn_bn_train_workspace(dt, rows, c)), dtype=torch.uint8, device=t.device)
    _lib.check(lib.sbn_bn_train(t.data_ptr(), dt, rows, c, g.data_ptr(), be.data_ptr(), float(bn.epsilon),
                                out.data_ptr(), mean.data_ptr(), var.data_ptr(), ws.data_ptr(), ws.numel(),
                                _lib.stream_handle(t.device)), "bn_train")
    return blocks.with_tensor(Tensor4D.from_nhwc(out, blocks.tensor.layout)), (mean, var)


# ----------------------------------------------------------------------------- residual unit

@dataclass(frozen=True, eq=False)
class ResidualUnitParams:
    """Bottleneck 1x1 (c->m), 3x3 (m->m), 1x1 (m->c) with per-conv BN
    (reference `layers.py:85-114`)."""

    conv1: FilterBank
    conv2: FilterBank
    conv3: FilterBank
    bn1: BnParams
    bn2: BnParams
    bn3: BnParams
    pre_activation: bool = True
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        if self.conv1.kernel != (1, 1) or self.conv3.kernel != (1, 1):
            raise ShapeMismatchError("conv1/conv3 must be 1x1")
        if self.conv2.kernel != (3, 3):
            raise ShapeMismatchError("conv2 must be 3x3")
        if self.conv1.c_out != self.conv2.c_in or self.conv2.c_out != self.conv3.c_in:
            raise ShapeMismatchError("unit channel chain is inconsistent")
        if self.conv3.c_out != self.conv1.c_in:
            raise ShapeMismatchError(
                f"identity shortcut needs c_out {self.conv3.c_out} == c_in {self.conv1.c_in}")

    @property
    def channels(self) -> int:
        return self.conv1.c_in

    @property
    def mid_channels(self) -> int:
        return self.conv1.c_out

    def c_params(self, dtype: torch.dtype, device, geometry=None, halo: int = 1):
        """UnitParams struct for the C-ABI (device tensors kept alive in the cache).  With
        a geometry on the tcgen05 path, the packed tensor-core weight image is built once
        (sbn_residual_unit_pack) and attached."""
        key = (dtype, str(device))
        if key not in self._cache:
            keep = []
            up = _lib.UnitParams()
            for i, fb in enumerate((self.conv1, self.conv2, self.conv3), 1):
                w, b = fb.device_tensors(dtype, device)
                if b is None:
                    b = torch.zeros(fb.c_out, dtype=dtype, device=device)
                keep += [w, b]
                setattr(up, f"w{i}", w.data_ptr())
                setattr(up, f"b{i}", b.data_ptr())
            for i, bn in enumerate((self.bn1, self.bn2, self.bn3), 1):
                s, t = bn.folded(dtype, device)
                keep += [s, t]
                setattr(up, f"bn{i}_scale", s.data_ptr())
                setattr(up, f"bn{i}_shift", t.data_ptr())
            up.tc_packed = None
            self._cache[key] = (up, keep)
        base = self._cache[key][0]
        if geometry is None:
            return base
        lib = _lib.load()
        # the image layout depends on the variant the geometry selects (block size AND the
        # candidate count n*gy*gx: fused single kernel vs wide three-launch unit); the image
        # is cached per (variant, byte count) and the C side rejects a mismatched image
        args = (dtype_code(dtype), self.channels, self.mid_channels, C.byref(geometry), halo,
                int(self.pre_activation))
        nb = int(lib.sbn_residual_unit_packed_bytes(*args))
        variant = int(lib.sbn_residual_unit_packed_variant(*args))
        gkey = key + (geometry.bh, geometry.bw, halo, variant, nb)
        if gkey not in self._cache:
            if nb == 0:
                self._cache[gkey] = (base, None)
            else:
                img = torch.empty(nb, dtype=torch.uint8, device=device)
                st = lib.sbn_residual_unit_pack(C.byref(base), dtype_code(dtype), self.channels,
                                                self.mid_channels, C.byref(geometry), halo,
                                                int(self.pre_activation), img.data_ptr(),
                                                _lib.stream_handle(device))
                _lib.check(st, "residual_unit_pack")
                up = _lib.UnitParams()
                C.memmove(C.byref(up), C.byref(base), C.sizeof(base))
                up.tc_packed = img.data_ptr()
                up.tc_packed_bytes = nb
                up.tc_packed_variant = variant
                self._cache[gkey] = (up, img)
        return self._cache[gkey][0]


def random_unit_params(rng: np.random.Generator, c: int, m: int, dtype=np.float32,
                       scale: float = 0.2, pre_activation: bool = True) -> ResidualUnitParams:
    """Seeded random unit; consumes the generator in the same order as the reference
    (`layers.py:117-134`) so equal seeds give equal weights on both sides."""
    def filt(kh, kw, ci, co):
        wts = rng.standard_normal((kh, kw, ci, co)).astype(dtype) * scale
        return FilterBank(wts, rng.standard_normal(co).astype(dtype) * scale)

    def norm(ch):
        gamma = (0.5 + rng.random(ch)).astype(dtype)
        beta = (rng.standard_normal(ch) * scale).astype(dtype)
        mean = (rng.standard_normal(ch) * scale).astype(dtype)
        var = (0.5 + rng.random(ch)).astype(dtype)
        return BnParams(gamma, beta, mean, var)

    first = norm(c if pre_activation else m)
    last = norm(m if pre_activation else c)
    f1, f2, f3 = filt(1, 1, c, m), filt(3, 3, m, m), filt(1, 1, m, c)
    mid = norm(m)
    return ResidualUnitParams(f1, f2, f3, first, mid, last, pre_activation)


def unit_spec(x_dims, block_size, halo: int = 1) -> BlockSpec:
    """Geometry of the shared gather/scatter pair around the unit's receptive growth:
    an effective (2*halo+1)^2 SAME conv (reference `layers.py:182-191`)."""
    if halo < 0:
        raise GeometryError(f"halo must be >= 0, got {halo}")
    k = 2 * halo + 1
    if block_size[0] < k or block_size[1] < k:
        raise GeometryError(f"block size {tuple(block_size)} too small for halo {halo}")
    eff = ConvParams(kernel=(k, k), stride=(1, 1), padding=Padding.SAME, filter_count=x_dims[3])
    return compute_block_spec(x_dims, eff, block_size)


def _dense_unit_bf16(t: torch.Tensor, u: "ResidualUnitParams") -> torch.Tensor:
    """The dense comparator of the bf16 unit at cuDNN's best: BN2/BN3 folded into conv1/conv2
    (per-output-channel weight scale + bias) with ReLU fused into the convolution
    (cudnn_convolution_relu), BN1+ReLU as one addcmul + in-place relu, conv3 + bias, then
    the residual add.  Same math as `_dense_branch` up to bf16 rounding."""
    key = ("dense_fused", str(t.device))
    if key not in u._cache:
        def fold(fb, bn):
            w, b = fb.device_tensors(torch.float32, t.device)
            b = b if b is not None else torch.zeros(fb.c_out, device=t.device)
            sc, sh = bn.folded(torch.float32, t.device)
            wf = (w * sc).permute(3, 2, 0, 1).contiguous(memory_format=torch.channels_last).to(torch.bfloat16)
            return wf, (b * sc + sh).to(torch.bfloat16)
        s1, t1 = u.bn1.folded(torch.float32, t.device)
        w1, b1 = fold(u.conv1, u.bn2)
        w2, b2 = fold(u.conv2, u.bn3)
        w3, b3 = u.conv3.device_tensors(torch.bfloat16, t.device)
        w3 = w3.permute(3, 2, 0, 1).contiguous(memory_format=torch.channels_last)
        u._cache[key] = (s1.to(torch.bfloat16), t1.to(torch.bfloat16), w1, b1, w2, b2, w3, b3)
    s1, t1, w1, b1, w2, b2, w3, b3 = u._cache[key]
    x = t.permute(0, 3, 1, 2)  # NCHW view of NHWC memory (channels_last)
    a = torch.addcmul(t1.view(1, -1, 1, 1), x, s1.view(1, -1, 1, 1)).relu_()
    c1 = torch.cudnn_convolution_relu(a, w1, b1, (1, 1), (0, 0), (1, 1), 1)
    c2 = torch.cudnn_convolution_relu(c1, w2, b2, (1, 1), (1, 1), (1, 1), 1)
    y = F.conv2d(c2, w3, b3)
    return (x + y).permute(0, 2, 3, 1).contiguous()


def _dense_branch(t: torch.Tensor, u: ResidualUnitParams) -> torch.Tensor:
    dt, dev = t.dtype, t.device
    w1, b1 = u.conv1.device_tensors(dt, dev)
    w2, b2 = u.conv2.device_tensors(dt, dev)
    w3, b3 = u.conv3.device_tensors(dt, dev)
    if u.pre_activation:
        r = torch.relu(bn_inference(t, u.bn1))
        r = torch.relu(bn_inference(dense_conv_nhwc(r, w1, b1, (1, 1), (0, 0)), u.bn2))
        r = torch.relu(bn_inference(dense_conv_nhwc(r, w2, b2, (1, 1), (1, 1)), u.bn3))
        return dense_conv_nhwc(r, w3, b3, (1, 1), (0, 0))
    r = torch.relu(bn_inference(dense_conv_nhwc(t, w1, b1, (1, 1), (0, 0)), u.bn1))
    r = torch.relu(bn_inference(dense_conv_nhwc(r, w2, b2, (1, 1), (1, 1)), u.bn2))
    return bn_inference(dense_conv_nhwc(r, w3, b3, (1, 1), (0, 0)), u.bn3)


def dense_residual_unit(x: Tensor4D, u: ResidualUnitParams,
                        bn_mode: BnMode = BnMode.INFERENCE, fused: bool = True) -> Tensor4D:
    """Dense unit with SAME 3x3 (reference `layers.py:194-200`) on cuDNN: the dense
    comparator of the sparse unit."""
    if u.channels != x.dims[3]:
        raise ShapeMismatchError(f"unit channels {u.channels} != input channels {x.dims[3]}")
    if bn_mode is not BnMode.INFERENCE:
        raise UnsupportedConfigError("dense_residual_unit: inference-mode BN only")
    t = cuda(x.nhwc())
    if fused and t.dtype == torch.bfloat16 and u.pre_activation:
        return Tensor4D.from_nhwc(_dense_unit_bf16(t, u), x.layout)
    return Tensor4D.from_nhwc(t + _dense_branch(t, u), x.layout)


def sparse_residual_unit(x: Tensor4D, mask: BinaryMask, u: ResidualUnitParams,
                         block_size: tuple[int, int], halo: int = 1,
                         bn_mode: BnMode = BnMode.INFERENCE,
                         _shared: tuple[BlockSpec, BlockIndexList] | None = None,
                         inplace: bool = False, algo="auto", blocking: bool = True) -> Tensor4D:
    """Residual unit inside one gather/scatter pair (reference `layers.py:203-229`);
    inactive pixels stay bit-identical to x.

    Default: functional like the reference (x is cloned, then the fused kernel
    scatter-adds into the clone).  ``inplace=True`` updates x's storage directly — the
    paper's fused scatter-add; the kernel snapshots the halo rims first, so neighbours'
    writes never leak into a window.

    ``inplace=True`` on a PINNED HOST frame updates the host frame: only the active
    blocks' input windows travel host->device and only their output windows travel back
    (`_host_frame_unit`).  With ``blocking=False`` that update is asynchronous on the
    current stream (synchronise before reading the frame), like ``copy_(non_blocking=True)``.
    """
    if u.channels != x.dims[3]:
        raise ShapeMismatchError(f"unit channels {u.channels} != input channels {x.dims[3]}")
    if bn_mode is not BnMode.INFERENCE:
        raise UnsupportedConfigError("sparse_residual_unit: inference-mode BN only (training is out of scope)")
    if inplace and _shared is None and not x.nhwc().is_cuda and x.nhwc().is_pinned():
        _check_mask(x, mask)
        _host_frame_unit(x.nhwc(), mask, u, block_size, halo, algo, blocking)
        return x
    if x.layout is Layout.CHANNELS_FIRST and _cf_windows_ok(x.dtype, (x.dims[3], block_size[1])):
        return _unit_channels_first(x, mask, u, block_size, halo, _shared, inplace, algo)
    xt = cuda(x.nhwc())
    if inplace and x.nhwc().is_cuda and xt.data_ptr() == x.nhwc().data_ptr():
        out = xt
    else:
        out = xt.clone()
    if _shared is None:
        _check_mask(x, mask)
        spec = unit_spec(x.dims, block_size, halo)
        sparse_residual_unit_into(out, out if (out is xt) else xt, cuda(mask.data), u, spec, halo, algo)
    else:
        spec, idx = _shared
        residual_unit_into(out, out if (out is xt) else xt, u, spec, idx, halo, algo)
    return Tensor4D.from_nhwc(out, x.layout)


def _unit_channels_first(x: Tensor4D, mask: BinaryMask, u: ResidualUnitParams, block_size, halo: int,
                         _shared, inplace: bool, algo) -> Tensor4D:
    """sparse_residual_unit for CHANNELS_FIRST storage at sparse cost: active input windows
    -> NHWC staging frame (transposing copy), the unit in place there, active output
    windows -> the (n, c, h, w) result; ``inplace`` updates x's own storage."""
    xc = cuda(x.data)
    n, h, w, c = x.dims
    if _shared is None:
        _check_mask(x, mask)
        spec = unit_spec(x.dims, block_size, halo)
        idx = reduce_mask(mask, spec)
    else:
        spec, idx = _shared
    idx.to_device(xc.device)
    stage = _SCRATCH.frame((n, h, w, c), xc.dtype, xc.device, tag="cf_unit")
    _copy_windows_t(xc, stage, c, spec, idx, 0, True)
    residual_unit_into(stage, stage, u, spec, idx, halo, algo)
    same = inplace and x.data.is_cuda and xc.data_ptr() == x.data.data_ptr()
    out = xc if same else xc.clone()
    _copy_windows_t(stage, out, c, spec, idx, 1, False)
    return x if same else Tensor4D(out, Layout.CHANNELS_FIRST)


class _HostFramePlan:
    """Everything the host-frame unit call needs, resolved once per (unit parameters,
    frame shape, dtype, block size, halo, algo, stream): the device staging frame, a
    device mask buffer, the index list, workspaces, the packed weight image and the
    geometry struct.  Per call only the mask copy and four C-ABI calls remain."""

    def __init__(self, u: ResidualUnitParams, shape, dtype, block_size, halo, algo, dev, stream):
        lib = _lib.load()
        n, h, w, c = shape
        self.lib = lib
        self.spec = unit_spec(tuple(shape), block_size, halo)
        self.g = self.spec.c_geometry(n)
        self.c, self.m, self.halo, self.pre = c, u.mid_channels, halo, int(u.pre_activation)
        self.dt = dtype_code(dtype)
        self.algo = _algo(algo)
        self.stage = torch.empty(shape, dtype=dtype, device=dev)
        self.md = torch.empty((n, h, w), dtype=torch.uint8, device=dev)
        self.cap = max(1, n * self.spec.grid_count[0] * self.spec.grid_count[1])
        self.rows = torch.empty((self.cap, 3), dtype=torch.int32, device=dev)
        self.count = torch.empty((1,), dtype=torch.int32, device=dev)
        gb = C.byref(self.g)
        self.rmws = torch.zeros(max(int(lib.sbn_reduce_mask_workspace(gb)), 4096), dtype=torch.uint8, device=dev)
        nb = lib.sbn_residual_unit_workspace(self.dt, c, self.m, gb, halo, self.algo)
        self.ws = torch.zeros(max(int(nb), 1 << 16), dtype=torch.uint8, device=dev)  # barrier words start at 0
        self.up = u.c_params(dtype, dev, self.g if self.algo != _lib.SBN_ALGO_SIMT else None, halo)
        self.thr = 1.0 / (self.spec.block_size[0] * self.spec.block_size[1])
        self.sh = stream.cuda_stream

    def run(self, xh: torch.Tensor, mask_data: torch.Tensor) -> None:
        lib, gb, sh = self.lib, C.byref(self.g), self.sh
        self.md.copy_(mask_data, non_blocking=True)
        _lib.check(lib.sbn_reduce_mask(self.md.data_ptr(), gb, _lib.SBN_POOL_MAX, self.thr, self.rows.data_ptr(),
                                       self.count.data_ptr(), self.rmws.data_ptr(), self.rmws.numel(), sh),
                   "reduce_mask")
        _lib.check(lib.sbn_copy_block_regions(xh.data_ptr(), self.stage.data_ptr(), self.dt, self.c, gb,
                                              self.rows.data_ptr(), self.count.data_ptr(), self.cap, 2, sh),
                   "copy_block_regions")
        _lib.check(lib.sbn_residual_unit(self.stage.data_ptr(), self.dt, self.c, self.m, gb, self.halo, self.pre,
                                         C.byref(self.up), self.rows.data_ptr(), self.count.data_ptr(), self.cap,
                                         self.stage.data_ptr(), self.ws.data_ptr(), self.ws.numel(), self.algo, sh),
                   "sparse_residual_unit")
        _lib.check(lib.sbn_copy_block_regions(self.stage.data_ptr(), xh.data_ptr(), self.dt, self.c, gb,
                                              self.rows.data_ptr(), self.count.data_ptr(), self.cap, 1, sh),
                   "copy_block_regions")


def _host_frame_unit(xh: torch.Tensor, mask: BinaryMask, u: ResidualUnitParams, block_size,
                     halo: int, algo, blocking: bool) -> None:
    """In-place unit on a pinned host frame (UVA): mask -> device, ordered reduce_mask,
    the union of the active blocks' input windows host -> device staging frame
    (sbn_copy_block_regions region 2 reads each needed host pixel once over PCIe), the
    fused unit in place on the staging frame, and the active output windows device -> host
    frame.  PCIe carries the mask plus exactly the
    bytes the sparse layer reads and writes, instead of two full frames."""
    if not xh.is_contiguous():
        raise ShapeMismatchError("host-frame unit needs a contiguous pinned NHWC frame")
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)
    key = ("host", tuple(xh.shape), xh.dtype, tuple(block_size), halo, str(algo), str(dev), stream.cuda_stream)
    plan = u._cache.get(key)
    if plan is None:
        plan = _HostFramePlan(u, xh.shape, xh.dtype, block_size, halo, algo, dev, stream)
        u._cache[key] = plan
    plan.run(xh, mask.data)
    if blocking:
        stream.synchronize()


def sparse_residual_unit_into(out: torch.Tensor, src: torch.Tensor, mask: torch.Tensor,
                              u: ResidualUnitParams, spec: BlockSpec, halo: int = 1,
                              algo="auto") -> None:
    """mask -> active blocks -> fused unit (sbn_sparse_residual_unit): one kernel on the
    tcgen05 path.  `out` holds src's values (clone) or is src (in place)."""
    lib = _lib.load()
    dt, dev = src.dtype, src.device
    n, _, _, c = src.shape
    g = spec.c_geometry(n)
    a = _algo(algo)
    nbytes = lib.sbn_sparse_residual_unit_workspace(dtype_code(dt), c, u.mid_channels, C.byref(g),
                                                    halo, a)
    ws = _SCRATCH.get(nbytes, dev, "fused_scratch")
    sync = _SCRATCH.get(lib.sbn_sparse_residual_unit_sync_bytes(C.byref(g)), dev, "fused_sync")
    up = u.c_params(dt, dev, g if a != _lib.SBN_ALGO_SIMT else None, halo)
    st = lib.sbn_sparse_residual_unit(src.data_ptr(), mask.data_ptr(), dtype_code(dt), c,
                                      u.mid_channels, C.byref(g), halo, int(u.pre_activation),
                                      C.byref(up), out.data_ptr(), sync.data_ptr(), sync.numel(),
                                      ws.data_ptr(), ws.numel(), a, _lib.stream_handle(dev))
    _lib.check(st, "sparse_residual_unit")


def residual_unit_into(out: torch.Tensor, src: torch.Tensor, u: ResidualUnitParams,
                       spec: BlockSpec, idx: BlockIndexList, halo: int = 1, algo="auto") -> None:
    """Fused unit: out[active] += branch(src windows).  `out` must hold src's values
    (either a clone, or `out is src` for the in-place form)."""
    lib = _lib.load()
    dt, dev = src.dtype, src.device
    n, _, _, c = src.shape
    m = u.mid_channels
    g = spec.c_geometry(n)
    a = _algo(algo)
    idx.to_device(dev)
    nbytes = lib.sbn_residual_unit_workspace(dtype_code(dt), c, m, C.byref(g), halo, a)
    ws = _SCRATCH.get(nbytes, dev)
    up = u.c_params(dt, dev, g if a != _lib.SBN_ALGO_SIMT else None, halo)
    st = lib.sbn_residual_unit(src.data_ptr(), dtype_code(dt), c, m, C.byref(g), halo,
                               int(u.pre_activation), C.byref(up), idx.rows.data_ptr(),
                               idx.count_dev.data_ptr(), idx.capacity, out.data_ptr(),
                               ws.data_ptr(), ws.numel(), a, _lib.stream_handle(dev))
    _lib.check(st, "sparse_residual_unit")


def residual_unit_algo(dtype: torch.dtype, u: ResidualUnitParams, spec: BlockSpec, halo=1) -> str:
    g = spec.c_geometry(1)
    a = _lib.load(False).sbn_residual_unit_algo(dtype_code(dtype), u.channels, u.mid_channels,
                                                C.byref(g), halo, int(u.pre_activation))
    return "tcgen05" if a == _lib.SBN_ALGO_TCGEN05 else "simt"


# ----------------------------------------------------------------------------- stages

@dataclass(frozen=True)
class StageConfig:
    unit_count: int
    channels: tuple[int, int, int]   # (c_in, c_mid, c_out)
    block_size: tuple[int, int]
    mask_scale: int = 1              # downsample factor from the base mask
    stride: int = 1                  # dense projection stride (stage transition)


@dataclass(frozen=True)
class Stage:
    config: StageConfig
    projection: FilterBank | None
    units: tuple[ResidualUnitParams, ...]


@dataclass(frozen=True)
class StageResult:
    output: Tensor4D
    mask: BinaryMask | None
    spec: BlockSpec | None
    indices: BlockIndexList | None


def build_stage(cfg: StageConfig, rng: np.random.Generator, dtype=np.float32,
                scale: float = 0.2) -> Stage:
    """Random stage weights, generator order as the reference (`layers.py:287-298`)."""
    c_in, c_mid, c_out = cfg.channels
    proj = None
    if cfg.stride != 1 or c_in != c_out:
        proj = FilterBank(rng.standard_normal((3, 3, c_in, c_out)).astype(dtype) * scale,
                          rng.standard_normal(c_out).astype(dtype) * scale)
    units = tuple(random_unit_params(rng, c_out, c_mid, dtype, scale) for _ in range(cfg.unit_count))
    return Stage(cfg, proj, units)


def run_stage(stage: Stage, x: Tensor4D, base_mask: BinaryMask | None, sparse: bool = True,
              bn_mode: BnMode = BnMode.INFERENCE, algo="auto", dense_fused: bool = True,
              _mask_at_scale: BinaryMask | None = None, _plan=None) -> StageResult:
    """Dense stride-s projection (tcgen05, bias fused), then residual units sharing ONE
    index list computed from the downsampled mask (reference `layers.py:311-329`).  The
    units run in place on the stage's private activation buffer (one clone at most)."""
    if bn_mode is not BnMode.INFERENCE:
        # the sparse / dense units are inference-BN only (sparse_residual_unit raises the same)
        raise UnsupportedConfigError("run_stage: inference-mode BN only")
    cfg = stage.config
    t = cuda(x.nhwc())
    owned = False
    if stage.projection is not None:
        p = ConvParams((3, 3), (cfg.stride, cfg.stride), Padding.SAME, cfg.channels[2])
        t = projection_conv(t, stage.projection, p)
        owned = True
    if not sparse:
        for u in stage.units:
            t = (_dense_unit_bf16(t, u) if (dense_fused and t.dtype == torch.bfloat16 and u.pre_activation)
                 else t + _dense_branch(t, u))
        return StageResult(Tensor4D.from_nhwc(t, x.layout), None, None, None)
    if _plan is not None:  # mask, spec and index list prepared ahead (run_backbone's side stream)
        mask, spec, idx, ready = _plan
        torch.cuda.current_stream(t.device).wait_event(ready)
    else:
        mask = _mask_at_scale if _mask_at_scale is not None else downsample_mask(base_mask, cfg.mask_scale)
        spec = None
    if mask.dims != tuple(t.shape[:3]):
        raise ShapeMismatchError(f"mask dims {mask.dims} != tensor (n, h, w) {tuple(t.shape[:3])}")
    if spec is None:
        spec = unit_spec(tuple(t.shape), cfg.block_size, halo=1)
        idx = reduce_mask(mask, spec, PoolMode.MAX)
    if not owned:
        t = t.clone()
    for u in stage.units:
        if u.channels != t.shape[3]:
            raise ShapeMismatchError(f"unit channels {u.channels} != input channels {t.shape[3]}")
        residual_unit_into(t, t, u, spec, idx, 1, algo)
    return StageResult(Tensor4D.from_nhwc(t, x.layout), mask, spec, idx)


@dataclass(frozen=True)
class Backbone:
    stages: tuple[Stage, ...]


def build_backbone(stage_cfgs, rng: np.random.Generator, dtype=np.float32,
                   scale: float = 0.2) -> Backbone:
    for prev, nxt in zip(stage_cfgs, stage_cfgs[1:]):
        if prev.channels[2] != nxt.channels[0]:
            raise ShapeMismatchError(f"stage channel chain broken: {prev.channels[2]} -> {nxt.channels[0]}")
    return Backbone(tuple(build_stage(cfg, rng, dtype, scale) for cfg in stage_cfgs))


class _SideStreams(threading.local):
    """One side stream per device for the backbone's mask pipeline."""

    def __init__(self):
        self.s = {}

    def get(self, device) -> torch.cuda.Stream:
        key = str(device)
        if key not in self.s:
            self.s[key] = torch.cuda.Stream(device=device)
        return self.s[key]


_SIDE = _SideStreams()


def _stage_out_hw(stage: Stage, h: int, w: int) -> tuple[int, int]:
    s = stage.config.stride if stage.projection is not None else 1
    return (h - 1) // s + 1, (w - 1) // s + 1  # SAME 3x3 stride-s projection


def _mask_plans(bb: Backbone, x: Tensor4D, base_mask: BinaryMask):
    """Every stage's downsampled mask, unit geometry and index list, computed on a side
    stream while the main stream runs the stages: the masks depend only on the base mask,
    so the mask kernels (latency-bound, a few SMs) overlap the projections and units
    instead of sitting between them.  Max-pool downsampling composes exactly (ceil dims,
    window = stride): each stage's mask comes from the previous stage's when the scale
    ratio is an integer, reading the small mask instead of the full-resolution one."""
    main = torch.cuda.current_stream()
    side = _SIDE.get(main.device)
    side.wait_stream(main)  # the base mask (and x) are ready
    plans = []
    n, h, w, _ = x.dims
    prev_scale, prev_mask = 1, base_mask
    with torch.cuda.stream(side):
        for stage in bb.stages:
            h, w = _stage_out_hw(stage, h, w)
            sc = stage.config.mask_scale
            if sc % prev_scale == 0:
                m_s = downsample_mask(prev_mask, sc // prev_scale)
                prev_scale, prev_mask = sc, m_s
            else:
                m_s = downsample_mask(base_mask, sc)
            if m_s.dims != (n, h, w):
                raise ShapeMismatchError(f"mask dims {m_s.dims} != stage tensor (n, h, w) {(n, h, w)}")
            spec = unit_spec((n, h, w, stage.config.channels[2]), stage.config.block_size, halo=1)
            idx = reduce_mask(m_s, spec, PoolMode.MAX)
            for t_ in (m_s.data, idx.rows, idx.count_dev):  # consumed on the main stream
                if isinstance(t_, torch.Tensor) and t_.is_cuda:
                    t_.record_stream(main)
            ready = torch.cuda.Event()
            ready.record(side)
            plans.append((m_s, spec, idx, ready))
    return plans


def run_backbone(bb: Backbone, x: Tensor4D, base_mask: BinaryMask | None, sparse: bool = True,
                 bn_mode: BnMode = BnMode.INFERENCE, algo="auto", dense_fused: bool = True) -> list[StageResult]:
    """Stages in sequence (reference `layers.py:346-353`); the sparse path prepares every
    stage's mask and index list up front on a side stream (_mask_plans)."""
    plans = [None] * len(bb.stages)
    if sparse and base_mask is not None and bb.stages:
        xt = cuda(x.nhwc())
        plans = _mask_plans(bb, Tensor4D.from_nhwc(xt, x.layout), BinaryMask(cuda(base_mask.data), validate=False))
        x = Tensor4D.from_nhwc(xt, x.layout)
    results = []
    for stage, plan in zip(bb.stages, plans):
        res = run_stage(stage, x, base_mask, sparse, bn_mode, algo, dense_fused, _plan=plan)
        results.append(res)
        x = res.output
    return results
