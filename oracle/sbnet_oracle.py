"""CPU oracle for the SBNet sparse-block hot path — TEST INFRASTRUCTURE ONLY.

This module is a from-scratch numpy restatement of the reference package
``blockconv`` (``/root/reference/pkg/src/blockconv``) for exactly the functions on
the hot path.  It is the *checker*: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import it.  The product package ``paper_1801_02108_b200`` never imports
anything under ``oracle/`` and has no CPU fallback.

Parity pinning: every function here is checked against golden vectors produced by
running the real reference in this container (``oracle/make_golden.py`` →
``tests/golden/*.npz``) and, when ``/root/reference`` is present, directly against the
reference on seeded random cases (``tests/test_oracle.py``).

Each function cites the reference ``file:line`` whose behaviour it restates.
Data conventions: activations are numpy arrays in logical NHWC order; masks are
uint8 (n, h, w); block index lists are (B, 3) int64 rows (frame, block_y, block_x)
in ascending order.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "Geometry", "geometry", "conv_out_size", "reduce_mask", "reduce_mask_scan",
    "downsample_mask",
    "gather", "gather_transpose", "in_bounds_map", "scatter", "scatter_transpose",
    "conv_nhwc", "bn_scale_shift", "bn_apply", "unit_branch", "sparse_conv2d",
    "dense_conv2d", "sparse_residual_unit", "dense_residual_unit", "unit_geometry",
    "rel_err", "active_region",
    "gather_grad", "scatter_grad", "conv_nhwc_grads", "sparse_conv2d_grads",
    "sparse_residual_unit_grads", "sparse_batch_norm_train",
    "random_unit", "build_stage", "run_stage", "run_backbone",
]


# --------------------------------------------------------------------------- geometry

def conv_out_size(h: int, w: int, kernel, stride, pad) -> tuple[int, int]:
    """Dense conv output extent (reference ``ops.py:55-63``)."""
    return ((h + 2 * pad[0] - kernel[0]) // stride[0] + 1,
            (w + 2 * pad[1] - kernel[1]) // stride[1] + 1)


@dataclass(frozen=True)
class Geometry:
    """Overlap-save tiling of one conv (reference ``BlockSpec``, ``tiling.py:47-61``)."""
    block: tuple[int, int]
    overlap: tuple[int, int]
    in_stride: tuple[int, int]
    out_block: tuple[int, int]
    origin: tuple[int, int]
    grid: tuple[int, int]
    kernel: tuple[int, int]
    stride: tuple[int, int]
    pad: tuple[int, int]
    in_size: tuple[int, int]
    out_size: tuple[int, int]


def geometry(h: int, w: int, kernel, stride, same: bool, block) -> Geometry:
    """Restates ``compute_block_spec`` (reference ``tiling.py:64-99``).

    SAME padding is k//2 per axis (``ops.py:50-53``); overlap = k - s; the input
    stride between blocks is block - overlap; each block yields a valid-conv output
    of (block - k)//s + 1 which is also the output stride; the grid covers the
    padded extent minus one overlap with a ceil-division, at least one block.
    Raises ValueError where the reference raises GeometryError.
    """
    kernel, stride, block = tuple(kernel), tuple(stride), tuple(block)
    pad = (kernel[0] // 2, kernel[1] // 2) if same else (0, 0)
    dims = []
    for ax in range(2):
        b, k, s = block[ax], kernel[ax], stride[ax]
        if b < k:
            raise ValueError(f"block {block} smaller than kernel {kernel}")
        if (b - k) % s:
            raise ValueError(f"stride {stride} does not divide block-kernel {block}-{kernel}")
        ov = k - s
        ins = b - ov
        ob = (b - k) // s + 1
        ext = (h, w)[ax] + 2 * pad[ax]
        g = max(1, math.ceil((ext - ov) / ins))
        dims.append((ov, ins, ob, g))
    out = conv_out_size(h, w, kernel, stride, pad)
    return Geometry(block=block, overlap=(dims[0][0], dims[1][0]),
                    in_stride=(dims[0][1], dims[1][1]), out_block=(dims[0][2], dims[1][2]),
                    origin=(-pad[0], -pad[1]), grid=(dims[0][3], dims[1][3]),
                    kernel=kernel, stride=stride, pad=pad, in_size=(h, w), out_size=out)


def unit_geometry(h: int, w: int, block, halo: int = 1) -> Geometry:
    """Effective (2*halo+1)^2 SAME spec of a residual unit (reference ``layers.py:182-191``)."""
    k = 2 * halo + 1
    return geometry(h, w, (k, k), (1, 1), True, block)


def _window(g: Geometry, by: int, bx: int):
    """Input window [ys, ys+bh) x [xs, xs+bw) of block (by, bx) and its in-image clip."""
    ys = g.origin[0] + by * g.in_stride[0]
    xs = g.origin[1] + bx * g.in_stride[1]
    h, w = g.in_size
    return ys, xs, max(ys, 0), max(xs, 0), min(ys + g.block[0], h), min(xs + g.block[1], w)


# --------------------------------------------------------------------------- masks

def reduce_mask(mask: np.ndarray, g: Geometry, pool: str = "max",
                threshold: float | None = None) -> np.ndarray:
    """Restates ``reduce_mask`` (reference ``tiling.py:138-160``, window sums ``:120-135``).

    A block is active when its input window (zero outside the image) holds any set
    pixel (max) or when count/(bh*bw) >= threshold - 1e-12 in float64 (avg; the
    *full* block area is the denominator even for clipped border windows).
    Output rows are in ascending (frame, by, bx) order.  Same algorithm class as the
    reference (summed-area table + four-corner lookup) so that the CPU baseline timed
    from this port is representative; ``reduce_mask_scan`` is an independent
    per-window scan used to cross-check it.
    """
    n, h, w = mask.shape
    area = g.block[0] * g.block[1]
    if threshold is None:
        threshold = 1.0 / area
    if not 0.0 < threshold <= 1.0:
        raise ValueError(f"threshold must be in (0, 1], got {threshold}")
    sat = np.zeros((n, h + 1, w + 1), np.int64)
    np.cumsum(np.cumsum(mask, axis=1, dtype=np.int64), axis=2, out=sat[:, 1:, 1:])
    y_lo = np.clip(g.origin[0] + g.in_stride[0] * np.arange(g.grid[0]), 0, h)
    y_hi = np.clip(g.origin[0] + g.in_stride[0] * np.arange(g.grid[0]) + g.block[0], 0, h)
    x_lo = np.clip(g.origin[1] + g.in_stride[1] * np.arange(g.grid[1]), 0, w)
    x_hi = np.clip(g.origin[1] + g.in_stride[1] * np.arange(g.grid[1]) + g.block[1], 0, w)
    cnt = (sat[:, y_hi][:, :, x_hi] - sat[:, y_lo][:, :, x_hi]
           - sat[:, y_hi][:, :, x_lo] + sat[:, y_lo][:, :, x_lo])
    if pool == "max":
        on = cnt > 0
    else:
        on = (cnt / np.float64(area)) >= threshold - 1e-12
    return np.argwhere(on).astype(np.int64).reshape(-1, 3)


def reduce_mask_scan(mask: np.ndarray, g: Geometry, pool: str = "max",
                     threshold: float | None = None) -> np.ndarray:
    """Brute-force per-window scan with the same semantics as :func:`reduce_mask`
    (mirrors the reference test oracle ``tests/oracles.py:31-46``, extended to avg)."""
    n = mask.shape[0]
    area = g.block[0] * g.block[1]
    thr = 1.0 / area if threshold is None else threshold
    rows = []
    for i in range(n):
        for by in range(g.grid[0]):
            for bx in range(g.grid[1]):
                _, _, y0, x0, y1, x1 = _window(g, by, bx)
                cnt = int(mask[i, y0:y1, x0:x1].astype(np.int64).sum()) if (y1 > y0 and x1 > x0) else 0
                on = cnt > 0 if pool == "max" else (np.float64(cnt) / np.float64(area)) >= thr - 1e-12
                if on:
                    rows.append((i, by, bx))
    return np.asarray(rows, np.int64).reshape(-1, 3)


def downsample_mask(mask: np.ndarray, factor: int) -> np.ndarray:
    """Max-pool window = stride = factor, ceil dims (reference ``tiling.py:163-174``)."""
    if factor < 1:
        raise ValueError("factor must be >= 1")
    n, h, w = mask.shape
    oh, ow = -(-h // factor), -(-w // factor)
    out = np.zeros((n, oh, ow), np.uint8)
    for y in range(oh):
        for x in range(ow):
            out[:, y, x] = mask[:, y * factor:(y + 1) * factor, x * factor:(x + 1) * factor].max(axis=(1, 2))
    return out


# --------------------------------------------------------------------------- data movement

def gather(x: np.ndarray, idx: np.ndarray, g: Geometry) -> np.ndarray:
    """(B, bh, bw, C) stack with zero-filled halo (reference ``blocks.py:57-74``)."""
    c = x.shape[3]
    out = np.zeros((len(idx), g.block[0], g.block[1], c), x.dtype)
    for b, (i, by, bx) in enumerate(idx):
        ys, xs, y0, x0, y1, x1 = _window(g, by, bx)
        if y1 > y0 and x1 > x0:
            out[b, y0 - ys:y1 - ys, x0 - xs:x1 - xs] = x[i, y0:y1, x0:x1]
    return out


def gather_transpose(x: np.ndarray, idx: np.ndarray, g: Geometry) -> np.ndarray:
    """(B, C, bh, bw) channels-first stack (reference ``blocks.py:77-94``)."""
    return np.ascontiguousarray(gather(x, idx, g).transpose(0, 3, 1, 2))


def in_bounds_map(idx: np.ndarray, g: Geometry) -> np.ndarray:
    """(B, bh, bw) bool: window position read a real pixel (reference ``blocks.py:97-112``)."""
    out = np.zeros((len(idx), g.block[0], g.block[1]), bool)
    for b, (_, by, bx) in enumerate(idx):
        ys, xs, y0, x0, y1, x1 = _window(g, by, bx)
        if y1 > y0 and x1 > x0:
            out[b, y0 - ys:y1 - ys, x0 - xs:x1 - xs] = True
    return out


def scatter(blocks: np.ndarray, idx: np.ndarray, g: Geometry, dst: np.ndarray,
            add: bool = False) -> np.ndarray:
    """Write/add each (obh, obw, C) block at (by*obh, bx*obw), clipped; returns a new
    array, ``dst`` untouched (reference ``blocks.py:125-152``)."""
    out = dst.copy()
    oh, ow = g.out_size
    obh, obw = g.out_block
    for b, (i, by, bx) in enumerate(idx):
        y0, x0 = by * obh, bx * obw
        y1, x1 = min(y0 + obh, oh), min(x0 + obw, ow)
        if add:
            out[i, y0:y1, x0:x1] += blocks[b, :y1 - y0, :x1 - x0]
        else:
            out[i, y0:y1, x0:x1] = blocks[b, :y1 - y0, :x1 - x0]
    return out


def scatter_transpose(blocks_cf: np.ndarray, idx: np.ndarray, g: Geometry,
                      dst: np.ndarray) -> np.ndarray:
    """Channels-first blocks into an NHWC destination (reference ``blocks.py:155-159``)."""
    return scatter(np.ascontiguousarray(blocks_cf.transpose(0, 2, 3, 1)), idx, g, dst)


# --------------------------------------------------------------------------- dense math

def conv_nhwc(a: np.ndarray, wts: np.ndarray, bias, stride=(1, 1), pad=(0, 0)) -> np.ndarray:
    """Direct conv as one batched GEMM per kernel tap, out-of-range taps skipped
    (= zero padding); bias added last (reference ``ops.py:130-164``)."""
    n, h, w, _ = a.shape
    kh, kw, _, co = wts.shape
    oh, ow = conv_out_size(h, w, (kh, kw), stride, pad)
    out = np.zeros((n, oh, ow, co), a.dtype)
    wts = wts.astype(a.dtype, copy=False)
    for i in range(kh):
        for j in range(kw):
            # output coordinates whose tap (i, j) lands inside the input
            oy = np.arange(oh)
            ox = np.arange(ow)
            iy = oy * stride[0] + i - pad[0]
            ix = ox * stride[1] + j - pad[1]
            vy = (iy >= 0) & (iy < h)
            vx = (ix >= 0) & (ix < w)
            if not vy.any() or not vx.any():
                continue
            patch = a[:, iy[vy]][:, :, ix[vx]]
            out[:, oy[vy][0]:oy[vy][-1] + 1, ox[vx][0]:ox[vx][-1] + 1] += patch @ wts[i, j]
    if bias is not None:
        out += np.asarray(bias).astype(a.dtype, copy=False)
    return out


def bn_scale_shift(gamma, beta, mean, var, eps, dtype):
    """Inference BN folded to per-channel scale/shift (reference ``ops.py:213-216``):
    both are computed in the parameter dtype, then cast to the activation dtype."""
    inv = gamma / np.sqrt(var + eps)
    return inv.astype(dtype), (beta - mean * inv).astype(dtype)


def bn_apply(a: np.ndarray, bn) -> np.ndarray:
    scale, shift = bn_scale_shift(bn["gamma"], bn["beta"], bn["mean"], bn["var"],
                                  bn.get("eps", 1e-5), a.dtype)
    return a * scale + shift


def unit_branch(a: np.ndarray, u: dict, conv2_pad, crop: int, valid=None) -> np.ndarray:
    """Bottleneck chain inside a block stack (reference ``layers.py:137-179``).

    ``u`` holds w1,b1,w2,b2,w3,b3 (HWIO filters), bn1,bn2,bn3 (dicts) and ``pre``.
    Pre-activation: BN1-ReLU-1x1-BN2-ReLU-xvalid-3x3-crop-BN3-ReLU-1x1.
    Post-activation: 1x1-BN1-ReLU-xvalid-3x3-crop-BN2-ReLU-1x1-BN3.
    """
    def cropped(t):
        return t[:, crop:t.shape[1] - crop, crop:t.shape[2] - crop] if crop else t

    if u.get("pre", True):
        t = np.maximum(bn_apply(a, u["bn1"]), 0)
        t = conv_nhwc(t, u["w1"], u["b1"])
        t = np.maximum(bn_apply(t, u["bn2"]), 0)
        if valid is not None:
            t = t * valid[..., None].astype(t.dtype)
        t = cropped(conv_nhwc(t, u["w2"], u["b2"], (1, 1), conv2_pad))
        t = np.maximum(bn_apply(t, u["bn3"]), 0)
        return conv_nhwc(t, u["w3"], u["b3"])
    t = np.maximum(bn_apply(conv_nhwc(a, u["w1"], u["b1"]), u["bn1"]), 0)
    if valid is not None:
        t = t * valid[..., None].astype(t.dtype)
    t = cropped(conv_nhwc(t, u["w2"], u["b2"], (1, 1), conv2_pad))
    t = np.maximum(bn_apply(t, u["bn2"]), 0)
    return bn_apply(conv_nhwc(t, u["w3"], u["b3"]), u["bn3"])


# --------------------------------------------------------------------------- composite ops

def sparse_conv2d(x, mask, wts, bias, stride, same: bool, block, pool="max",
                  threshold=None, dst=None):
    """reduce_mask -> gather -> valid conv per block -> scatter (reference ``layers.py:27-47``)."""
    n, h, w, _ = x.shape
    g = geometry(h, w, wts.shape[:2], stride, same, block)
    idx = reduce_mask(mask, g, pool, threshold)
    if dst is None:
        dst = np.zeros((n, g.out_size[0], g.out_size[1], wts.shape[3]), x.dtype)
    if len(idx) == 0:
        return dst.copy()
    blk = conv_nhwc(gather(x, idx, g), wts, bias, stride, (0, 0))
    return scatter(blk, idx, g, dst)


def dense_conv2d(x, wts, bias, stride, same: bool):
    """Dense oracle (reference ``ops.py:200-204``)."""
    pad = (wts.shape[0] // 2, wts.shape[1] // 2) if same else (0, 0)
    return conv_nhwc(x, wts, bias, stride, pad)


def sparse_residual_unit(x, mask, u: dict, block, halo: int = 1, shared=None):
    """Gather -> branch -> scatter_add onto a copy of x (reference ``layers.py:203-229``)."""
    n, h, w, _ = x.shape
    if shared is None:
        g = unit_geometry(h, w, block, halo)
        idx = reduce_mask(mask, g, "max")
    else:
        g, idx = shared
    if len(idx) == 0:
        return x.copy()
    conv2_pad = (0, 0) if halo >= 1 else (1, 1)
    crop = halo - 1 if halo >= 1 else 0
    branch = unit_branch(gather(x, idx, g), u, conv2_pad, crop, in_bounds_map(idx, g))
    return scatter(branch, idx, g, x, add=True)


def dense_residual_unit(x, u: dict):
    """Dense oracle of the unit, SAME 3x3 (reference ``layers.py:194-200``)."""
    return x + unit_branch(x, u, (1, 1), 0)


# --------------------------------------------------------------------------- stages / backbone

def random_unit(rng: np.random.Generator, c: int, m: int, dtype=np.float32, scale: float = 0.2,
                pre: bool = True) -> dict:
    """Seeded unit parameters as a dict, drawing from ``rng`` in the reference's order
    (``layers.py:117-134``): first BN, last BN, conv1, conv2, conv3 (weights then bias
    each), mid BN."""
    def filt(kh, kw, ci, co):
        return (rng.standard_normal((kh, kw, ci, co)).astype(dtype) * scale,
                rng.standard_normal(co).astype(dtype) * scale)

    def norm(ch):
        gamma = (0.5 + rng.random(ch)).astype(dtype)
        beta = (rng.standard_normal(ch) * scale).astype(dtype)
        mean = (rng.standard_normal(ch) * scale).astype(dtype)
        var = (0.5 + rng.random(ch)).astype(dtype)
        return dict(gamma=gamma, beta=beta, mean=mean, var=var)

    first = norm(c if pre else m)
    last = norm(m if pre else c)
    (w1, b1), (w2, b2), (w3, b3) = filt(1, 1, c, m), filt(3, 3, m, m), filt(1, 1, m, c)
    mid = norm(m)
    return dict(pre=pre, w1=w1, b1=b1, w2=w2, b2=b2, w3=w3, b3=b3, bn1=first, bn2=mid, bn3=last)


def build_stage(rng: np.random.Generator, units: int, channels, block, mask_scale: int = 1,
                stride: int = 1, dtype=np.float32, scale: float = 0.2) -> dict:
    """Stage weights in the reference's draw order (``layers.py:287-298``): the 3x3
    projection (only when the stride or the channel count changes), then the units."""
    c_in, c_mid, c_out = channels
    proj = None
    if stride != 1 or c_in != c_out:
        proj = (rng.standard_normal((3, 3, c_in, c_out)).astype(dtype) * scale,
                rng.standard_normal(c_out).astype(dtype) * scale)
    us = [random_unit(rng, c_out, c_mid, dtype, scale) for _ in range(units)]
    return dict(proj=proj, stride=stride, block=tuple(block), mask_scale=mask_scale, units=us)


def run_stage(stage: dict, x: np.ndarray, base_mask, sparse: bool = True):
    """One backbone stage (reference ``layers.py:311-329``): dense SAME 3x3 stride-s
    projection, then the units, all sharing ONE index list reduced from
    ``downsample_mask(base_mask, mask_scale)`` with the unit geometry (halo 1).
    Returns (output, stage mask, index rows)."""
    if stage["proj"] is not None:
        w, b = stage["proj"]
        x = dense_conv2d(x, w, b, (stage["stride"], stage["stride"]), True)
    if not sparse:
        for u in stage["units"]:
            x = dense_residual_unit(x, u)
        return x, None, None
    mask = downsample_mask(base_mask, stage["mask_scale"])
    if mask.shape != x.shape[:3]:
        raise ValueError(f"mask dims {mask.shape} != tensor (n, h, w) {x.shape[:3]}")
    g = unit_geometry(x.shape[1], x.shape[2], stage["block"], 1)
    idx = reduce_mask(mask, g, "max")
    for u in stage["units"]:
        x = sparse_residual_unit(x, mask, u, stage["block"], 1, shared=(g, idx))
    return x, mask, idx


def run_backbone(stages, x: np.ndarray, base_mask, sparse: bool = True):
    """Stages in sequence (reference ``layers.py:346-353``); a list of per-stage
    (output, mask, index rows)."""
    out = []
    for st in stages:
        res = run_stage(st, x, base_mask, sparse)
        out.append(res)
        x = res[0]
    return out


# --------------------------------------------------------------------------- training path

def gather_grad(gblk: np.ndarray, idx: np.ndarray, g: Geometry, dims) -> np.ndarray:
    """Adjoint of gather: block gradients accumulated over their (overlapping) input
    windows, clipped, in index order into zeros (reference ``blocks.py:162-188``)."""
    out = np.zeros(dims, gblk.dtype)
    for b, (i, by, bx) in enumerate(idx):
        ys, xs, y0, x0, y1, x1 = _window(g, by, bx)
        if y1 > y0 and x1 > x0:
            out[i, y0:y1, x0:x1] += gblk[b, y0 - ys:y1 - ys, x0 - xs:x1 - xs]
    return out


def scatter_grad(gout: np.ndarray, idx: np.ndarray, g: Geometry) -> np.ndarray:
    """Adjoint of scatter: the upstream gradient over each block's clipped write window,
    zero outside the image (reference ``blocks.py:191-204``)."""
    oh, ow = g.out_size
    obh, obw = g.out_block
    out = np.zeros((len(idx), obh, obw, gout.shape[3]), gout.dtype)
    for b, (i, by, bx) in enumerate(idx):
        y0, x0 = by * obh, bx * obw
        y1, x1 = min(y0 + obh, oh), min(x0 + obw, ow)
        out[b, :y1 - y0, :x1 - x0] = gout[i, y0:y1, x0:x1]
    return out


def conv_nhwc_grads(a: np.ndarray, wts: np.ndarray, stride, pad, gout: np.ndarray):
    """(dx, dw, db) of ``conv_nhwc`` (reference ``ops.py:167-197``): per tap, dW is the
    patch/gradient contraction and dx accumulates gradient @ W^T at the tap's strided
    input positions."""
    n, h, w, _ = a.shape
    kh, kw, _, _ = wts.shape
    oh, ow = gout.shape[1], gout.shape[2]
    dx = np.zeros_like(a)
    dw = np.zeros(wts.shape, a.dtype)
    wt = wts.astype(a.dtype, copy=False)
    for i in range(kh):
        oy = np.arange(oh)
        iy = oy * stride[0] + i - pad[0]
        vy = (iy >= 0) & (iy < h)
        if not vy.any():
            continue
        for j in range(kw):
            ox = np.arange(ow)
            ix = ox * stride[1] + j - pad[1]
            vx = (ix >= 0) & (ix < w)
            if not vx.any():
                continue
            patch = a[:, iy[vy]][:, :, ix[vx]]
            gg = gout[:, oy[vy]][:, :, ox[vx]]
            dw[i, j] = np.einsum("nyxc,nyxk->ck", patch, gg)
            dx[:, iy[vy][0]:iy[vy][-1] + 1:stride[0], ix[vx][0]:ix[vx][-1] + 1:stride[1]] += gg @ wt[i, j].T
    return dx, dw, gout.sum(axis=(0, 1, 2))


def sparse_conv2d_grads(x, mask, wts, bias, stride, same: bool, block, gout, pool="max", threshold=None):
    """Input/weight/bias gradients of sparse_conv2d (reference ``layers.py:50-65``)."""
    n, h, w, _ = x.shape
    g = geometry(h, w, wts.shape[:2], stride, same, block)
    idx = reduce_mask(mask, g, pool, threshold)
    if len(idx) == 0:
        return np.zeros_like(x), np.zeros_like(wts), np.zeros(wts.shape[3], x.dtype)
    dxb, dw, db = conv_nhwc_grads(gather(x, idx, g), wts, stride, (0, 0), scatter_grad(gout, idx, g))
    return gather_grad(dxb, idx, g, x.shape), dw, db


def sparse_residual_unit_grads(x, mask, u: dict, block, gout, halo: int = 1):
    """Input and conv-weight gradients of the pre-activation inference-BN sparse unit
    (reference ``layers.py:232-270``): the branch is recomputed on the gathered stack with
    its intermediates, then differentiated back through 1x1 / ReLU / BN scale / crop /
    3x3 / in-bounds map / 1x1 / ReLU / BN1 scale, and gather_grad'ed onto gout."""
    n, h, w, _ = x.shape
    g = unit_geometry(h, w, block, halo)
    idx = reduce_mask(mask, g, "max")
    if len(idx) == 0:
        z = {k: (np.zeros_like(u[f"w{k[-1]}"]), np.zeros(u[f"w{k[-1]}"].shape[3])) for k in ("conv1", "conv2", "conv3")}
        return gout.copy(), z
    a = gather(x, idx, g)
    conv2_pad = (0, 0) if halo >= 1 else (1, 1)
    crop = halo - 1 if halo >= 1 else 0
    valid = in_bounds_map(idx, g).astype(x.dtype)
    b1 = bn_apply(a, u["bn1"])
    r1 = np.maximum(b1, 0)
    c1 = conv_nhwc(r1, u["w1"], u["b1"])
    b2 = bn_apply(c1, u["bn2"])
    r2 = np.maximum(b2, 0) * valid[..., None]
    c2 = conv_nhwc(r2, u["w2"], u["b2"], (1, 1), conv2_pad)
    c2c = c2[:, crop:c2.shape[1] - crop, crop:c2.shape[2] - crop] if crop else c2
    b3 = bn_apply(c2c, u["bn3"])
    r3 = np.maximum(b3, 0)

    def sc(bn, dt):
        return (bn["gamma"] / np.sqrt(bn["var"] + bn.get("eps", 1e-5))).astype(dt)

    gb = scatter_grad(gout, idx, g)
    d_r3, dw3, db3 = conv_nhwc_grads(r3, u["w3"], (1, 1), (0, 0), gb)
    d_c2c = d_r3 * (b3 > 0) * sc(u["bn3"], d_r3.dtype)
    if crop:
        pd = np.zeros(c2.shape, d_c2c.dtype)
        pd[:, crop:-crop, crop:-crop, :] = d_c2c
        d_c2c = pd
    d_r2, dw2, db2 = conv_nhwc_grads(r2, u["w2"], (1, 1), conv2_pad, d_c2c)
    d_c1 = d_r2 * valid[..., None] * (b2 > 0) * sc(u["bn2"], d_r2.dtype)
    d_r1, dw1, db1 = conv_nhwc_grads(r1, u["w1"], (1, 1), (0, 0), d_c1)
    d_a0 = d_r1 * (b1 > 0) * sc(u["bn1"], d_r1.dtype)
    return gout + gather_grad(d_a0, idx, g, x.shape), {"conv1": (dw1, db1), "conv2": (dw2, db2),
                                                       "conv3": (dw3, db3)}


def sparse_batch_norm_train(stack: np.ndarray, gamma, beta, eps: float = 1e-5):
    """TRAIN_STATS batch norm over the gathered positions only (reference ``layers.py:68-82``)."""
    mean = stack.mean(axis=(0, 1, 2))
    var = stack.var(axis=(0, 1, 2))
    scale = (gamma / np.sqrt(var + eps)).astype(stack.dtype)
    return (stack - mean.astype(stack.dtype)) * scale + np.asarray(beta).astype(stack.dtype), mean, var


# --------------------------------------------------------------------------- metrics

def rel_err(a, b) -> float:
    """max|a-b| / max|b| in float64 (reference ``verify.py:20-27``)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-12))


def active_region(g: Geometry, idx: np.ndarray, n: int) -> np.ndarray:
    """(n, oh, ow) bool map of output pixels inside active write regions
    (reference ``verify.py:50-57``)."""
    oh, ow = g.out_size
    obh, obw = g.out_block
    region = np.zeros((n, oh, ow), bool)
    for i, by, bx in idx:
        region[i, by * obh:min((by + 1) * obh, oh), bx * obw:min((bx + 1) * obw, ow)] = True
    return region
