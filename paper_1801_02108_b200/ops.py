"""Layer parameter types and the dense comparator (reference `ops.py`).

``ConvParams`` / ``FilterBank`` / ``BnParams`` keep the reference's fields, validation
and error classes (`ops.py:33-113`).  Dense convolution (`conv2d_direct`, the oracle
semantics of `ops.py:200-204`) runs on the GPU through cuDNN (torch.nn.functional.conv2d
on a channels-last view, TF32 disabled for fp32): it is the *dense baseline* the
sparse kernels are measured against and the stride-2 stage projection of
`layers.py:316-318`, not part of the sparse hot path.
"""
from __future__ import annotations

import contextlib
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch
import torch.nn.functional as F

from .errors import ShapeMismatchError
from .tensor import Layout, Tensor4D, as_torch, compute_dtype, cuda


class Padding(Enum):
    VALID = "valid"
    SAME = "same"


class BnMode(Enum):
    INFERENCE = "inference"
    TRAIN_STATS = "train_stats"


class PoolMode(Enum):
    MAX = "max"
    AVG = "avg"


@dataclass(frozen=True)
class ConvParams:
    kernel: tuple[int, int]
    stride: tuple[int, int] = (1, 1)
    padding: Padding = Padding.VALID
    filter_count: int = 1

    def __post_init__(self):
        (kh, kw), (sh, sw) = self.kernel, self.stride
        if min(kh, kw) < 1:
            raise ShapeMismatchError(f"kernel must be >= 1, got {self.kernel}")
        if min(sh, sw) < 1:
            raise ShapeMismatchError(f"stride must be >= 1, got {self.stride}")
        if sh > kh or sw > kw:  # keeps the block tiling gap-free
            raise ShapeMismatchError(f"stride {self.stride} exceeds kernel {self.kernel}")

    @property
    def pad(self) -> tuple[int, int]:
        return (self.kernel[0] // 2, self.kernel[1] // 2) if self.padding is Padding.SAME else (0, 0)

    def out_size(self, h: int, w: int) -> tuple[int, int]:
        (kh, kw), (sh, sw), (ph, pw) = self.kernel, self.stride, self.pad
        if self.padding is Padding.VALID and (h < kh or w < kw):
            raise ShapeMismatchError(f"input {h}x{w} smaller than kernel {kh}x{kw} under valid padding")
        return ((h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1)


def _np(a):
    if isinstance(a, torch.Tensor):
        t = a.detach().cpu()
        return (t.float() if t.dtype == torch.bfloat16 else t).numpy()
    return np.asarray(a)


@dataclass(frozen=True, eq=False)
class FilterBank:
    weights: object              # (kh, kw, c_in, c_out), numpy or torch
    bias: object | None = None   # (c_out,)
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        shape = tuple(self.weights.shape)
        if len(shape) != 4:
            raise ShapeMismatchError(f"filter weights must be 4-d, got {len(shape)}-d")
        if self.bias is not None and tuple(self.bias.shape) != (shape[3],):
            raise ShapeMismatchError(
                f"bias length {tuple(self.bias.shape)} does not match filter count {shape[3]}")

    @property
    def c_in(self) -> int:
        return int(self.weights.shape[2])

    @property
    def c_out(self) -> int:
        return int(self.weights.shape[3])

    @property
    def kernel(self) -> tuple[int, int]:
        return (int(self.weights.shape[0]), int(self.weights.shape[1]))

    def device_tensors(self, dtype: torch.dtype, device) -> tuple[torch.Tensor, torch.Tensor | None]:
        """HWIO weights and bias as contiguous `dtype` tensors on `device` (cached)."""
        key = (dtype, str(device))
        if key not in self._cache:
            w = cuda(as_torch(self.weights).to(dtype), device)
            b = None if self.bias is None else cuda(as_torch(self.bias).to(dtype), device)
            self._cache[key] = (w, b)
        return self._cache[key]


@dataclass(frozen=True, eq=False)
class BnParams:
    gamma: object
    beta: object
    running_mean: object
    running_var: object
    epsilon: float = 1e-5
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        c = tuple(self.gamma.shape)
        for name in ("beta", "running_mean", "running_var"):
            if tuple(getattr(self, name).shape) != c:
                raise ShapeMismatchError(f"bn {name} shape {tuple(getattr(self, name).shape)} != gamma shape {c}")
        if np.any(_np(self.running_var) < 0):
            raise ShapeMismatchError("bn running_var must be >= 0")
        if self.epsilon <= 0:
            raise ShapeMismatchError("bn epsilon must be > 0")

    @classmethod
    def identity(cls, c: int, dtype=np.float32) -> "BnParams":
        return cls(np.ones(c, dtype), np.zeros(c, dtype), np.zeros(c, dtype), np.ones(c, dtype))

    @property
    def channels(self) -> int:
        return int(self.gamma.shape[0])

    def folded(self, act_dtype: torch.dtype, device) -> tuple[torch.Tensor, torch.Tensor]:
        """Inference BN as per-channel (scale, shift), evaluated on the host in the
        parameter dtype with the reference's exact expression (`ops.py:213-216`),
        then cast to the kernels' compute dtype."""
        key = (act_dtype, str(device))
        if key not in self._cache:
            g, b, m, v = (_np(a) for a in (self.gamma, self.beta, self.running_mean, self.running_var))
            sc = g / np.sqrt(v + self.epsilon)
            sh = b - m * g / np.sqrt(v + self.epsilon)
            cd = compute_dtype(act_dtype)
            npd = np.float64 if cd == torch.float64 else np.float32
            if act_dtype in (torch.float32, torch.float64):
                npd = np.float32 if act_dtype == torch.float32 else np.float64
            self._cache[key] = (cuda(torch.from_numpy(np.ascontiguousarray(sc.astype(npd))), device),
                                cuda(torch.from_numpy(np.ascontiguousarray(sh.astype(npd))), device))
        return self._cache[key]


def _check_conv_shapes(x: Tensor4D, f: FilterBank, p: ConvParams) -> None:
    n, h, w, c = x.dims
    if f.kernel != tuple(p.kernel):
        raise ShapeMismatchError(f"filter spatial dims {f.kernel} do not match kernel {p.kernel}")
    if f.c_in != c:
        raise ShapeMismatchError(f"input channels {c} != filter c_in {f.c_in}")
    if f.c_out != p.filter_count:
        raise ShapeMismatchError(f"filter_count {p.filter_count} != filter bank c_out {f.c_out}")
    p.out_size(h, w)


@contextlib.contextmanager
def exact_fp32():
    """Disable TF32 in cuDNN/cuBLAS so fp32 comparators are true fp32."""
    a, b = torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        yield
    finally:
        torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32 = a, b


def dense_conv_nhwc(x: torch.Tensor, w_hwio: torch.Tensor, bias, stride, pad) -> torch.Tensor:
    """cuDNN convolution of an NHWC tensor; returns a contiguous NHWC tensor."""
    xin = x.permute(0, 3, 1, 2)  # NCHW logical, channels-last memory: no copy
    w = w_hwio.permute(3, 2, 0, 1).contiguous(memory_format=torch.channels_last)
    with exact_fp32():
        y = F.conv2d(xin, w, bias, stride=tuple(stride), padding=tuple(pad))
    return y.permute(0, 2, 3, 1).contiguous()


def projection_conv(t: torch.Tensor, f: FilterBank, p: ConvParams) -> torch.Tensor:
    """Dense conv + bias of an NHWC CUDA tensor — the stage-transition projection of
    `run_stage` (reference `layers.py:316-318`).  bf16 1x1 / 3x3 / 5x5 shapes with a tcgen05
    instantiation run `sbn_dense_conv` (bias fused in the epilogue: no separate bias pass);
    other shapes and dtypes run cuDNN."""
    from . import _lib
    lib = _lib.load()
    n, h, w, c = t.shape
    kh, kw = p.kernel
    if (t.dtype == torch.bfloat16 and
            lib.sbn_dense_conv_supported(2, c, f.c_out, kh, kw, p.stride[0], p.stride[1])):
        key = ("dense_tc", str(t.device))
        if key not in f._cache:
            wt, bt = f.device_tensors(torch.bfloat16, t.device)
            img = torch.empty(int(lib.sbn_dense_conv_packed_bytes(c, f.c_out, kh)), dtype=torch.uint8,
                              device=t.device)
            _lib.check(lib.sbn_dense_conv_pack(wt.data_ptr(), c, f.c_out, kh, img.data_ptr(),
                                               _lib.stream_handle(t.device)), "dense_conv_pack")
            bf = (bt.float() if bt is not None else torch.zeros(f.c_out, device=t.device)).contiguous()
            f._cache[key] = (img, bf)
        img, bf = f._cache[key]
        oh, ow = p.out_size(h, w)
        out = torch.empty((n, oh, ow, f.c_out), dtype=t.dtype, device=t.device)
        tc_ = t.contiguous()
        _lib.check(lib.sbn_dense_conv(tc_.data_ptr(), n, h, w, c, f.c_out, kh, p.stride[0], p.stride[1], p.pad[0],
                                      p.pad[1], oh, ow, img.data_ptr(), bf.data_ptr(), out.data_ptr(),
                                      _lib.stream_handle(t.device)), "dense_conv")
        return out
    w_, b_ = f.device_tensors(t.dtype, t.device)
    return dense_conv_nhwc(t, w_, b_, p.stride, p.pad)


def conv2d_direct(x: Tensor4D, f: FilterBank, p: ConvParams) -> Tensor4D:
    """Dense convolution (reference oracle semantics, `ops.py:200-204`) via cuDNN."""
    _check_conv_shapes(x, f, p)
    xt = cuda(x.nhwc())
    w, b = f.device_tensors(xt.dtype, xt.device)
    return Tensor4D.from_nhwc(dense_conv_nhwc(xt, w, b, p.stride, p.pad), x.layout)


def bn_inference(t: torch.Tensor, bn: BnParams) -> torch.Tensor:
    scale, shift = bn.folded(t.dtype, t.device)
    return (t * scale.to(t.dtype) + shift.to(t.dtype))


def batch_norm(x: Tensor4D, bn: BnParams, mode: BnMode = BnMode.INFERENCE):
    """Inference-mode per-channel batch norm (reference `ops.py:219-230`).  TRAIN_STATS
    returns (tensor, (mean, var)) over all n*h*w positions."""
    t = cuda(x.nhwc())
    if bn.channels != t.shape[3]:
        raise ShapeMismatchError(f"bn channels {bn.channels} != tensor channels {t.shape[3]}")
    if mode is BnMode.INFERENCE:
        return Tensor4D.from_nhwc(bn_inference(t, bn), x.layout)
    mean = t.mean(dim=(0, 1, 2))
    var = t.var(dim=(0, 1, 2), unbiased=False)
    g = cuda(as_torch(bn.gamma).to(t.dtype), t.device)
    be = cuda(as_torch(bn.beta).to(t.dtype), t.device)
    out = (t - mean) * (g / torch.sqrt(var + bn.epsilon)) + be
    return Tensor4D.from_nhwc(out, x.layout), (mean, var)


def relu(x: Tensor4D) -> Tensor4D:
    return Tensor4D(torch.clamp_min(x.data, 0), x.layout)


# ----------------------------------------------------------------------------- dense utilities
# The reference's dense helpers outside the sparse path (`ops.py:167-269`, `winograd.py`),
# on cuDNN so a caller switching packages finds them; exact fp32 (no TF32).

def conv_forward_nhwc(x: torch.Tensor, w_hwio: torch.Tensor, bias, stride, pad) -> torch.Tensor:
    """Direct NHWC convolution + bias of a float32 / float64 CUDA tensor on the native kernel
    (`sbn_conv_forward`; reference `ops.py:145-164`, taps accumulated in order) — the
    training path's recomputation."""
    from . import _lib
    from .tensor import dtype_code
    lib = _lib.load()
    x = x.contiguous()
    w = w_hwio.to(x.dtype).contiguous()
    n, h, wd, cin = x.shape
    kh, kw, _, cout = w.shape
    (sh, sw), (ph, pw) = tuple(stride), tuple(pad)
    oh, ow = (h + 2 * ph - kh) // sh + 1, (wd + 2 * pw - kw) // sw + 1
    y = torch.empty((n, oh, ow, cout), dtype=x.dtype, device=x.device)
    b = None if bias is None else bias.to(x.dtype).contiguous()
    _lib.check(lib.sbn_conv_forward(x.data_ptr(), dtype_code(x.dtype), n, h, wd, cin, oh, ow, cout, w.data_ptr(), kh,
                                    kw, sh, sw, ph, pw, None if b is None else b.data_ptr(), y.data_ptr(),
                                    _lib.stream_handle(x.device)), "conv_forward")
    return y


def bn_relu_nhwc(x: torch.Tensor, scale: torch.Tensor, shift: torch.Tensor, valid=None):
    """(pre, post) = (x * scale + shift, relu(pre) * valid) per channel on the native kernel
    (`sbn_bn_relu`; reference `ops.py:213-216`, `:233-234`); valid: one 0/1 value per pixel."""
    from . import _lib
    from .tensor import dtype_code
    lib = _lib.load()
    x = x.contiguous()
    pre, post = torch.empty_like(x), torch.empty_like(x)
    v = None if valid is None else valid.to(x.dtype).contiguous()
    _lib.check(lib.sbn_bn_relu(x.data_ptr(), dtype_code(x.dtype), x.numel(), x.shape[-1], scale.data_ptr(),
                               shift.data_ptr(), None if v is None else v.data_ptr(), pre.data_ptr(), post.data_ptr(),
                               _lib.stream_handle(x.device)), "bn_relu")
    return pre, post


def bn_relu_grad_nhwc(g: torch.Tensor, pre: torch.Tensor, scale: torch.Tensor, valid=None) -> torch.Tensor:
    """Adjoint of bn_relu_nhwc: g * valid * (pre > 0) * scale (`sbn_bn_relu_grad`)."""
    from . import _lib
    from .tensor import dtype_code
    lib = _lib.load()
    g, pre = g.contiguous(), pre.contiguous()
    out = torch.empty_like(g)
    v = None if valid is None else valid.to(g.dtype).contiguous()
    _lib.check(lib.sbn_bn_relu_grad(g.data_ptr(), pre.data_ptr(), dtype_code(g.dtype), g.numel(), g.shape[-1],
                                    scale.data_ptr(), None if v is None else v.data_ptr(), out.data_ptr(),
                                    _lib.stream_handle(g.device)), "bn_relu_grad")
    return out


def add_nhwc(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """a + b on the native kernel (`sbn_add`)."""
    from . import _lib
    from .tensor import dtype_code
    lib = _lib.load()
    a, b = a.contiguous(), b.contiguous()
    out = torch.empty_like(a)
    _lib.check(lib.sbn_add(a.data_ptr(), b.data_ptr(), dtype_code(a.dtype), a.numel(), out.data_ptr(),
                           _lib.stream_handle(a.device)), "add")
    return out


def conv_grads_nhwc(a: torch.Tensor, w_hwio: torch.Tensor, stride, pad, g: torch.Tensor):
    """(dx, dw, db) of a conv on an NHWC CUDA tensor for upstream gradient g (reference
    `ops.py:167-197`): the native gradient kernels (csrc/conv_grad.cu), deterministic."""
    import ctypes as C
    from . import _lib
    from .tensor import dtype_code
    lib = _lib.load()
    a, g = a.contiguous(), g.contiguous()
    w = w_hwio.to(a.dtype).contiguous()
    n, h, wd, cin = a.shape
    kh, kw, _, cout = w.shape
    oh, ow = g.shape[1], g.shape[2]
    (sh, sw), (ph, pw) = tuple(stride), tuple(pad)
    dt, sh_ = dtype_code(a.dtype), _lib.stream_handle(a.device)
    dx = torch.empty_like(a)
    _lib.check(lib.sbn_conv_grad_input(g.data_ptr(), dt, n, h, wd, cin, oh, ow, cout, w.data_ptr(), kh, kw, sh, sw,
                                       ph, pw, dx.data_ptr(), sh_), "conv_grad_input")
    dw = torch.empty_like(w)
    db = torch.empty(cout, dtype=a.dtype, device=a.device)
    ws = torch.empty(int(lib.sbn_conv_grad_weight_workspace(dt, n, oh, ow, cin, cout, kh, kw)), dtype=torch.uint8,
                     device=a.device)
    _lib.check(lib.sbn_conv_grad_weight(a.data_ptr(), g.data_ptr(), dt, n, h, wd, cin, oh, ow, cout, kh, kw, sh, sw,
                                        ph, pw, dw.data_ptr(), db.data_ptr(), ws.data_ptr(), ws.numel(), sh_),
               "conv_grad_weight")
    return dx, dw, db


def conv2d_direct_grads(x: Tensor4D, f: FilterBank, p: ConvParams, g_out: Tensor4D):
    """Dense conv gradients (reference `ops.py:207-210`)."""
    _check_conv_shapes(x, f, p)
    xt = cuda(x.nhwc())
    w, _ = f.device_tensors(xt.dtype, xt.device)
    dx, dw, db = conv_grads_nhwc(xt, w, p.stride, p.pad, cuda(g_out.nhwc(), xt.device))
    return Tensor4D.from_nhwc(dx, x.layout), dw, db
