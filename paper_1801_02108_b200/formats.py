"""On-disk formats of the reference package, byte-compatible.

* SBT4 — one 4-d tensor (reference `tensor.py:77-110`): a little-endian 20-byte header
  ``"SBT4", version u8 = 1, dtype u8 (0 f32, 1 f64), layout u8 (0 ChannelsLast,
  1 ChannelsFirst), reserved u8, n, h, w, c as u32`` followed by the raw little-endian
  payload in storage order.  bf16 tensors are written with dtype code 2 (an extension the
  reference's loader rejects; f32/f64 files are interchangeable both ways).
* SBMK — one binary mask (reference `tiling.py:237-263`): ``"SBMK", version u8 = 1,
  n, h, w as u32`` then n*h*w bytes of 0/1.
* weights manifest — a directory of SBT4 files plus ``manifest.json``
  (``{"format": "blockconv-weights", "version": 1, "stages": [...]}``, reference
  `layers.py:355-468`), the same file names and entries, so backbones saved by either
  package load in the other.

Host-side I/O only: tensors are staged through host memory (torch) and returned as
Tensor4D / BinaryMask on the host; the GPU ops move them on first use.
"""
from __future__ import annotations

import json
import os
import struct

import numpy as np
import torch

from .errors import FormatError, ShapeMismatchError
from .tensor import Layout, Tensor4D
from .tiling import BinaryMask

SBT4_MAGIC = b"SBT4"
SBT4_HEADER = struct.Struct("<4sBBBB4I")
SBMK_MAGIC = b"SBMK"
SBMK_HEADER = struct.Struct("<4sB3I")
_DT_CODE = {torch.float32: 0, torch.float64: 1, torch.bfloat16: 2}
_CODE_DT = {0: ("<f4", torch.float32), 1: ("<f8", torch.float64), 2: ("<u2", torch.bfloat16)}


def _host(t) -> torch.Tensor:
    t = t.data if isinstance(t, Tensor4D) else t
    t = torch.as_tensor(t) if not isinstance(t, torch.Tensor) else t
    return t.detach().to("cpu").contiguous()


# ----------------------------------------------------------------------------- SBT4

def save_sbt4(path, t: Tensor4D) -> None:
    """Write a Tensor4D (storage order as held) to an SBT4 file."""
    if not isinstance(t, Tensor4D):
        t = Tensor4D(t)
    data = _host(t)
    if data.dtype not in _DT_CODE:
        raise FormatError(f"SBT4 holds float32/float64/bfloat16, not {data.dtype}")
    n, h, w, c = t.dims
    payload = data.view(torch.int16).numpy().astype("<i2") if data.dtype == torch.bfloat16 \
        else data.numpy().astype(_CODE_DT[_DT_CODE[data.dtype]][0], copy=False)
    with open(path, "wb") as f:
        f.write(SBT4_HEADER.pack(SBT4_MAGIC, 1, _DT_CODE[data.dtype], t.layout.value, 0, n, h, w, c))
        f.write(payload.tobytes())


def load_sbt4(path) -> Tensor4D:
    """Read an SBT4 file; every malformation raises FormatError with its byte offset."""
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < SBT4_HEADER.size:
        raise FormatError(f"SBT4 header truncated: {len(raw)} bytes", offset=len(raw))
    magic, version, code, layout_code, _, n, h, w, c = SBT4_HEADER.unpack_from(raw)
    if magic != SBT4_MAGIC:
        raise FormatError(f"bad magic {magic!r}, expected {SBT4_MAGIC!r}", offset=0)
    if version != 1:
        raise FormatError(f"unsupported SBT4 version {version}", offset=4)
    if code not in _CODE_DT:
        raise FormatError(f"unknown dtype code {code}", offset=5)
    if layout_code not in (0, 1):
        raise FormatError(f"unknown layout code {layout_code}", offset=6)
    np_dt, t_dt = _CODE_DT[code]
    count = n * h * w * c
    need = SBT4_HEADER.size + count * np.dtype(np_dt).itemsize
    if len(raw) != need:
        raise FormatError(f"payload size mismatch: have {len(raw)} bytes, expected {need}",
                          offset=min(len(raw), need))
    arr = np.frombuffer(raw, dtype=np_dt, count=count, offset=SBT4_HEADER.size)
    layout = Layout(layout_code)
    shape = (n, h, w, c) if layout is Layout.CHANNELS_LAST else (n, c, h, w)
    if t_dt == torch.bfloat16:
        data = torch.from_numpy(arr.astype(np.int16)).view(torch.bfloat16).reshape(shape)
    else:
        data = torch.from_numpy(arr.astype(np.dtype(np_dt).newbyteorder("="))).reshape(shape)
    return Tensor4D(data, layout)


# ----------------------------------------------------------------------------- SBMK

def save_sbmk(path, mask: BinaryMask) -> None:
    n, h, w = mask.dims
    data = _host(mask.data).to(torch.uint8).numpy()
    with open(path, "wb") as f:
        f.write(SBMK_HEADER.pack(SBMK_MAGIC, 1, n, h, w))
        f.write(data.tobytes())


def load_sbmk(path) -> BinaryMask:
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < SBMK_HEADER.size:
        raise FormatError(f"SBMK header truncated: {len(raw)} bytes", offset=len(raw))
    magic, version, n, h, w = SBMK_HEADER.unpack_from(raw)
    if magic != SBMK_MAGIC:
        raise FormatError(f"bad magic {magic!r}, expected {SBMK_MAGIC!r}", offset=0)
    if version != 1:
        raise FormatError(f"unsupported SBMK version {version}", offset=4)
    need = SBMK_HEADER.size + n * h * w
    if len(raw) != need:
        raise FormatError(f"payload size mismatch: have {len(raw)} bytes, expected {need}",
                          offset=min(len(raw), need))
    body = np.frombuffer(raw, np.uint8, offset=SBMK_HEADER.size)
    if body.size and body.max() > 1:
        k = int(np.argmax(body > 1))
        raise FormatError(f"mask byte is {body[k]}, expected 0 or 1", offset=SBMK_HEADER.size + k)
    return BinaryMask(body.reshape(n, h, w).copy())


# ----------------------------------------------------------------------------- weights manifest

def _put(dirpath, name, arr) -> str:
    t = _host(torch.as_tensor(np.asarray(arr)) if not isinstance(arr, torch.Tensor) else arr)
    if t.ndim == 1:
        t = t.reshape(1, 1, 1, -1)
    fname = f"{name}.sbt4"
    save_sbt4(os.path.join(dirpath, fname), Tensor4D(t))
    return fname


def _get(dirpath, fname, vector=False) -> np.ndarray:
    t = load_sbt4(os.path.join(dirpath, fname)).data
    a = t.float().numpy() if t.dtype == torch.bfloat16 else t.numpy()
    return a.reshape(-1) if vector else a


def _filter_out(dirpath, name, fb) -> dict:
    return {"weights": _put(dirpath, f"{name}_w", fb.weights),
            "bias": None if fb.bias is None else _put(dirpath, f"{name}_b", fb.bias)}


def _filter_in(dirpath, e):
    from .ops import FilterBank
    return FilterBank(_get(dirpath, e["weights"]), _get(dirpath, e["bias"], True) if e["bias"] else None)


def _bn_out(dirpath, name, bn) -> dict:
    return {"gamma": _put(dirpath, f"{name}_gamma", bn.gamma), "beta": _put(dirpath, f"{name}_beta", bn.beta),
            "mean": _put(dirpath, f"{name}_mean", bn.running_mean),
            "var": _put(dirpath, f"{name}_var", bn.running_var), "epsilon": bn.epsilon}


def _bn_in(dirpath, e):
    from .ops import BnParams
    return BnParams(_get(dirpath, e["gamma"], True), _get(dirpath, e["beta"], True),
                    _get(dirpath, e["mean"], True), _get(dirpath, e["var"], True), epsilon=e["epsilon"])


def save_backbone(dirpath, bb) -> None:
    """Every weight as an SBT4 file plus manifest.json (reference `layers.py:406-437`)."""
    os.makedirs(dirpath, exist_ok=True)
    stages = []
    for si, st in enumerate(bb.stages):
        cfg = st.config
        units = []
        for ui, u in enumerate(st.units):
            tag = f"s{si}_u{ui}"
            units.append({"pre_activation": u.pre_activation,
                          **{nm: _filter_out(dirpath, f"{tag}_{nm}", getattr(u, nm)) for nm in ("conv1", "conv2", "conv3")},
                          **{nm: _bn_out(dirpath, f"{tag}_{nm}", getattr(u, nm)) for nm in ("bn1", "bn2", "bn3")}})
        stages.append({"unit_count": cfg.unit_count, "channels": list(cfg.channels),
                       "block_size": list(cfg.block_size), "mask_scale": cfg.mask_scale, "stride": cfg.stride,
                       "projection": None if st.projection is None else _filter_out(dirpath, f"s{si}_proj", st.projection),
                       "units": units})
    with open(os.path.join(dirpath, "manifest.json"), "w") as f:
        json.dump({"format": "blockconv-weights", "version": 1, "stages": stages}, f, indent=2)


def load_backbone(dirpath):
    """Inverse of save_backbone (reference `layers.py:440-468`)."""
    from .layers import Backbone, ResidualUnitParams, Stage, StageConfig
    with open(os.path.join(dirpath, "manifest.json")) as f:
        man = json.load(f)
    if man.get("format") != "blockconv-weights":
        raise ShapeMismatchError("not a blockconv weights manifest")
    stages = []
    for e in man["stages"]:
        cfg = StageConfig(unit_count=e["unit_count"], channels=tuple(e["channels"]),
                          block_size=tuple(e["block_size"]), mask_scale=e["mask_scale"], stride=e["stride"])
        proj = _filter_in(dirpath, e["projection"]) if e["projection"] else None
        units = tuple(ResidualUnitParams(conv1=_filter_in(dirpath, ue["conv1"]), conv2=_filter_in(dirpath, ue["conv2"]),
                                         conv3=_filter_in(dirpath, ue["conv3"]), bn1=_bn_in(dirpath, ue["bn1"]),
                                         bn2=_bn_in(dirpath, ue["bn2"]), bn3=_bn_in(dirpath, ue["bn3"]),
                                         pre_activation=ue["pre_activation"])
                      for ue in e["units"])
        stages.append(Stage(cfg, proj, units))
    return Backbone(tuple(stages))
