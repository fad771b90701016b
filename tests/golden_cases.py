"""Loaders for the golden fixtures in tests/golden (written by oracle/make_golden.py
from the real reference).  Shared by the oracle tests (CPU) and parity tests (GPU)."""
from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def cases(npz, prefix="c"):
    """Group keys '<prefix><i>_<field>' into a list of dicts ordered by i."""
    out = {}
    for key in npz.files:
        if not key.startswith(prefix):
            continue
        head, _, field = key.partition("_")
        try:
            i = int(head[len(prefix):])
        except ValueError:
            continue
        out.setdefault(i, {})[field] = npz[key]
    return [out[i] for i in sorted(out)]


def conv_cfg(cfg):
    """(h, w, kernel, stride, same, block) from a stored cfg row."""
    h, w, kh, kw, sh, sw, same, bh, bw = (int(v) for v in cfg[:9])
    return h, w, (kh, kw), (sh, sw), bool(same), (bh, bw)


def unit_dict(case):
    """Oracle-style unit dict from a residual fixture case."""
    u = {"pre": bool(case["pre"][0])}
    for i in (1, 2, 3):
        u[f"w{i}"] = case[f"conv{i}_w"]
        u[f"b{i}"] = case[f"conv{i}_b"]
        u[f"bn{i}"] = {"gamma": case[f"bn{i}_gamma"], "beta": case[f"bn{i}_beta"],
                       "mean": case[f"bn{i}_mean"], "var": case[f"bn{i}_var"], "eps": 1e-5}
    return u


def backbone_case(tag: str):
    """(cfg, stage rows, x, mask, per-stage [(y, mask, idx)]) of the backbone fixture
    (reference run_backbone on a partial blob mask; tag 'det' = the config-4 detector chain
    at reduced H x W, 'demo' = the reference's own DEMO_STAGES)."""
    z = load("backbone")
    stages = z[f"{tag}_stages"]
    res = [(z[f"{tag}_s{i}_y"], z[f"{tag}_s{i}_mask"], z[f"{tag}_s{i}_idx"]) for i in range(len(stages))]
    return z[f"{tag}_cfg"], stages, z[f"{tag}_x"], z[f"{tag}_mask"], res
