"""Small eager driver for ncu --set full captures of every hot kernel:
fused unit (config 2, fused mask), cluster reduce_mask, tcgen05 conv (config 3, 10% and
100%), gather, scatter."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200 import _lib
from paper_1801_02108_b200.layers import sparse_conv_into, sparse_residual_unit_into

dev = torch.device("cuda", 0)
what = sys.argv[1] if len(sys.argv) > 1 else "all"
if what in ("all", "unit"):
    xs = [torch.randn(1, 400, 400, 64, device=dev).bfloat16() for _ in range(8)]
    ms = [P.synth_mask_blobs((1, 400, 400), 0.9, f).cuda() for f in range(8)]
    u = P.random_unit_params(np.random.default_rng(0), 64, 32)
    spec = P.unit_spec((1, 400, 400, 64), (16, 16))
    for i in range(12):
        sparse_residual_unit_into(xs[i % 8], xs[i % 8], ms[i % 8].data, u, spec)
        P.reduce_mask(ms[i % 8], spec)
    torch.cuda.synchronize()
if what in ("all", "conv"):
    x = torch.randn(1, 800, 700, 128, device=dev).bfloat16()
    out = torch.zeros_like(x)
    rng = np.random.default_rng(3)
    fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, 128, 128)) / 34).astype(np.float32)).bfloat16(),
                      torch.from_numpy(rng.standard_normal(128).astype(np.float32)).bfloat16())
    p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, 128)
    spec = P.compute_block_spec((1, 800, 700, 128), p, (16, 16))
    for d in (0.1, 1.0, 0.1, 1.0):
        sparse_conv_into(x, out, fb, p, spec, P.reduce_mask(P.synth_mask_topleft((1, 800, 700), 1 - d).cuda(), spec))
    torch.cuda.synchronize()
if what in ("all", "gs"):
    lib = _lib.load()
    x = torch.randn(1, 800, 700, 128, device=dev).bfloat16()
    p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, 128)
    spec = P.compute_block_spec((1, 800, 700, 128), p, (16, 16))
    idx = P.reduce_mask(P.BinaryMask.full(1, 800, 700).cuda(), spec)
    B = idx.count
    st = torch.empty(B, 16, 16, 128, device=dev, dtype=torch.bfloat16)
    bl = torch.randn(B, 14, 14, 128, device=dev).bfloat16()
    g = spec.c_geometry(1)
    for _ in range(3):
        lib.sbn_gather(x.data_ptr(), 2, 128, C.byref(g), idx.rows.data_ptr(), idx.count_dev.data_ptr(), B, 0,
                       st.data_ptr(), _lib.stream_handle())
        lib.sbn_scatter(bl.data_ptr(), 2, 128, C.byref(g), idx.rows.data_ptr(), idx.count_dev.data_ptr(), B, 0, 0,
                        x.data_ptr(), _lib.stream_handle())
    torch.cuda.synchronize()
print("done")
