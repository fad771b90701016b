"""Per-call host cost of the pieces of the host-frame unit call."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200 import _lib  # noqa: E402
from paper_1801_02108_b200.layers import residual_unit_into, _SCRATCH  # noqa: E402
from paper_1801_02108_b200.tensor import dtype_code  # noqa: E402

H, W, Cc, M = 400, 400, 64, 32
dev = torch.device("cuda", 0)
lib = _lib.load()
u = P.random_unit_params(np.random.default_rng(0), Cc, M)
hx = torch.randn(1, H, W, Cc).bfloat16().pin_memory()
mk = P.synth_mask_blobs((1, H, W), 0.9, 0)
hm = P.BinaryMask(mk.data.pin_memory(), validate=False)
md = mk.data.to(dev)
spec = P.unit_spec((1, H, W, Cc), (16, 16))
g = spec.c_geometry(1)
stage = torch.empty(1, H, W, Cc, dtype=torch.bfloat16, device=dev)
idx = P.reduce_mask(P.BinaryMask(md, validate=False), spec)
sh = _lib.stream_handle(dev)


def tm(name, fn, n=300):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name:40s} {(t1 - t0) / n * 1e6:8.1f} us/call host")


tm("torch.cuda.current_stream", lambda: torch.cuda.current_stream(dev))
tm("_lib.stream_handle", lambda: _lib.stream_handle(dev))
tm("spec = unit_spec", lambda: P.unit_spec((1, H, W, Cc), (16, 16)))
tm("spec.c_geometry", lambda: spec.c_geometry(1))
tm("mask H2D (cuda())", lambda: hm.data.to(dev, non_blocking=True))
tm("reduce_mask (python)", lambda: P.reduce_mask(P.BinaryMask(md, validate=False), spec))
tm("sbn_copy_block_regions (ctypes)", lambda: lib.sbn_copy_block_regions(hx.data_ptr(), stage.data_ptr(), 2, Cc, C.byref(g), idx.rows.data_ptr(), idx.count_dev.data_ptr(), idx.capacity, 0, sh))
tm("residual_unit_into (python)", lambda: residual_unit_into(stage, stage, u, spec, idx))
tm("u.c_params", lambda: u.c_params(torch.bfloat16, dev, g, 1))
nbytes = lib.sbn_residual_unit_workspace(2, Cc, M, C.byref(g), 1, 0)
ws = _SCRATCH.get(nbytes, dev)
up = u.c_params(torch.bfloat16, dev, g, 1)
tm("sbn_residual_unit (ctypes)", lambda: lib.sbn_residual_unit(stage.data_ptr(), 2, Cc, M, C.byref(g), 1, 1, C.byref(up), idx.rows.data_ptr(), idx.count_dev.data_ptr(), idx.capacity, stage.data_ptr(), ws.data_ptr(), ws.numel(), 0, sh))
rmws = _SCRATCH.get(lib.sbn_reduce_mask_workspace(C.byref(g)), dev, "rm_sync")
tm("sbn_reduce_mask (ctypes)", lambda: lib.sbn_reduce_mask(md.data_ptr(), C.byref(g), 0, 1.0 / 256, idx.rows.data_ptr(), idx.count_dev.data_ptr(), rmws.data_ptr(), rmws.numel(), sh))
tm("full public call", lambda: P.sparse_residual_unit(P.Tensor4D(hx), hm, u, (16, 16), inplace=True, blocking=False))
