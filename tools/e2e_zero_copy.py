"""Experiment: the fused in-place unit reading/writing a PINNED HOST frame directly
(UVA zero-copy), mask copied to the device; frames/s over a ring of host frames."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200 import _lib  # noqa: E402
from paper_1801_02108_b200.layers import _SCRATCH  # noqa: E402
from paper_1801_02108_b200.tensor import dtype_code  # noqa: E402

H, W, Cc, M = 400, 400, 64, 32
dev = torch.device("cuda", 0)
lib = _lib.load()
nf = 4
hx = [torch.randn(1, H, W, Cc).bfloat16().pin_memory() for _ in range(nf)]
ref_in = [h.clone() for h in hx]
hm = [P.synth_mask_blobs((1, H, W), 0.9, f).data.pin_memory() for f in range(nf)]
md = [torch.empty(1, H, W, dtype=torch.uint8, device=dev) for _ in range(2)]
u = P.random_unit_params(np.random.default_rng(0), Cc, M)
spec = P.unit_spec((1, H, W, Cc), (16, 16))
g = spec.c_geometry(1)
a = _lib.SBN_ALGO_AUTO
nbytes = lib.sbn_sparse_residual_unit_workspace(dtype_code(torch.bfloat16), Cc, M, C.byref(g), 1, a)
ws = _SCRATCH.get(nbytes, dev, "fused_scratch")
sync = _SCRATCH.get(lib.sbn_sparse_residual_unit_sync_bytes(C.byref(g)), dev, "fused_sync")
up = u.c_params(torch.bfloat16, dev, g, 1)
s = torch.cuda.current_stream(dev)


def step(i):
    f, b = i % nf, i % 2
    md[b].copy_(hm[f], non_blocking=True)
    st = lib.sbn_sparse_residual_unit(hx[f].data_ptr(), md[b].data_ptr(), dtype_code(torch.bfloat16), Cc, M,
                                      C.byref(g), 1, 1, C.byref(up), hx[f].data_ptr(), sync.data_ptr(),
                                      sync.numel(), ws.data_ptr(), ws.numel(), a, _lib.stream_handle(dev))
    _lib.check(st, "sparse_residual_unit")


# correctness on frame 0 vs the device path
xd = ref_in[0].to(dev)
y = P.sparse_residual_unit(P.Tensor4D(xd), P.BinaryMask(hm[0].to(dev), validate=False), u, (16, 16))
step(0)
torch.cuda.synchronize()
print("zero-copy == device path:", torch.equal(hx[0], y.data.cpu()))
for i in range(20):
    step(i)
torch.cuda.synchronize()
n = 400
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for i in range(n):
    step(i)
e1.record()
e1.synchronize()
print(f"zero-copy e2e: {e0.elapsed_time(e1) / n * 1e3:.1f} us/frame, {n / (e0.elapsed_time(e1) / 1e3):.0f} frames/s "
      f"(host wall {(time.perf_counter() - t0) / n * 1e6:.1f} us/frame)")
