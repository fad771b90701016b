"""Probe: sbn_gather from a pinned HOST frame and sbn_scatter into it (UVA zero-copy),
config-2 geometry (108 active 16x16 blocks of a 400x400x64 bf16 frame)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200 import _lib  # noqa: E402

H, W, Cc = 400, 400, 64
dev = torch.device("cuda", 0)
lib = _lib.load()
hx = torch.randn(1, H, W, Cc).bfloat16().pin_memory()
dx = hx.to(dev)
spec = P.unit_spec((1, H, W, Cc), (16, 16))
mk = P.synth_mask_blobs((1, H, W), 0.9, 0).cuda()
idx = P.reduce_mask(mk, spec)
B = idx.count
g = spec.c_geometry(1)
stack = torch.empty(B, 16, 16, Cc, dtype=torch.bfloat16, device=dev)
blocks = torch.randn(B, 14, 14, Cc, device=dev).bfloat16()
sh = _lib.stream_handle(dev)


def t(fn, n=200):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / n * 1e3


gat = lambda src: _lib.check(lib.sbn_gather(src.data_ptr(), _lib.SBN_BF16, Cc, C.byref(g), idx.rows.data_ptr(),  # noqa: E731
                                            idx.count_dev.data_ptr(), B, 0, stack.data_ptr(), sh), "g")
sca = lambda dst: _lib.check(lib.sbn_scatter(blocks.data_ptr(), _lib.SBN_BF16, Cc, C.byref(g), idx.rows.data_ptr(),  # noqa: E731
                                             idx.count_dev.data_ptr(), B, 0, 0, dst.data_ptr(), sh), "s")
rb = B * 256 * Cc * 2
wb = B * 196 * Cc * 2
for name, fn, byts in (("gather dev", lambda: gat(dx), rb), ("gather host", lambda: gat(hx), rb),
                       ("scatter dev", lambda: sca(dx), wb), ("scatter host", lambda: sca(hx), wb)):
    us = t(fn)
    print(f"{name:14s} {us:8.1f} us  {byts / us / 1e3:6.2f} GB/s  ({byts / 1e6:.2f} MB)")
full = torch.empty_like(dx)
print(f"H2D full frame  {t(lambda: full.copy_(hx, non_blocking=True)):8.1f} us (20.5 MB)")
print(f"D2H full frame  {t(lambda: hx.copy_(full, non_blocking=True)):8.1f} us (20.5 MB)")
