"""GPU time of each piece of the host-frame unit call, and PCIe duplex overlap."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200 import _lib  # noqa: E402
from paper_1801_02108_b200.layers import _HostFramePlan  # noqa: E402

H, W, Cc, M = 400, 400, 64, 32
dev = torch.device("cuda", 0)
u = P.random_unit_params(np.random.default_rng(0), Cc, M)
hx = [torch.randn(1, H, W, Cc).bfloat16().pin_memory() for _ in range(2)]
hm = P.synth_mask_blobs((1, H, W), 0.9, 0).data.pin_memory()
ss = [torch.cuda.Stream(), torch.cuda.Stream()]
plans = []
for i in range(2):
    with torch.cuda.stream(ss[i]):
        plans.append(_HostFramePlan(u, hx[0].shape, torch.bfloat16, (16, 16), 1, "auto", dev, ss[i]))
        plans[i].run(hx[i], hm)
torch.cuda.synchronize()
lib = _lib.load()


def piece(pl, which, xh):
    gb = C.byref(pl.g)
    if which == "mask":
        pl.md.copy_(hm, non_blocking=True)
    elif which == "rm":
        lib.sbn_reduce_mask(pl.md.data_ptr(), gb, 0, pl.thr, pl.rows.data_ptr(), pl.count.data_ptr(), pl.rmws.data_ptr(), pl.rmws.numel(), pl.sh)
    elif which == "in":
        lib.sbn_copy_block_regions(xh.data_ptr(), pl.stage.data_ptr(), pl.dt, pl.c, gb, pl.rows.data_ptr(), pl.count.data_ptr(), pl.cap, 0, pl.sh)
    elif which == "unit":
        lib.sbn_residual_unit(pl.stage.data_ptr(), pl.dt, pl.c, pl.m, gb, 1, 1, C.byref(pl.up), pl.rows.data_ptr(), pl.count.data_ptr(), pl.cap, pl.stage.data_ptr(), pl.ws.data_ptr(), pl.ws.numel(), pl.algo, pl.sh)
    elif which == "out":
        lib.sbn_copy_block_regions(pl.stage.data_ptr(), xh.data_ptr(), pl.dt, pl.c, gb, pl.rows.data_ptr(), pl.count.data_ptr(), pl.cap, 1, pl.sh)


def timed(fn, n=200):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(ss[0])
    ss[1].wait_stream(ss[0])
    for i in range(n):
        fn(i)
    ss[0].wait_stream(ss[1])
    b.record(ss[0])
    b.synchronize()
    return a.elapsed_time(b) / n * 1e3


for w in ("mask", "rm", "in", "unit", "out"):
    print(f"{w:6s} one stream {timed(lambda i: piece(plans[0], w, hx[0])):7.1f} us")
print(f"in ‖ out (two streams) {timed(lambda i: (piece(plans[0], 'in', hx[0]), piece(plans[1], 'out', hx[1]))):7.1f} us per pair")
print(f"full run, 1 stream   {timed(lambda i: plans[0].run(hx[0], hm)):7.1f} us")
print(f"full run, 2 streams  {timed(lambda i: plans[i % 2].run(hx[i % 2], hm)):7.1f} us")
