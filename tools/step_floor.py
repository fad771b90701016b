"""Per-step cost of the fused config-2 unit in a CUDA graph as a function of the active
block count: empty mask (fixed cost: launch, prologue, mask scan, hand-off), 1 block,
and the bench's 10% blob masks.  Splits the 18 us step into its fixed and per-block parts."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200.layers import sparse_residual_unit_into

H, W, C, M = 400, 400, 64, 32
dev = torch.device("cuda", 0)
nf = 16
xs = [torch.randn(1, H, W, C, device=dev).bfloat16() for _ in range(nf)]
u = P.random_unit_params(np.random.default_rng(0), C, M)
spec = P.unit_spec((1, H, W, C), (16, 16))


def graph_us(masks, steps=2000):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(4):
            sparse_residual_unit_into(xs[i % nf], xs[i % nf], masks[i % len(masks)], u, spec)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(steps):
                sparse_residual_unit_into(xs[i % nf], xs[i % nf], masks[i % len(masks)], u, spec)
        torch.cuda.synchronize()
        t_end = time.time() + 0.2
        while time.time() < t_end:
            g.replay()
            torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / steps


empty = [torch.zeros(1, H, W, dtype=torch.uint8, device=dev)]
one = torch.zeros(1, H, W, dtype=torch.uint8, device=dev)
one[0, 200, 200] = 1
blobs = [P.synth_mask_blobs((1, H, W), 0.9, f).data.to(dev) for f in range(nf)]
for name, mk in (("empty", empty), ("1 block", [one]), ("10% blobs", blobs)):
    print(f"{name:>10}: {graph_us(mk):6.2f} us/step", flush=True)
