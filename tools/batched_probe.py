"""Fused unit at several frame counts (config-2 shapes, 10 % / 20 % blobs), graph-timed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200.layers import sparse_residual_unit_into

dev = torch.device("cuda", 0)
u = P.random_unit_params(np.random.default_rng(0), 64, 32)
for nf, d in ((1, 0.1), (2, 0.1), (4, 0.1), (8, 0.1), (8, 0.2)):
    x = torch.randn(nf, 400, 400, 64, device=dev).bfloat16()
    mk = torch.cat([P.synth_mask_blobs((1, 400, 400), 1 - d, f).data for f in range(nf)]).to(dev)
    spec = P.unit_spec(tuple(x.shape), (16, 16))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            sparse_residual_unit_into(x, x, mk, u, spec)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(50):
                sparse_residual_unit_into(x, x, mk, u, spec)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.replay()
        b.record(s)
        b.synchronize()
    us = a.elapsed_time(b) / 50 * 1e3
    print(f"{sys.argv[1] if len(sys.argv) > 1 else ''} frames {nf} density {d}: {us:7.1f} us  {nf / us * 1e6:9.0f} frames/s", flush=True)
