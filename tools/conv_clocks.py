"""SM clock and throttle reasons while the config-3 sparse conv (100 % density, 16x16
blocks) runs back to back for ~2 s: is the tensor-heavy kernel power-capped?"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200.layers import sparse_conv_into
from bench import ClockSampler

dev = torch.device("cuda", 0)
C, H, W = 128, 800, 700
rng = np.random.default_rng(1)
x = torch.randn(1, H, W, C, device=dev).bfloat16()
fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, C, C)) / 34).astype(np.float32)).bfloat16(),
                  torch.from_numpy(rng.standard_normal(C).astype(np.float32)).bfloat16())
p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, C)
spec = P.compute_block_spec((1, H, W, C), p, (16, 16))
for d in (1.0, 0.1):
    idx = P.reduce_mask(P.synth_mask_topleft((1, H, W), 1 - d).cuda(), spec)
    o = torch.zeros_like(x)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        sparse_conv_into(x, o, fb, p, spec, idx)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(200):
                sparse_conv_into(x, o, fb, p, spec, idx)
        g.replay()
        torch.cuda.synchronize()
        with ClockSampler(0) as clk:
            t_end = time.time() + 2.0
            n = 0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            while time.time() < t_end:
                g.replay()
                n += 1
            e1.record(s)
            e1.synchronize()
    print(f"density {d}: {e0.elapsed_time(e1) / (n * 200) * 1e3:.1f} us/conv, clocks {clk.summary()}", flush=True)
