"""Config-3 conv: mask-fused single kernel (sparse_conv_masked_into) vs reduce_mask + conv
(sparse_conv_into) in CUDA graphs, same process."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200.layers import sparse_conv_into, sparse_conv_masked_into

dev = torch.device("cuda", 0)
H, W, C = 800, 700, 128
xs = [torch.randn(1, H, W, C, device=dev).bfloat16() for _ in range(4)]
rng = np.random.default_rng(3)
fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, C, C)) / 34).astype(np.float32)).bfloat16(),
                  torch.from_numpy(rng.standard_normal(C).astype(np.float32)).bfloat16())
p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, C)
out = torch.zeros_like(xs[0])


def timed(fn, reps=40):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(2)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn(reps)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.replay()
        b.record(s)
        b.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for blk in (16, 8):
    spec = P.compute_block_spec((1, H, W, C), p, (blk, blk))
    for d in (0.1, 0.5, 1.0):
        mk = P.synth_mask_topleft((1, H, W), 1 - d).cuda()
        t2 = timed(lambda k: [sparse_conv_into(xs[i % 4], out, fb, p, spec, P.reduce_mask(mk, spec)) for i in range(k)])
        t1 = timed(lambda k: [sparse_conv_masked_into(xs[i % 4], out, mk.data, fb, p, spec) for i in range(k)])
        idx = P.reduce_mask(mk, spec)
        t0 = timed(lambda k: [sparse_conv_into(xs[i % 4], out, fb, p, spec, idx) for i in range(k)])
        print(f"block {blk} density {d}: fused {t1:6.1f} us   reduce_mask+conv {t2:6.1f} us   conv only {t0:6.1f} us", flush=True)
