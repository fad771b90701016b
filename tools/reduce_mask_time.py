"""Warm, graph-timed reduce_mask at the shapes the hot paths use (config 3: 800x700 with
8/16/32 blocks; config 2: 400x400 / 16; backbone stage masks)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1801_02108_b200 as P

dev = torch.device("cuda", 0)
for (n, h, w, blk, d) in ((1, 800, 700, 16, 0.1), (1, 800, 700, 8, 0.1), (1, 800, 700, 32, 0.1), (1, 400, 400, 16, 0.1),
                          (8, 400, 350, 16, 0.2), (64, 400, 400, 16, 0.2)):
    mk = P.synth_mask_topleft((n, h, w), 1 - d).cuda() if n == 1 else P.synth_mask_blobs((n, h, w), 1 - d, 1).cuda()
    p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, 8)
    spec = P.compute_block_spec((n, h, w, 8), p, (blk, blk))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            P.reduce_mask(mk, spec)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(50):
                P.reduce_mask(mk, spec)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.replay()
        b.record(s)
        b.synchronize()
    print(f"reduce_mask n={n} {h}x{w} block {blk}: {a.elapsed_time(b) / 50 * 1e3:6.2f} us "
          f"({spec.grid_count[0] * spec.grid_count[1] * n} candidates)", flush=True)
