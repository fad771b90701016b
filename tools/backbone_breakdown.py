"""Warm, graph-timed breakdown of one config-4 backbone pass (8 frames, 20 % blobs): per
stage the projection, the mask (downsample + reduce_mask) and each wide unit."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200 import perf
from paper_1801_02108_b200.layers import residual_unit_into, unit_spec
from paper_1801_02108_b200.ops import projection_conv

dev = torch.device("cuda", 0)
frames, dens = 8, 0.2
hh, ww, cin = perf.DETECTOR_INPUT
bb = P.build_backbone(perf.detector_stage_configs(), np.random.default_rng(4))
x = torch.randn(frames, hh, ww, cin, device=dev).bfloat16()
mk = np.concatenate([P.synth_mask_blobs((1, hh, ww), 1.0 - dens, s).numpy() for s in range(frames)])
mask = P.BinaryMask(torch.from_numpy(mk).to(dev), validate=False)


def timed(fn, reps=10):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.replay()
        b.record(s)
        b.synchronize()
    return a.elapsed_time(b) / reps * 1e3


t = x
total = 0.0
for si, st in enumerate(bb.stages):
    cfg = st.config
    p = P.ConvParams((3, 3), (cfg.stride, cfg.stride), P.Padding.SAME, cfg.channels[2])
    tp = timed(lambda: projection_conv(t, st.projection, p)) if st.projection is not None else 0.0
    t2 = projection_conv(t, st.projection, p) if st.projection is not None else t
    m2 = P.downsample_mask(mask, cfg.mask_scale)
    spec = unit_spec(tuple(t2.shape), cfg.block_size, halo=1)
    tm = timed(lambda: P.reduce_mask(P.downsample_mask(mask, cfg.mask_scale), spec))
    idx = P.reduce_mask(m2, spec)
    u = st.units[0]
    work = t2.clone()
    tu = timed(lambda: residual_unit_into(work, work, u, spec, idx, 1))
    n_units = len(st.units)
    stage_t = tp + tm + n_units * tu
    total += stage_t
    print(f"stage {si}: {tuple(t2.shape)} blocks {idx.count:5d}  projection {tp:6.1f} us  masks {tm:5.1f} us  "
          f"unit {tu:6.1f} us x {n_units}  = {stage_t:6.1f} us", flush=True)
    t = t2
print(f"sum {total:.1f} us", flush=True)
