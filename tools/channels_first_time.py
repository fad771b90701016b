"""CHANNELS_FIRST vs CHANNELS_LAST sparse_conv2d / sparse_residual_unit (graph-timed): the
CF path transposes only the active windows (sbn_copy_block_regions_t)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1801_02108_b200 as P

dev = torch.device("cuda", 0)


def timed(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(2):
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


rng = np.random.default_rng(0)
H, W, C = 800, 700, 128
x = torch.randn(1, H, W, C, device=dev).bfloat16()
xcf = P.Tensor4D(x.permute(0, 3, 1, 2).contiguous(), P.Layout.CHANNELS_FIRST)
xcl = P.Tensor4D(x)
fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, C, C)) / 34).astype(np.float32)).bfloat16(),
                  torch.from_numpy(rng.standard_normal(C).astype(np.float32)).bfloat16())
p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, C)
for d in (0.1, 0.3):
    mk = P.synth_mask_topleft((1, H, W), 1 - d).cuda()
    tcl = timed(lambda: P.sparse_conv2d(xcl, mk, fb, p, (16, 16)))
    tcf = timed(lambda: P.sparse_conv2d(xcf, mk, fb, p, (16, 16)))
    print(f"sparse_conv2d 800x700x128 density {d}: channels_last {tcl:7.1f} us   channels_first {tcf:7.1f} us", flush=True)
u = P.random_unit_params(rng, 64, 32)
y = torch.randn(1, 400, 400, 64, device=dev).bfloat16()
ycf = P.Tensor4D(y.permute(0, 3, 1, 2).contiguous(), P.Layout.CHANNELS_FIRST)
ycl = P.Tensor4D(y)
mk = P.synth_mask_blobs((1, 400, 400), 0.9, 0).cuda()
tcl = timed(lambda: P.sparse_residual_unit(ycl, mk, u, (16, 16), inplace=True))
tcf = timed(lambda: P.sparse_residual_unit(ycf, mk, u, (16, 16), inplace=True))
print(f"sparse_residual_unit 400x400x64 10%, in place: channels_last {tcl:7.1f} us   channels_first {tcf:7.1f} us", flush=True)
