"""Config-3 sparse conv (800x700x128 bf16, 3x3 SAME, top-left masks): the single-window
row-shift kernel (conv_tc) vs the strided-TMA tap-GEMM kernel (conv_dense_tc, forced with
SBN_DEBUG_CONV_TMA) per block size and density, CUDA-graph timed, plus cuDNN dense."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200 import _lib
from paper_1801_02108_b200.layers import sparse_conv_into, sparse_conv_algo
from paper_1801_02108_b200.ops import dense_conv_nhwc

dev = torch.device("cuda", 0)
lib = _lib.load()
H, W, C = 800, 700, 128
nfr = 4
xs = [torch.randn(1, H, W, C, device=dev).bfloat16() for _ in range(nfr)]
rng = np.random.default_rng(3)
fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, C, C)) / 34).astype(np.float32)).bfloat16(),
                  torch.from_numpy(rng.standard_normal(C).astype(np.float32)).bfloat16())
p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, C)
out = torch.zeros_like(xs[0])
wd, bd = fb.device_tensors(torch.bfloat16, dev)


def timed(fn, reps=30):
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


dense = timed(lambda k: [dense_conv_nhwc(xs[i % nfr], wd, None, (1, 1), (1, 1)) for i in range(k)])
print(f"dense cuDNN {dense:.1f} us")
for blk in (8, 16, 32):
    spec = P.compute_block_spec((1, H, W, C), p, (blk, blk))
    for d in (0.1, 0.3, 0.5, 1.0):
        mk = P.synth_mask_topleft((1, H, W), 1 - d).cuda()
        idx = P.reduce_mask(mk, spec)
        row = []
        for flag in (0, 16):
            old = lib.sbn_debug_set_flags(flag)
            try:
                algo = sparse_conv_algo(torch.bfloat16, fb, p, spec)
                t = timed(lambda k: [sparse_conv_into(xs[i % nfr], out, fb, p, spec, idx) for i in range(k)])
            finally:
                lib.sbn_debug_set_flags(old)
            row.append(f"{'tma' if flag else 'default'}({algo}) {t:7.1f} us")
        fl = idx.count * 2 * spec.out_block_size[0] * spec.out_block_size[1] * 9 * C * C
        print(f"block {blk:2d} density {d:.1f} blocks {idx.count:5d}: " + "   ".join(row) + f"   ({fl / 1e9:.1f} GFLOP)", flush=True)
