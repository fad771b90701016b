"""CTA-pair (cta_group::2) sparse conv vs the single-CTA double-buffered kernel: bit
identity over block counts / channel widths, then timing on config 3 (16x16 blocks)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200 import _lib
from paper_1801_02108_b200.layers import sparse_conv_into

dev = torch.device("cuda", 0)
lib = _lib.load()
for C, (H, W), d in ((128, (120, 104), 0.3), (64, (200, 176), 0.5), (32, (96, 96), 1.0), (128, (800, 700), 0.1), (128, (800, 700), 1.0)):
    rng = np.random.default_rng(C)
    x = torch.from_numpy(rng.standard_normal((1, H, W, C)).astype(np.float32)).bfloat16().to(dev)
    fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, C, C)) / np.sqrt(9 * C)).astype(np.float32)).bfloat16(),
                      torch.from_numpy(rng.standard_normal(C).astype(np.float32)).bfloat16())
    p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, C)
    spec = P.compute_block_spec((1, H, W, C), p, (16, 16))
    mk = P.synth_mask_topleft((1, H, W), 1 - d).cuda() if H == 800 else P.synth_mask_blobs((1, H, W), 1 - d, 3).cuda()
    idx = P.reduce_mask(mk, spec)
    outs = []
    for flag in (32, 0):
        old = lib.sbn_debug_set_flags(flag)
        try:
            o = torch.zeros_like(x)
            sparse_conv_into(x, o, fb, p, spec, idx)
            torch.cuda.synchronize()
            outs.append(o)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    sparse_conv_into(x, o, fb, p, spec, idx)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(20):
                    sparse_conv_into(x, o, fb, p, spec, idx)
                e1.record(s)
                e1.synchronize()
            t = e0.elapsed_time(e1) / 20 * 1e3
        finally:
            lib.sbn_debug_set_flags(old)
        print(f"C={C} {H}x{W} d={d} blocks={idx.count} {'pair' if flag == 32 else 'single'}: {t:8.1f} us", flush=True)
    same = torch.equal(outs[0], outs[1])
    err = (outs[0].float() - outs[1].float()).abs().max().item()
    print(f"   bit-identical: {same}  max|diff| {err:.3g}", flush=True)
