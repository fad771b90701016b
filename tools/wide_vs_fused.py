"""Fused single-kernel unit vs the wide three-launch unit on config-2 shapes (c=64, m=32,
16x16 blocks) as the number of frames per launch grows."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200 import _lib  # noqa: E402
from paper_1801_02108_b200.layers import residual_unit_into, sparse_residual_unit_into  # noqa: E402

dev = torch.device("cuda", 0)
lib = _lib.load()
MASKED = os.environ.get("MASKED", "1") == "1"  # mask-fused public path (sparse_residual_unit)
DENS = float(os.environ.get("DENSITY", 0.2))
for nf in (1, 2, 3, 4, 6, 8, 16, 64):
    x = torch.randn(nf, 400, 400, 64, device=dev).bfloat16()
    mk = P.synth_mask_blobs((nf, 400, 400), 1 - DENS, 3).cuda()
    spec = P.unit_spec(tuple(x.shape), (16, 16))
    idx = P.reduce_mask(mk, spec)
    res = {}
    for name, flag in (("fused", 8), ("wide", 4)):
        u = P.random_unit_params(np.random.default_rng(0), 64, 32)
        prev = lib.sbn_debug_set_flags(flag)
        try:
            def run():
                if MASKED:
                    sparse_residual_unit_into(x, x, mk.data, u, spec)
                else:
                    residual_unit_into(x, x, u, spec, idx)
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                run()
            b.record()
            b.synchronize()
            res[name] = a.elapsed_time(b) / 20 * 1e3
        finally:
            lib.sbn_debug_set_flags(prev)
    print(f"frames {nf:3d} blocks {idx.count:6d}: fused {res['fused']:8.1f} us   wide {res['wide']:8.1f} us")
