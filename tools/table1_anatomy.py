"""Where the time goes in the paper's Table-1 rows (one 3x3 conv, 90 % sparse top-left
mask, N=1): reduce_mask alone, the conv on a precomputed list, the whole
sparse_conv_masked_into path, and an empty graph node for the launch floor (graph-timed)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200.layers import sparse_conv_into, sparse_conv_masked_into  # noqa: E402

dev = torch.device("cuda", 0)
from paper_1801_02108_b200 import _lib  # noqa: E402
_lib.load().sbn_debug_set_flags(int(os.environ.get("SBN_FLAGS", 0)))  # kernel-variant A/B


def timed(fn, reps=200):
    g, st = bench.time_graph(torch, fn, reps, 2, soak_s=0.05)
    with torch.cuda.stream(st):
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record(st)
        g.replay()
        b_.record(st)
        b_.synchronize()
    return a_.elapsed_time(b_) / reps * 1e3


rng = np.random.default_rng(0)
for name, h, w, c, _ in bench.PAPER_TABLE1:
    x = torch.randn(1, h, w, c, device=dev).bfloat16()
    out = torch.zeros_like(x)
    fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, c, c)) / np.sqrt(9 * c)).astype(np.float32)).bfloat16(),
                      torch.from_numpy(rng.standard_normal(c).astype(np.float32)).bfloat16())
    p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, c)
    mk = P.synth_mask_topleft((1, h, w), 0.9).cuda()
    for blk in (8, 16, 32):
        spec = P.compute_block_spec((1, h, w, c), p, (blk, blk))
        idx = P.reduce_mask(mk, spec)
        nb = idx.count
        t_rm = timed(lambda k: [P.reduce_mask(mk, spec) for _ in range(k)])
        t_cv = timed(lambda k: [sparse_conv_into(x, out, fb, p, spec, idx) for _ in range(k)])
        t_all = timed(lambda k: [sparse_conv_masked_into(x, out, mk.data, fb, p, spec) for _ in range(k)])
        print(f"{name} {h}x{w}x{c} block {blk:2d} ({nb:4d} blocks): reduce_mask {t_rm:6.2f}  conv {t_cv:6.2f}  "
              f"masked path {t_all:6.2f} us", flush=True)
