"""reduce_mask A/B: the ranges kernel (several block rows per CTA) vs the one-row-per-CTA
look-back kernel (SBN_DEBUG_ROW_REDUCE_MASK), CUDA-graph timed at the shapes the hot paths
use; the big case also with a rotation of masks larger than L2; indices compared."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200 import _lib  # noqa: E402

lib = _lib.load()
ROW = 8192


def timed(fn, reps=50):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn(0)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(reps):
                fn(i)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.replay()
        b.record(s)
        b.synchronize()
    return a.elapsed_time(b) / reps * 1e3


cases = [(1, 800, 700, 16, 0.1, 1), (1, 800, 700, 8, 0.1, 1), (1, 400, 400, 16, 0.1, 1), (8, 400, 350, 16, 0.2, 1),
         (8, 800, 700, 16, 0.2, 1), (64, 400, 400, 16, 0.2, 1), (64, 800, 700, 16, 0.2, 1), (64, 800, 700, 16, 0.2, 4)]
for (n, h, w, blk, d, rot) in cases:
    masks = [(P.synth_mask_topleft((n, h, w), 1 - d) if n == 1 else P.synth_mask_blobs((n, h, w), 1 - d, k + 1)).cuda()
             for k in range(rot)]
    spec = P.unit_spec((n, h, w, 8), (blk, blk))
    res = {}
    for name, fl in (("row", ROW), ("ranges", 0)):
        old = lib.sbn_debug_set_flags(fl)
        try:
            t = timed(lambda i: P.reduce_mask(masks[i % rot], spec))
            ent = P.reduce_mask(masks[0], spec).entries
        finally:
            lib.sbn_debug_set_flags(old)
        res[name] = (t, ent)
    same = np.array_equal(res["row"][1], res["ranges"][1])
    mb = n * h * w / 1e6
    print(f"n={n} {h}x{w} block {blk} rot {rot} ({mb:.1f} MB/mask, {n * spec.grid_count[0] * spec.grid_count[1]} cand): "
          f"row {res['row'][0]:6.2f} us, ranges {res['ranges'][0]:6.2f} us ({mb * 1e-3 / (res['ranges'][0] * 1e-6):.0f} GB/s), "
          f"same indices {same}", flush=True)
