"""Config-3 conv at 10 %: the whole sparse_conv2d path (reduce_mask + conv) vs the conv with a
precomputed index list vs reduce_mask alone, CUDA graphs (where does the time go?)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200.layers import sparse_conv_into, sparse_conv_masked_into  # noqa: E402

from paper_1801_02108_b200 import _lib  # noqa: E402

_lib.load().sbn_debug_set_flags(int(os.environ.get("SBN_FLAGS", 0)))  # kernel-variant A/B
dev = torch.device("cuda", 0)
Hc, Wc, Cc = 800, 700, 128
rng = np.random.default_rng(3)
xs = [torch.randn(1, Hc, Wc, Cc, device=dev).bfloat16() for _ in range(8)]
fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, Cc, Cc)) / np.sqrt(9 * Cc)).astype(np.float32)).bfloat16(),
                  torch.from_numpy(rng.standard_normal(Cc).astype(np.float32)).bfloat16())
p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, Cc)
out = torch.zeros(1, Hc, Wc, Cc, device=dev).bfloat16()
T = lambda fn: bench._timed_graph(torch, bench.time_graph, fn, 40) * 1e3  # noqa: E731
for blk in [int(b) for b in os.environ.get("BLOCKS", "8,16,32").split(",")]:
    for d in (0.05, 0.1, 0.3):
        spec = P.compute_block_spec((1, Hc, Wc, Cc), p, (blk, blk))
        mk = P.synth_mask_topleft((1, Hc, Wc), 1 - d).cuda()
        idx = P.reduce_mask(mk, spec)
        t_all = T(lambda k: [sparse_conv_masked_into(xs[i % 8], out, mk.data, fb, p, spec) for i in range(k)])
        t_conv = T(lambda k: [sparse_conv_into(xs[i % 8], out, fb, p, spec, idx) for i in range(k)])
        t_rm = T(lambda k: [P.reduce_mask(mk, spec) for _ in range(k)])
        print(f"block {blk} density {d}: path {t_all:.1f} us, conv only {t_conv:.1f} us, reduce_mask {t_rm:.1f} us, "
              f"blocks {idx.count}", flush=True)
