"""Config-3 block-16 conv at a few densities under SBN debug flags (A/B of kernel variants):
python tools/conv_variant_time.py [flags...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200 import _lib  # noqa: E402
from paper_1801_02108_b200.layers import sparse_conv_masked_into  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
Hc, Wc, Cc = 800, 700, 128
rng = np.random.default_rng(3)
xs = [torch.randn(1, Hc, Wc, Cc, device=dev).bfloat16() for _ in range(8)]
fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, Cc, Cc)) / np.sqrt(9 * Cc)).astype(np.float32)).bfloat16(),
                  torch.from_numpy(rng.standard_normal(Cc).astype(np.float32)).bfloat16())
p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, Cc)
out = torch.zeros(1, Hc, Wc, Cc, device=dev).bfloat16()
blk = int(os.environ.get("BLOCK", 16))
spec = P.compute_block_spec((1, Hc, Wc, Cc), p, (blk, blk))
for flags in [int(f) for f in sys.argv[1:]] or [0]:
    row = []
    for d in (0.05, 0.1, 0.3, 1.0):
        mk = P.synth_mask_topleft((1, Hc, Wc), 1.0 - d).cuda()
        lib.sbn_debug_set_flags(flags)
        t = bench._timed_graph(torch, bench.time_graph, lambda k: [sparse_conv_masked_into(xs[i % 8], out, mk.data, fb, p, spec)
                                                               for i in range(k)], 40)
        lib.sbn_debug_set_flags(0)
        row.append(f"{d}: {t * 1e3:.1f} us")
    print("flags", flags, "block", blk, " | ".join(row), flush=True)
