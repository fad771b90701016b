"""One Table-1 conv (argv: h w c block) through sparse_conv2d's masked path, a few times:
the command profiled by ncu for profiles/r1_table1_*."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200.layers import sparse_conv_masked_into  # noqa: E402

h, w, c, blk = (int(v) for v in sys.argv[1:5])
rng = np.random.default_rng(0)
x = torch.randn(1, h, w, c, device="cuda").bfloat16()
out = torch.zeros_like(x)
fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, c, c)) / np.sqrt(9 * c)).astype(np.float32)).bfloat16(),
                  torch.from_numpy(rng.standard_normal(c).astype(np.float32)).bfloat16())
p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, c)
spec = P.compute_block_spec((1, h, w, c), p, (blk, blk))
mk = P.synth_mask_topleft((1, h, w), 0.9).cuda()
for _ in range(3):
    sparse_conv_masked_into(x, out, mk.data, fb, p, spec)
torch.cuda.synchronize()
print("done")
