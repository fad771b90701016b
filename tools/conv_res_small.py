"""Small resident-pair conv case (list and mask-fused modes) vs the double-buffered kernel,
for compute-sanitizer runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200 import _lib  # noqa: E402
from paper_1801_02108_b200.layers import sparse_conv_into, sparse_conv_masked_into  # noqa: E402

lib = _lib.load()
rng = np.random.default_rng(5)
n, h, w, c = int(os.environ.get("N", 1)), int(os.environ.get("H", 150)), int(os.environ.get("W", 136)), 128
x = torch.from_numpy(rng.standard_normal((n, h, w, c)).astype(np.float32)).bfloat16().cuda()
fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, c, c)) / np.sqrt(9 * c)).astype(np.float32)).bfloat16(),
                  torch.from_numpy(rng.standard_normal(c).astype(np.float32)).bfloat16())
p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, c)
spec = P.compute_block_spec((n, h, w, c), p, (16, 16))
for d in (0.3, 1.0, 0.0):
    mk = (P.synth_mask_blobs((n, h, w), 1.0 - d, 4) if d < 1 else P.BinaryMask.full(n, h, w)).cuda()
    idx = P.reduce_mask(mk, spec)
    outs = []
    for fl in (2048, 16384):  # single-CTA / resident pair with the one-launch global list
        old = lib.sbn_debug_set_flags(fl)
        o = torch.zeros_like(x)
        sparse_conv_into(x, o, fb, p, spec, idx)
        torch.cuda.synchronize()
        o2 = torch.zeros_like(x)
        sparse_conv_masked_into(x, o2, mk.data, fb, p, spec)
        torch.cuda.synchronize()
        lib.sbn_debug_set_flags(old)
        outs.append((o, o2))
    (a, a2), (b, b2) = outs
    rel = ((a.float() - b.float()).norm() / max(a.float().norm().item(), 1e-9)).item()
    print(f"density {d}: blocks {idx.count}: db list==masked {torch.equal(a, a2)}, res list==masked {torch.equal(b, b2)}, "
          f"rel diff {rel:.2e}", flush=True)
