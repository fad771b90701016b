"""Where the CTA-pair conv's MMA issuer waits (clock64 totals per pair, config 3 at 100%)."""
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
lib.sbn_debug_set_flags(int(os.environ.get('FLAGS', 32)))  # 32: CTA-pair variant, 0: single-CTA double-buffered
C, H, W = 128, 800, 700
rng = np.random.default_rng(C)
x = torch.from_numpy(rng.standard_normal((1, H, W, C)).astype(np.float32)).bfloat16().to(dev)
fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, C, C)) / np.sqrt(9 * C)).astype(np.float32)).bfloat16(),
                  torch.from_numpy(rng.standard_normal(C).astype(np.float32)).bfloat16())
p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, C)
spec = P.compute_block_spec((1, H, W, C), p, (16, 16))
for d in (1.0, 0.1):
    mk = P.synth_mask_topleft((1, H, W), 1 - d).cuda()
    idx = P.reduce_mask(mk, spec)
    o = torch.zeros_like(x)
    for _ in range(3):
        sparse_conv_into(x, o, fb, p, spec, idx)
    buf = torch.zeros(4096 * 8, dtype=torch.int64, device=dev)
    torch.cuda.synchronize()
    lib.sbn_debug_set_trace(buf.data_ptr())
    sparse_conv_into(x, o, fb, p, spec, idx)
    torch.cuda.synchronize()
    lib.sbn_debug_set_trace(None)
    t = buf.view(-1, 8).cpu().numpy()
    t = t[t[:, 4] > 0]
    tot = t[:, 0].astype(float)
    print(f"density {d}: {len(t)} issuers, blocks/pair {t[:, 4].mean():.1f}, issuer span {tot.mean() / 1965:.1f} us")
    for i, nm in ((1, "wait window"), (2, "wait acc_empty"), (3, "wait weights")):
        print(f"   {nm:>15}: {t[:, i].mean() / tot.mean() * 100:5.1f} %  ({t[:, i].mean() / 1965:.1f} us)")
