"""Per-CTA %globaltimer timeline of the resident-weight CTA-pair conv (config 3, 16x16
blocks), mask-fused path and list path: entry -> pdl -> list known -> first chunk landed ->
last MMA issued -> last epilogue done -> exit, relative to the earliest entry (us)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200 import _lib  # noqa: E402
from paper_1801_02108_b200.layers import sparse_conv_into, sparse_conv_masked_into  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
H, W, C = 800, 700, 128
rng = np.random.default_rng(3)
x = torch.randn(1, H, W, C, device=dev).bfloat16()
fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, C, C)) / np.sqrt(9 * C)).astype(np.float32)).bfloat16(),
                  torch.from_numpy(rng.standard_normal(C).astype(np.float32)).bfloat16())
p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, C)
spec = P.compute_block_spec((1, H, W, C), p, (16, 16))
names = ["entry", "pdl", "list", "chunk0", "lastmma", "epi_done", "exit"]
for d in [float(v) for v in os.environ.get("DENS", "0.1,1.0").split(",")]:
    mk = P.synth_mask_topleft((1, H, W), 1 - d).cuda()
    idx = P.reduce_mask(mk, spec)
    o = torch.zeros_like(x)
    for mode in ("masked", "list"):
        fn = (lambda: sparse_conv_masked_into(x, o, mk.data, fb, p, spec)) if mode == "masked" else \
             (lambda: sparse_conv_into(x, o, fb, p, spec, idx))
        for _ in range(3):
            fn()
        buf = torch.zeros(4096 * 8, dtype=torch.int64, device=dev)
        torch.cuda.synchronize()
        lib.sbn_debug_set_trace(buf.data_ptr())
        fn()
        torch.cuda.synchronize()
        lib.sbn_debug_set_trace(None)
        tt = buf.view(-1, 8).cpu().numpy()
        t = tt[2048:2048 + 1024]
        sub = tt[3072:][: len(t)]
        keep = t[:, 0] > 0
        t, sub = t[keep].astype(np.float64), sub[keep].astype(np.float64)
        t0 = t[:, 0].min()
        print(f"density {d} {mode}: {len(t)} CTAs, B={int(t[0, 7])}, span entry->last exit {(t[:, 6].max() - t0) / 1e3:.2f} us")
        for i, nm in enumerate(names):
            col = t[:, i]
            col = col[col > 0]
            if len(col):
                r = (col - t0) / 1e3
                print(f"   {nm:>9}: min {r.min():6.2f}  med {np.median(r):6.2f}  max {r.max():6.2f}")
