"""Warm timing of the config-4 stage projections: tcgen05 dense conv vs cuDNN (+bias)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200.ops import dense_conv_nhwc, projection_conv  # noqa: E402

dev = torch.device("cuda", 0)
for (h, w, cin, cout) in ((800, 700, 32, 96), (400, 350, 96, 192), (200, 175, 192, 256), (100, 88, 256, 384)):
    x = torch.randn(8, h, w, cin, device=dev).bfloat16()
    f = P.FilterBank(torch.randn(3, 3, cin, cout).bfloat16() * 0.05, torch.randn(cout).bfloat16())
    p = P.ConvParams((3, 3), (2, 2), P.Padding.SAME, cout)
    wd, bd = f.device_tensors(torch.bfloat16, dev)

    def t(fn, n=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / n * 1e3
    ours = t(lambda: projection_conv(x, f, p))
    cud = t(lambda: dense_conv_nhwc(x, wd, bd, (2, 2), (1, 1)))
    fl = 2 * 8 * (h // 2) * (w // 2) * 9 * cin * cout
    print(f"{cin:4d}->{cout:4d} at {h}x{w}: tcgen05 {ours:7.1f} us ({fl / ours / 1e6:6.0f} TF/s)   cuDNN+bias {cud:7.1f} us")
