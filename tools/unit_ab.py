"""A/B of fused-unit builds (SBN_LIB_PATH=... python tools/unit_ab.py OUT.npz [REF.npz]):
config-2 step time per density (CUDA graph of back-to-back in-place steps over a 32-frame
ring, as bench.py) and the result of three chained in-place units on fresh seeded frames,
saved to OUT.npz and compared bit for bit with REF.npz when given."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200.layers import sparse_residual_unit_into  # noqa: E402

from paper_1801_02108_b200 import _lib  # noqa: E402

_lib.load().sbn_debug_set_flags(int(os.environ.get("SBN_FLAGS", 0)))  # kernel-variant A/B
H, W, C, M = 400, 400, 64, 32
u = P.random_unit_params(np.random.default_rng(0), C, M)
spec = P.unit_spec((1, H, W, C), (16, 16))
nf = 32
g = torch.Generator(device="cuda").manual_seed(1)
xs = [torch.randn(1, H, W, C, device="cuda", generator=g).bfloat16() for _ in range(nf)]
outs = {}
for dens in (0.02, 0.1, 0.2, 0.3, 0.5, 1.0):
    if dens >= 1.0:
        masks = [torch.ones((1, H, W), dtype=torch.uint8, device="cuda") for _ in range(nf)]
    else:
        masks = [P.synth_mask_blobs((1, H, W), 1 - dens, f).data.cuda() for f in range(nf)]
    y = torch.randn(1, H, W, C, device="cuda", generator=torch.Generator(device="cuda").manual_seed(7)).bfloat16()
    for r in range(3):
        sparse_residual_unit_into(y, y, masks[r], u, spec)
    outs[f"d{dens}"] = y.float().cpu().numpy()
    t = bench._timed_graph(torch, bench.time_graph, lambda k: [sparse_residual_unit_into(xs[i % nf], xs[i % nf],
                                                                                     masks[i % nf], u, spec)
                                                               for i in range(k)], 2000)
    line = f"density {dens:4.2f}: {t * 1e3:6.2f} us/step"
    if len(sys.argv) > 2:
        ref = np.load(sys.argv[2])[f"d{dens}"]
        line += f"  bit-identical to ref: {bool(np.array_equal(ref, outs[f'd{dens}']))}"
    print(line, flush=True)
np.savez(sys.argv[1], **outs)
