"""Config-4 backbone (8 frames, 20 % blobs) and the paper's Table-2 unit chains at block 32
under the current build: used to A/B SBN_WIDE_MAX_ROWS (168: wide unit for b <= 18; 200:
b <= 35)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200.layers import residual_unit_algo, residual_unit_into  # noqa: E402

dev = torch.device("cuda", 0)
tag = sys.argv[1] if len(sys.argv) > 1 else ""
bb = bench.run_backbone_leg(P, torch, dev, bench.time_graph, frames=8, density=0.2, reps=10, per_stage=True, dense=False)
if bb:
    print(tag, "backbone ms", bb["sparse_ms"], [s["sparse_ms"] for s in bb["stages"]], flush=True)
rng = np.random.default_rng(0)
for name, units, h, w, c, _ in bench.PAPER_TABLE2:
    x = torch.randn(1, h, w, c, device=dev).bfloat16()
    u = P.random_unit_params(rng, c, c // 2)
    mk = P.synth_mask_topleft((1, h, w), 0.9).cuda()
    spec = P.unit_spec((1, h, w, c), (32, 32))
    algo = residual_unit_algo(torch.bfloat16, u, spec)
    if algo != "tcgen05":
        print(tag, name, "block 32:", algo, flush=True)
        continue
    idx = P.reduce_mask(mk, spec)
    g, st = bench.time_graph(torch, lambda k: [residual_unit_into(x, x, u, spec, idx) for _ in range(k)], 20, 2, soak_s=0.05)
    with torch.cuda.stream(st):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); g.replay(); b.record(st); b.synchronize()
    print(tag, name, "block 32 unit", round(a.elapsed_time(b) / 20 * 1e3, 1), "us", flush=True)
