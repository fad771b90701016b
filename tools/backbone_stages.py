"""Sparse config-4 backbone only (no dense legs): whole-backbone and per-stage times from
CUDA graphs, N frames at a density; for A/B runs of compile-time variants
(SBN_LIB_PATH=... SBN_FLAGS=... python tools/backbone_stages.py [frames] [density])."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200 import perf  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dens = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2
dev = torch.device("cuda", 0)
if os.environ.get("SBN_FLAGS"):  # runtime debug flags (e.g. 256: wide unit IN and MID as two launches)
    from paper_1801_02108_b200 import _lib
    _lib.load().sbn_debug_set_flags(int(os.environ["SBN_FLAGS"]))
hh, ww, cin = perf.DETECTOR_INPUT
bb = P.build_backbone(perf.detector_stage_configs(), np.random.default_rng(4))
x = P.Tensor4D(torch.randn(frames, hh, ww, cin, device=dev).bfloat16())
mk = np.concatenate([P.synth_mask_blobs((1, hh, ww), 1.0 - dens, s).numpy() for s in range(frames)])
mask = P.BinaryMask(torch.from_numpy(mk).to(dev), validate=False)
res = P.run_backbone(bb, x, mask)
torch.cuda.synchronize()
out = {"lib": os.environ.get("SBN_LIB_PATH", "default"), "flags": os.environ.get("SBN_FLAGS", "0"), "frames": frames,
       "total_ms": round(bench._timed_graph(torch, bench.time_graph, lambda k: [P.run_backbone(bb, x, mask)
                                                                               for _ in range(k)], 5), 4),
       "stages_ms": []}
inp = x
for st, r in zip(bb.stages, res):
    out["stages_ms"].append(round(bench._timed_graph(torch, bench.time_graph,
                                                     lambda k, st=st, inp=inp: [P.run_stage(st, inp, mask)
                                                                                for _ in range(k)], 5), 4))
    inp = r.output
print(json.dumps(out), flush=True)
