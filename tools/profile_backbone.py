"""Eager config-4 backbone (sparse), for ncu launch lists: one warm-up pass, then one
profiled pass between cudaProfilerStart/Stop.
    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python tools/profile_backbone.py [frames] [density]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200 import perf  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dens = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2
sparse = not (len(sys.argv) > 3 and sys.argv[3] == "dense")
dev = torch.device("cuda", 0)
hh, ww, cin = perf.DETECTOR_INPUT
bb = P.build_backbone(perf.detector_stage_configs(), np.random.default_rng(4))
x = P.Tensor4D(torch.randn(frames, hh, ww, cin, device=dev).bfloat16())
mk = np.concatenate([P.synth_mask_blobs((1, hh, ww), 1.0 - dens, s).numpy() for s in range(frames)])
mask = P.BinaryMask(torch.from_numpy(mk).to(dev), validate=False)
P.run_backbone(bb, x, mask, sparse=sparse)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
P.run_backbone(bb, x, mask, sparse=sparse)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
