"""Eager (non-graph) run of the benchmark step for ncu: warm-up, then a few steps of
reduce_mask + fused unit (in place) on distinct cold frames, then the dense unit.

    ncu --metrics gpu__time_duration.sum --clock-control none python tools/profile_step.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200.layers import residual_unit_into

H, W, C, M = 400, 400, 64, 32
nf = int(os.environ.get("FRAMES", 16))
steps = int(os.environ.get("STEPS", 8))
block = int(os.environ.get("BLOCK", 16))
density = float(os.environ.get("DENSITY", 0.1))
algo = os.environ.get("ALGO", "auto")
dev = torch.device("cuda", 0)
xs = [torch.randn(1, H, W, C, device=dev).bfloat16() for _ in range(nf)]
ms = [P.synth_mask_blobs((1, H, W), 1 - density, f).cuda() for f in range(nf)]
u = P.random_unit_params(np.random.default_rng(0), C, M)
spec = P.unit_spec((1, H, W, C), (block, block))
for f in range(nf):  # warm-up: builds packed weights, workspaces
    residual_unit_into(xs[f], xs[f], u, spec, P.reduce_mask(ms[f], spec), 1, algo)
torch.cuda.synchronize()
for i in range(steps):
    f = i % nf
    residual_unit_into(xs[f], xs[f], u, spec, P.reduce_mask(ms[f], spec), 1, algo)
torch.cuda.synchronize()
if os.environ.get("DENSE", "1") == "1":
    for i in range(2):
        P.dense_residual_unit(P.Tensor4D(xs[i]), u)
    torch.cuda.synchronize()
print("done")
