"""Per-phase timeline of the fused tcgen05 unit kernel (config 2) from %globaltimer
stamps (sbn_debug_set_trace).  Prints median phase durations over active CTAs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200 import _lib
from paper_1801_02108_b200.layers import residual_unit_into, sparse_residual_unit_into

H, W, C, M = 400, 400, 64, 32
block = int(os.environ.get("BLOCK", 16))
density = float(os.environ.get("DENSITY", 0.1))
nf = 8
dev = torch.device("cuda", 0)
xs = [torch.randn(1, H, W, C, device=dev).bfloat16() for _ in range(nf)]
ms = [P.synth_mask_blobs((1, H, W), 1 - density, f).cuda() for f in range(nf)]
u = P.random_unit_params(np.random.default_rng(0), C, M)
spec = P.unit_spec((1, H, W, C), (block, block))
lib = _lib.load()
FUSED = os.environ.get("FUSED", "1") == "1"


def run(f):
    if FUSED:
        sparse_residual_unit_into(xs[f], xs[f], ms[f].data, u, spec)
        idx = P.reduce_mask(ms[f], spec)  # only for the block count
        return idx
    idx = P.reduce_mask(ms[f], spec)
    residual_unit_into(xs[f], xs[f], u, spec, idx)
    return idx


for f in range(nf):
    run(f)
torch.cuda.synchronize()
buf = torch.zeros(4096 * 32, dtype=torch.int64, device=dev)
names = ["entry", "prologue", "pdl+count", "loads", "barrier", "staged", "gemm1", "epi1", "gemm2",
         "epi2", "gemm3", "epi3"]
for f in range(4):
    torch.cuda.synchronize()
    buf.zero_()
    lib.sbn_debug_set_trace(buf.data_ptr())
    if FUSED:
        sparse_residual_unit_into(xs[f], xs[f], ms[f].data, u, spec)
    else:
        residual_unit_into(xs[f], xs[f], u, spec, P.reduce_mask(ms[f], spec))
    torch.cuda.synchronize()
    lib.sbn_debug_set_trace(None)
    idx = P.reduce_mask(ms[f], spec)
    t = buf.view(-1, 32).cpu().numpy().astype(np.int64)
    B = idx.count
    act = t[t[:, 11] > 0]  # CTAs that processed a block (2 per block in the CTA-pair variant)
    t0 = act[:, 0].min()
    print(f"frame {f}: B={B}, grid {int((t[:, 0] > 0).sum())} CTAs, active {len(act)}, span {(act[:, 11].max() - t0) / 1e3:.2f} us "
          f"(first entry -> last epi3 end); idle CTAs: {int((t[B:, 0] > 0).sum())}")
    d = np.diff(act[:, :12], axis=1)
    for i in range(11):
        print(f"   {names[i]:>10} -> {names[i + 1]:<10} median {np.median(d[:, i]) / 1e3:6.2f} us  max {d[:, i].max() / 1e3:6.2f}")
    print(f"   entry spread {(act[:, 0].max() - t0) / 1e3:.2f} us")
    for nm, a_, b_ in (("gemm1 issue", 5, 12), ("gemm2 issue", 7, 13), ("gemm3 issue", 9, 14)):
        dd = (act[:, b_] - act[:, a_]) / 1e3
        print(f"   {nm:>12}: median {np.median(dd):.2f} us (issue of all MMAs + commit, thread 0)")
    if FUSED:
        for nm, a_, b_ in (("prologue->mask flags", 1, 12), ("flags->done", 12, 14), ("done->entry", 14, 2)):
            dd = (act[:, b_] - act[:, a_]) / 1e3
            print(f"   {nm:>20}: median {np.median(dd):.2f} us  max {dd.max():.2f}")
