"""Inter-kernel gap of the fused config-2 unit inside a CUDA graph: two consecutive steps
traced into separate buffers (%globaltimer at entry / after griddepcontrol.wait / exit per
CTA).  Shows how much of the step is the kernel and how much the launch hand-off."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200 import _lib
from paper_1801_02108_b200.layers import sparse_residual_unit_into

H, W, C, M = 400, 400, 64, 32
dev = torch.device("cuda", 0)
nf = 4
xs = [torch.randn(1, H, W, C, device=dev).bfloat16() for _ in range(nf)]
u = P.random_unit_params(np.random.default_rng(0), C, M)
spec = P.unit_spec((1, H, W, C), (16, 16))
dens = float(os.environ.get("DENSITY", 0.1))
masks = [P.synth_mask_blobs((1, H, W), 1 - dens, f).data.to(dev) for f in range(nf)]
if os.environ.get("EMPTY"):
    masks = [torch.zeros_like(m) for m in masks]
lib = _lib.load()
K = 3
bufs = [torch.zeros(4096 * 32, dtype=torch.int64, device=dev) for _ in range(K)]
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for i in range(4):
        sparse_residual_unit_into(xs[i % nf], xs[i % nf], masks[i % nf], u, spec)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(K):
            lib.sbn_debug_set_trace(bufs[i].data_ptr())
            sparse_residual_unit_into(xs[i % nf], xs[i % nf], masks[i % nf], u, spec)
        lib.sbn_debug_set_trace(None)
    for rep in range(3):
        for b in bufs:
            b.zero_()
        g.replay()
        torch.cuda.synchronize()
ts = [b.view(-1, 32).cpu().numpy().astype(np.int64) for b in bufs]
t0 = min(t[t[:, 0] > 0, 0].min() for t in ts)
for i, t in enumerate(ts):
    live = t[t[:, 0] > 0]
    ent, wait, ext = live[:, 0] - t0, live[:, 16] - t0, live[:, 17] - t0
    print(f"step {i}: {len(live)} CTAs  entry {ent.min()/1e3:7.2f}..{ent.max()/1e3:7.2f}  "
          f"pdl_wait done {wait.min()/1e3:7.2f}..{wait.max()/1e3:7.2f}  exit {ext.min()/1e3:7.2f}..{ext.max()/1e3:7.2f} us")
t = ts[1]
act = t[t[:, 11] > 0]
chain = [(16, "pdl"), (12, "flags"), (14, "done"), (2, "entry"), (18, "loop top"), (3, "loads"), (4, "staged"), (5, "A1"),
         (6, "gemm1"), (20, "clwait"), (21, "epi1 st"), (7, "cl.sync"), (13, "g2 issued"), (8, "gemm2"), (22, "res ld"),
         (9, "epi2"), (23, "gemm3"), (10, "gate"), (11, "epi3"), (17, "exit")]
chain = [c for c in chain if len(act) and (act[:, c[0]] > 0).all()]  # phases this kernel records
if len(act):
    print(f"active CTAs {len(act)}; phase (min / median / max us):")
    for (a_, na), (b_, nb) in zip(chain, chain[1:]):
        d = (act[:, b_] - act[:, a_]) / 1e3
        print(f"  {na:>10} -> {nb:<10} {d.min():6.2f} {np.median(d):6.2f} {d.max():6.2f}")
    tot = (act[:, 17] - act[:, 16]) / 1e3
    print(f"  pdl -> exit total {tot.min():6.2f} {np.median(tot):6.2f} {tot.max():6.2f}")
    slow = act[np.argmax(act[:, 17])]
    print("  slowest CTA:", " ".join(f"{nb}={(slow[b_] - slow[16]) / 1e3:.2f}" for b_, nb in chain[1:]))
    t1 = ts[1]
    prod = t1[t1[:, 19] > 0]
    for nm, a_, b_ in (("flags -> slot atomic", 12, 19), ("slot atomic -> done", 19, 14), ("pdl -> flags", 16, 12)):
        if not len(prod):
            break
        d = (prod[:, b_] - prod[:, a_]) / 1e3
        print(f"  producers with active blocks ({len(prod)}): {nm:>22} {d.min():6.2f} {np.median(d):6.2f} {d.max():6.2f}")
    # consumer wait vs the producer that published its entry is not traced; show entry poll by slot order
    ent = (act[:, 2] - act[:, 16]) / 1e3
    print(f"  pdl -> entry for active CTAs: {ent.min():.2f} {np.median(ent):.2f} {ent.max():.2f}")
