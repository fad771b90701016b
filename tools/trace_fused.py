"""CTA-0 event timeline of the one-launch wide unit (unit_wide_fused_kernel) on a
config-4 stage (16x16 blocks): per block k of CTA 0, when the loader issued its first
window chunk (load), the first chunk landed (landed), BN1 finished the last chunk (bn),
GEMM1 of both tiles was issued (g1), epilogue 1 published A2 (e1), GEMM2 was issued (g2),
epilogue 2 saw its accumulator (e2a) and released it (e2); microseconds from the first
stamp; g1s / g3 / e1s / e3: GEMM1 issue start, GEMM3 issue, epilogue 1 start, epilogue 3 done.
Needs the diagnostics build: tools/build_variant.sh trace -DSBN_TRACE_WIDE, then
SBN_LIB_PATH=tools/bin/trace.so.
    python tools/trace_fused.py [stage 2|3, or 0 for config-2 frames] [frames]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200 import _lib, perf  # noqa: E402
from paper_1801_02108_b200.layers import residual_unit_into  # noqa: E402

stage = int(sys.argv[1]) if len(sys.argv) > 1 else 2  # 2..3: config-4 stage; 0: config-2 frames (c=64)
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dev = torch.device("cuda", 0)
if stage == 0:
    c, m, hh, ww = 64, 32, 400, 400
    mask = P.synth_mask_blobs((frames, hh, ww), 0.8, 3).cuda()
    blk = (16, 16)
else:
    cfg = perf.detector_stage_configs()[stage - 2]
    c, m = cfg.channels[2], cfg.channels[1]
    hh, ww = -(-800 // cfg.mask_scale), -(-700 // cfg.mask_scale)  # downsample_mask rounds up
    mk = np.concatenate([P.synth_mask_blobs((1, 800, 700), 0.8, s).numpy() for s in range(frames)])
    mask = P.downsample_mask(P.BinaryMask(torch.from_numpy(mk).to(dev), validate=False), cfg.mask_scale)
    blk = cfg.block_size
x = torch.randn(frames, hh, ww, c, device=dev).bfloat16()
u = P.random_unit_params(np.random.default_rng(0), c, m)
spec = P.unit_spec(tuple(x.shape), blk)
idx = P.reduce_mask(mask, spec)
for _ in range(3):
    residual_unit_into(x, x, u, spec, idx)
torch.cuda.synchronize()
lib = _lib.load()
buf = torch.zeros(4096 * 16, dtype=torch.int64, device=dev)
prev = lib.sbn_debug_set_flags(0)
lib.sbn_debug_set_trace(buf.data_ptr())
residual_unit_into(x, x, u, spec, idx)
torch.cuda.synchronize()
lib.sbn_debug_set_trace(None)
lib.sbn_debug_set_flags(prev)
names = ["load", "landed", "bn", "g1", "e1", "g2", "e2a", "e2", "g1s", "g3", "e1s", "e3", "g2e"]
t = buf.cpu().numpy()[:len(names) * 64].reshape(len(names), 64).astype(np.int64)
nb = int((t[0] > 0).sum())
t0 = t[t > 0].min()
print(f"stage {stage} c={c} m={m} blocks={idx.count} (CTA 0: {nb} blocks)")
print("blk  " + " ".join(f"{n:>7s}" for n in names))
for k in range(nb):
    print(f"{k:3d}  " + " ".join(f"{(t[e, k] - t0) / 1e3:7.2f}" if t[e, k] else "      -" for e in range(len(names))))
if nb > 2:
    per = (t[7, nb - 1] - t[7, 1]) / 1e3 / (nb - 2)
    print(f"steady-state period (e2 to e2): {per:.2f} us per block")
