"""CTA-0 event timeline of the wide unit kernels (IN / MID / OUT) on a config-4 stage:
per tile, when the A producers started issuing (iss), published the tile's last chunk
(pub), the MMA thread started it (mma), the epilogue saw the accumulator (acc) and
released it (epi); microseconds from the first stamp.  Only the LAST launch's stamps
survive (each launch overwrites), so STAGE_KERNEL picks which of the three is traced.
    python tools/trace_wide.py [stage 2..5] [in|mid|out]
Needs the diagnostics build: tools/build_variant.sh trace -DSBN_TRACE_WIDE, then
SBN_LIB_PATH=tools/bin/trace.so."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200 import _lib, perf  # noqa: E402

stage = int(sys.argv[1]) if len(sys.argv) > 1 else 2
which = sys.argv[2] if len(sys.argv) > 2 else "in"
dev = torch.device("cuda", 0)
cfg = perf.detector_stage_configs()[stage - 2]
c, m = cfg.channels[2], cfg.channels[1]
hh, ww = -(-800 // cfg.mask_scale), -(-700 // cfg.mask_scale)  # downsample_mask rounds up
frames = 8
x = torch.randn(frames, hh, ww, c, device=dev).bfloat16()
mk = np.concatenate([P.synth_mask_blobs((1, 800, 700), 0.8, s).numpy() for s in range(frames)])
mask = P.downsample_mask(P.BinaryMask(torch.from_numpy(mk).to(dev), validate=False), cfg.mask_scale)
u = P.random_unit_params(np.random.default_rng(0), c, m)
spec = P.unit_spec(tuple(x.shape), cfg.block_size)
idx = P.reduce_mask(mask, spec)
from paper_1801_02108_b200.layers import residual_unit_into  # noqa: E402
residual_unit_into(x, x, u, spec, idx)
torch.cuda.synchronize()
lib = _lib.load()
buf = torch.zeros(4096 * 16, dtype=torch.int64, device=dev)
names = ["pub", "mma", "acc", "epi", "iss", "empty", "data"]
order = {"in": 0, "mid": 1, "out": 2}[which]
prev = lib.sbn_debug_set_flags(order << 3)
lib.sbn_debug_set_trace(buf.data_ptr())
residual_unit_into(x, x, u, spec, idx)
torch.cuda.synchronize()
lib.sbn_debug_set_trace(None)
lib.sbn_debug_set_flags(prev)
t = buf.cpu().numpy()[:7 * 64].reshape(7, 64).astype(np.int64)
ntile = int((t[0] > 0).sum())
t0 = t[t > 0].min()
print(f"stage {stage} {which} c={c} m={m} blocks={idx.count}")
print("tile " + " ".join(f"{n:>8s}" for n in names))
for k in range(min(ntile, 40)):
    print(f"{k:4d} " + " ".join(f"{(t[e, k] - t0) / 1e3:8.2f}" if t[e, k] else "       -" for e in range(7)))

cl = buf.cpu().numpy()[1024:1024 + 7 * 64].reshape(7, 64).astype(np.int64)
k0, k1 = 0, min(ntile, 40) - 1
dt = (t[0, k1] - t[0, k0]) / 1e9
dc = cl[0, k1] - cl[0, k0]
print(f"SM clock over the trace: {dc / dt / 1e6:.0f} MHz")

ch = buf.cpu().numpy()[7 * 64:13 * 64].reshape(6, 64).astype(np.int64)
nm = ["iss", "data", "empty", "mma_sees", "pub", "pre_empty"]
print("chunk " + " ".join(f"{n:>9s}" for n in nm))
for c in range(min(40, int((ch[0] > 0).sum()))):
    print(f"{c:4d}  " + " ".join(f"{(ch[e, c] - t0) / 1e3:9.2f}" if ch[e, c] else "        -" for e in range(6)))
