"""Per-CTA %globaltimer phases of the reduce_mask ranges kernel (N=64 x 800x700, 16x16 unit
blocks): entry -> ticket -> column sums -> flags+scan -> look-back -> compaction (us)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200 import _lib  # noqa: E402

lib = _lib.load()
n, h, w = int(os.environ.get("N", 64)), 800, 700
mk = P.synth_mask_blobs((n, h, w), 0.8, 1).cuda()
spec = P.unit_spec((n, h, w, 8), (16, 16))
for _ in range(5):
    P.reduce_mask(mk, spec)
buf = torch.zeros(8 * 8192, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
lib.sbn_debug_set_trace(buf.data_ptr())
P.reduce_mask(mk, spec)
torch.cuda.synchronize()
lib.sbn_debug_set_trace(None)
t = buf.view(-1, 8).cpu().numpy().astype(np.float64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
print(f"{len(t)} ranges; span {(t[:, 5].max() - t0) / 1e3:.2f} us")
for i, nm in enumerate(["entry", "ticket", "colsum", "scan", "lookback", "compact"]):
    r = (t[:, i] - t0) / 1e3
    print(f"  {nm:>9}: min {r.min():6.2f} med {np.median(r):6.2f} max {r.max():6.2f}")
