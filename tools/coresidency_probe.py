"""Does the hardware co-schedule 2 tcgen05 unit CTAs per SM?  Barrier-free launch
(two-launch path, out of place) with the grid forced to 2 CTAs/SM; records %smid and
entry time per CTA."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1801_02108_b200 as P
from paper_1801_02108_b200 import _lib
from paper_1801_02108_b200.layers import residual_unit_into
lib = _lib.load()
x = torch.randn(2, 400, 400, 64, device="cuda").bfloat16()
u = P.random_unit_params(np.random.default_rng(0), 64, 32)
mk = P.BinaryMask.full(2, 400, 400).cuda()
spec = P.unit_spec((2, 400, 400, 64), (16, 16))
idx = P.reduce_mask(mk, spec)
out = x.clone()
lib.sbn_debug_set_flags(1)  # single-CTA kernel (grid sized from the computed residency)
residual_unit_into(out, x, u, spec, idx)
torch.cuda.synchronize()
buf = torch.zeros(4096 * 32, dtype=torch.int64, device="cuda")
lib.sbn_debug_set_trace(buf.data_ptr())
residual_unit_into(out, x, u, spec, idx)
torch.cuda.synchronize()
lib.sbn_debug_set_trace(None)
t = buf.view(-1, 32).cpu().numpy()
g = t[t[:, 0] > 0]
print("grid", len(g), "blocks", idx.count)
ent = (g[:, 0] - g[:, 0].min()) / 1e3
sm = g[:, 15]
print("distinct SMs", len(set(sm.tolist())), "max CTAs on one SM", np.bincount(sm.astype(int)).max())
print("entry time quantiles us", np.quantile(ent, [0, 0.25, 0.5, 0.75, 0.9, 1.0]).round(2))
# first-wave CTAs: entry before the earliest CTA finished its first block
first_done = (g[:, 11].min() - g[:, 0].min()) / 1e3
print("earliest first-block completion us", round(first_done, 2), "CTAs entered before it", int((ent < first_done).sum()))
