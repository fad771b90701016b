"""Print the grid the fused unit kernels get (via the trace buffer) for single vs pair."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1801_02108_b200 as P
from paper_1801_02108_b200 import _lib
from paper_1801_02108_b200.layers import sparse_residual_unit_into
lib = _lib.load()
x = torch.randn(1, 400, 400, 64, device="cuda").bfloat16()
u = P.random_unit_params(np.random.default_rng(0), 64, 32)
mk = P.synth_mask_blobs((1, 400, 400), 0.9, 0).cuda()
spec = P.unit_spec((1, 400, 400, 64), (16, 16))
buf = torch.zeros(4096 * 32, dtype=torch.int64, device="cuda")
for flags in (1, 0):
    lib.sbn_debug_set_flags(flags)
    sparse_residual_unit_into(x, x, mk.data, u, spec)
    torch.cuda.synchronize()
    buf.zero_()
    lib.sbn_debug_set_trace(buf.data_ptr())
    sparse_residual_unit_into(x, x, mk.data, u, spec)
    torch.cuda.synchronize()
    lib.sbn_debug_set_trace(None)
    t = buf.view(-1, 32).cpu().numpy()
    print("pair" if flags == 0 else "single", "grid", int((t[:, 0] > 0).sum()), "active", int((t[:, 11] > 0).sum()),
          "span_us", (t[t[:, 11] > 0, 11].max() - t[t[:, 0] > 0, 0].min()) / 1e3,
          "occ", lib.sbn_debug_last_occupancy(0), "clusters", lib.sbn_debug_last_occupancy(1),
          "regs/static/maxdyn/dyn/local", [lib.sbn_debug_last_occupancy(i) for i in range(2, 7)])
