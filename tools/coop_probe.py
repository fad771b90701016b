"""Can the grid-barrier unit kernels be launched cooperatively (cudaLaunchAttributeCooperative,
the driver then guarantees co-residency or refuses the launch)?  For the config-2 fused
in-place unit (CTA-pair, cluster 2) and the single-CTA variant, prints the grid the
launcher computes from the real per-SM limits, what the occupancy API reports, and whether
a cooperative launch of that grid is accepted and produces the same bits."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200 import _lib  # noqa: E402
from paper_1801_02108_b200.layers import sparse_residual_unit_into  # noqa: E402

lib = _lib.load()
COOP, NOPAIR = 64, 1
u = P.random_unit_params(np.random.default_rng(0), 64, 32)
spec = P.unit_spec((1, 400, 400, 64), (16, 16))
for dens, label in ((0.1, "10% blobs"), (1.0, "full mask")):
    mk = (P.synth_mask_blobs((1, 400, 400), 1 - dens, 0) if dens < 1 else P.BinaryMask.full(1, 400, 400)).cuda()
    x0 = torch.randn(1, 400, 400, 64, device="cuda").bfloat16()
    for extra, kname in ((0, "pair"), (NOPAIR, "single")):
        res = {}
        for flags in (extra, extra | COOP):
            lib.sbn_debug_set_flags(flags)
            x = x0.clone()
            try:
                sparse_residual_unit_into(x, x, mk.data, u, spec)
                torch.cuda.synchronize()
                res[flags] = ("ok", x)
            except Exception as e:  # noqa: BLE001
                res[flags] = (f"refused: {e}", None)
            occ = [lib.sbn_debug_last_occupancy(i) for i in range(8)]
            print(f"{label:10s} {kname:6s} coop={bool(flags & COOP)}: {res[flags][0][:120]}; "
                  f"occ(single/SM)={occ[0]} pairs={occ[1]} api_clusters={occ[7]} regs={occ[2]}")
        a, b = res[extra][1], res[extra | COOP][1]
        if a is not None and b is not None:
            print("   bit-identical:", bool(torch.equal(a, b)))
lib.sbn_debug_set_flags(0)
