"""Config-3 conv, 16x16 blocks: the resident-weight CTA-pair kernel vs the single-CTA
double-buffered kernel (SBN_DEBUG_CONV_NO_RESIDENT), CUDA-graph timings of the whole
sparse_conv2d path (mask fused) and of the conv on a given list, plus the agreement of the
two outputs (different fp32 accumulation order: close, not bit-identical)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1801_02108_b200 as P  # noqa: E402
from paper_1801_02108_b200 import _lib  # noqa: E402
from paper_1801_02108_b200.layers import sparse_conv_into, sparse_conv_masked_into  # noqa: E402

NO_RES = 2048
lib = _lib.load()
dev = torch.device("cuda", 0)
Hc, Wc, Cc = 800, 700, 128
rng = np.random.default_rng(3)
xs = [torch.randn(1, Hc, Wc, Cc, device=dev).bfloat16() for _ in range(8)]
fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, Cc, Cc)) / np.sqrt(9 * Cc)).astype(np.float32)).bfloat16(),
                  torch.from_numpy(rng.standard_normal(Cc).astype(np.float32)).bfloat16())
p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, Cc)
T = lambda fn: bench._timed_graph(torch, bench.time_graph, fn, 40) * 1e3  # noqa: E731
spec = P.compute_block_spec((1, Hc, Wc, Cc), p, (16, 16))
dens = [float(d) for d in os.environ.get("DENS", "0.05,0.1,0.2,0.3,0.5,1.0").split(",")]
VARIANTS = [("db", NO_RES), ("pair_res", 0)] + [(f"flags{v}", int(v)) for v in os.environ.get("EXTRA", "").split(",") if v]
ROUNDS = int(os.environ.get("ROUNDS", 1))
for d in dens:
    mk = P.synth_mask_topleft((1, Hc, Wc), 1 - d).cuda()
    idx = P.reduce_mask(mk, spec)
    res = {}
    for name, fl in VARIANTS * ROUNDS:
        old = lib.sbn_debug_set_flags(fl)
        try:
            o1 = torch.zeros_like(xs[0])
            sparse_conv_masked_into(xs[0], o1, mk.data, fb, p, spec)
            o2 = torch.zeros_like(xs[0])
            sparse_conv_into(xs[0], o2, fb, p, spec, idx)
            torch.cuda.synchronize()
            t_all = T(lambda k: [sparse_conv_masked_into(xs[i % 8], o1, mk.data, fb, p, spec) for i in range(k)])
            t_conv = T(lambda k: [sparse_conv_into(xs[i % 8], o2, fb, p, spec, idx) for i in range(k)])
        finally:
            lib.sbn_debug_set_flags(old)
        if name in res:  # min over rounds
            t_all, t_conv = min(t_all, res[name][2]), min(t_conv, res[name][3])
        res[name] = (o1, o2, t_all, t_conv)
    a, b = res["db"], res["pair_res"]
    extra = "; ".join(f"{k} path {v[2]:.1f} / conv {v[3]:.1f}" for k, v in res.items() if k.startswith("flags"))
    same_path = torch.equal(b[0], b[1])
    diff = (a[0].float() - b[0].float()).abs()
    rel = (diff.norm() / a[0].float().norm()).item()
    nb = idx.count
    fl = nb * 2 * 14 * 14 * 9 * Cc * Cc
    print(f"density {d}: blocks {nb}: db path {a[2]:.1f} / conv {a[3]:.1f} us; pair_res path {b[2]:.1f} / conv {b[3]:.1f} us "
          f"({fl / (b[2] * 1e-6) / 1e12:.0f} TF/s path); masked==list {same_path}; rel diff vs db {rel:.2e}, "
          f"max {diff.max().item():.3g}; {extra}", flush=True)
