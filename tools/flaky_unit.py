"""Repeat the fused / two-launch / CTA-pair unit variants on one input and count bit
mismatches (used to chase the workspace-aliasing bug fixed by fixed-offset slot words)."""
import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1801_02108_b200 as P
from paper_1801_02108_b200 import _lib
from paper_1801_02108_b200.layers import residual_unit_into
lib = _lib.load()
for density, nframes in [(0.1, 1), (0.5, 2), (1.0, 3)]:
    rng = np.random.default_rng(12)
    x = torch.from_numpy(rng.standard_normal((nframes, 240, 224, 64)).astype(np.float32)).bfloat16().cuda()
    u = P.random_unit_params(rng, 64, 32)
    mk = (P.synth_mask_blobs((nframes, 240, 224), 1.0 - density, 9) if density < 1 else P.BinaryMask.full(nframes, 240, 224)).cuda()
    spec = P.unit_spec(tuple(x.shape), (16, 16))
    for flags in (1, 0):
        old = lib.sbn_debug_set_flags(flags)
        bad = [0, 0, 0]
        for rep in range(20):
            a = P.sparse_residual_unit(P.Tensor4D(x), mk, u, (16, 16)).data
            b = x.clone(); P.sparse_residual_unit(P.Tensor4D(b), mk, u, (16, 16), inplace=True)
            c = x.clone(); residual_unit_into(c, c, u, spec, P.reduce_mask(mk, spec))
            d = x.clone(); residual_unit_into(d, x, u, spec, P.reduce_mask(mk, spec))
            torch.cuda.synchronize()
            bad[0] += not torch.equal(a, b); bad[1] += not torch.equal(a, c); bad[2] += not torch.equal(a, d)
        lib.sbn_debug_set_flags(old)
        print(density, nframes, "flags", flags, "mismatch a!=b_inplace_fused, a!=c_inplace_2launch, a!=d_functional_2launch:", bad, flush=True)
