"""Host-side cost of the public host-frame call vs its GPU time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1801_02108_b200 as P  # noqa: E402

H, W, Cc, M = 400, 400, 64, 32
u = P.random_unit_params(np.random.default_rng(0), Cc, M)
hx = [torch.randn(1, H, W, Cc).bfloat16().pin_memory() for _ in range(4)]
hm = [P.BinaryMask(P.synth_mask_blobs((1, H, W), 0.9, f).data.pin_memory(), validate=False) for f in range(4)]
ss = [torch.cuda.Stream(), torch.cuda.Stream()]
for i in range(20):
    with torch.cuda.stream(ss[i % 2]):
        P.sparse_residual_unit(P.Tensor4D(hx[i % 4]), hm[i % 4], u, (16, 16), inplace=True, blocking=False)
torch.cuda.synchronize()
n = 400
t0 = time.perf_counter()
for i in range(n):
    with torch.cuda.stream(ss[i % 2]):
        P.sparse_residual_unit(P.Tensor4D(hx[i % 4]), hm[i % 4], u, (16, 16), inplace=True, blocking=False)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {(t1 - t0) / n * 1e6:.1f} us/call, wall incl. drain {(t2 - t0) / n * 1e6:.1f} us/call")
import cProfile, pstats  # noqa: E401,E402
pr = cProfile.Profile()
pr.enable()
for i in range(200):
    with torch.cuda.stream(ss[i % 2]):
        P.sparse_residual_unit(P.Tensor4D(hx[i % 4]), hm[i % 4], u, (16, 16), inplace=True, blocking=False)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
