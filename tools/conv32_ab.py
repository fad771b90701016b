import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
import paper_1801_02108_b200 as P
from paper_1801_02108_b200.layers import sparse_conv_masked_into
dev = torch.device("cuda", 0)
rng = np.random.default_rng(3)
xs = [torch.randn(1, 800, 700, 128, device=dev).bfloat16() for _ in range(4)]
fb = P.FilterBank(torch.from_numpy((rng.standard_normal((3, 3, 128, 128)) / 34).astype(np.float32)).bfloat16(),
                  torch.from_numpy(rng.standard_normal(128).astype(np.float32)).bfloat16())
p = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, 128)
out = torch.zeros(1, 800, 700, 128, device=dev).bfloat16()
res = []
for d in (0.1, 0.5, 1.0):
    mk = P.synth_mask_topleft((1, 800, 700), 1 - d).cuda()
    spec = P.compute_block_spec((1, 800, 700, 128), p, (32, 32))
    ts = []
    for rep in range(3):
        g, st = bench.time_graph(torch, lambda k: [sparse_conv_masked_into(xs[i % 4], out, mk.data, fb, p, spec) for i in range(k)], 40, 2, soak_s=0.05)
        with torch.cuda.stream(st):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st); g.replay(); b.record(st); b.synchronize()
        ts.append(a.elapsed_time(b) / 40 * 1e3)
    res.append(f"{d}: {min(ts):.1f}")
print(sys.argv[1], "block32:", "  ".join(res))
