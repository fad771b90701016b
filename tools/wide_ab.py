"""Wide three-launch unit on 64 config-2 frames (graph-timed): A/B probe for unit_wide.cu
changes; argv[1] labels the run."""
import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1801_02108_b200 as P
from paper_1801_02108_b200 import _lib
from paper_1801_02108_b200.layers import residual_unit_into
dev = torch.device("cuda", 0)
lib = _lib.load(); lib.sbn_debug_set_flags(4 | int(os.environ.get("SBN_FLAGS", "0")))
x = torch.randn(64, 400, 400, 64, device=dev).bfloat16()
mk = P.synth_mask_blobs((64, 400, 400), 0.8, 3).cuda()
spec = P.unit_spec(tuple(x.shape), (16, 16)); idx = P.reduce_mask(mk, spec)
u = P.random_unit_params(np.random.default_rng(0), 64, 32)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3): residual_unit_into(x, x, u, spec, idx)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(10): residual_unit_into(x, x, u, spec, idx)
    g.replay(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); g.replay(); b.record(s); b.synchronize(); ts.append(a.elapsed_time(b) / 10 * 1e3)
print(sys.argv[1], "wide unit 64 frames:", min(ts), "us")
