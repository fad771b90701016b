import sys, os, json
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_1801_02108_b200 as P
import numpy as np
dev = torch.device("cuda", 0)
u = P.random_unit_params(np.random.default_rng(0), 64, 32)
mk = P.synth_mask_blobs((1, 400, 400), 0.9, 0).cuda()
print(json.dumps(bench.run_fp32(P, torch, dev, bench.time_graph, u, mk)))
