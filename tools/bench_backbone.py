"""Config-4 backbone leg of bench.py on its own: python tools/bench_backbone.py [frames] [density]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1801_02108_b200 as P  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dens = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2
dev = torch.device("cuda", 0)
print(json.dumps(bench.run_backbone_leg(P, torch, dev, bench.time_graph, frames, dens)), flush=True)
