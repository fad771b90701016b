"""bench.py's config-3 conv sweep on its own (python tools/conv_sweep_only.py)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1801_02108_b200 as P  # noqa: E402

r = bench.run_conv_sweep(P, torch, torch.device("cuda", 0), bench.time_graph)
for row in r["rows"]:
    print(row["density"], row["block"], row["blocks"], row["sparse_ms"], row["frac"])
print(json.dumps(r["autotuned_block"]))
