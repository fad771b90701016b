"""The paper's layerwise Tables 1-2 re-measured on this GPU: the same
leg bench.py runs (`paper_tables`), standalone.
    python tools/paper_tables.py [sparsity]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1801_02108_b200 as P  # noqa: E402

sp = float(sys.argv[1]) if len(sys.argv) > 1 else 0.9
r = bench.run_paper_tables(P, torch, torch.device("cuda", 0), bench.time_graph, sp)
print(json.dumps(r, indent=1))
