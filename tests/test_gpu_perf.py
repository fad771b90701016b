"""perf.py on the GPU: the block-size autotuner (reference perf.py:167-195) times every
valid candidate with CUDA events and returns the fastest; invalid candidates are skipped
and an all-invalid list raises like the reference."""
import numpy as np
import pytest
import torch

import paper_1801_02108_b200 as P
from paper_1801_02108_b200 import perf
from paper_1801_02108_b200.errors import GeometryError

pytestmark = pytest.mark.gpu


def test_autotune_block_size_on_gpu(cuda_device):
    conv = P.ConvParams((3, 3), (1, 1), P.Padding.SAME, 64)
    layer = perf.LayerConfig((1, 120, 104, 64), conv, seed=3, dtype=torch.bfloat16)
    mask = P.synth_mask_blobs((1, 120, 104), 0.8, 2)
    chosen, table = perf.autotune_block_size(layer, mask, [(8, 8), (16, 16), (32, 32), (2, 2)], warmup=2, iters=3)
    blocks = [b for b, _ in table]
    assert (2, 2) not in blocks and set(blocks) == {(8, 8), (16, 16), (32, 32)}
    assert all(r.mean_ns > 0 for _, r in table)
    best = min(table, key=lambda t: (t[1].mean_ns, t[0][0] * t[0][1]))[0]
    assert chosen == best
    with pytest.raises(GeometryError):
        perf.autotune_block_size(layer, mask, [(2, 2)], warmup=1, iters=1)
