"""Multi-process (world_size 2, gloo, CPU) check of the batch-sharding plumbing: per-rank
local index lists merged in rank order equal the global reduce_mask output."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1801_02108_b200.shard import merge_index_lists, shard_bounds


def test_shard_bounds_cover_exactly():
    for n in (1, 7, 64, 65):
        for world in (1, 2, 3, 8):
            if world > n:
                continue
            spans = [shard_bounds(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_frames, q):
    """CPU-only plumbing check (no GPU here): the per-rank index lists come from the oracle
    as a stand-in for the device reduce_mask; tests/test_gpu_shard.py runs the same
    two-rank flow with the CUDA reduce_mask / backbone on cuda:0."""
    from types import SimpleNamespace as NS

    import torch.distributed as dist
    from oracle import sbnet_oracle as O
    from paper_1801_02108_b200.shard import ShardedBackbone
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    masks = (rng.random((n_frames, 40, 36)) < 0.02).astype(np.uint8)
    sb = ShardedBackbone(None, n_frames)  # rank / world from the process group
    assert (sb.rank, sb.world) == (rank, world)
    assert (sb.lo, sb.hi) == shard_bounds(n_frames, rank, world)
    geos = [O.unit_geometry(40, 36, (10, 10)), O.unit_geometry(40, 36, (6, 6))]
    local = [NS(indices=NS(entries=O.reduce_mask(masks[sb.lo:sb.hi], g))) for g in geos]
    merged = sb.index_lists(local)
    ok = all(np.array_equal(mg, O.reduce_mask(masks, g)) for mg, g in zip(merged, geos))
    q.put((rank, bool(ok), len(merged[0])))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_index_lists_merge_to_global_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 7, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert all(n > 0 for _, _, n in res)


def test_merge_index_lists_offsets():
    a = np.array([[0, 1, 2], [1, 0, 0]])
    b = np.array([[0, 3, 3]])
    m = merge_index_lists([a, b], [0, 2])
    assert m.tolist() == [[0, 1, 2], [1, 0, 0], [2, 3, 3]]
