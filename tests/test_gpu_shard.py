"""Batch sharding on the GPU path (per-rank unit of work = reference
`layers.py:346-353`): two ranks (gloo process group, both on cuda:0 — this run has one
GPU) each run the CUDA reduce_mask + backbone on their shard of ONE global batch through
`ShardedBackbone`; the merged per-stage index lists equal the single-process global
reduce_mask bit for bit, and every rank's outputs equal the matching frames of a
single-process run of the whole batch."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N_FRAMES, H, W = 5, 96, 80


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch(P):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((N_FRAMES, H, W, 8)).astype(np.float32)
    mk = np.concatenate([P.synth_mask_blobs((1, H, W), 0.8, f).numpy() for f in range(N_FRAMES)])
    return x, mk


def _backbone(P):
    cfgs = [P.StageConfig(1, (8, 12, 24), (16, 16), 1, 1), P.StageConfig(2, (24, 24, 48), (12, 12), 2, 2),
            P.StageConfig(1, (48, 32, 64), (8, 8), 4, 2)]
    return P.build_backbone(cfgs, np.random.default_rng(7))


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist

        import paper_1801_02108_b200 as P
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        x, mk = _batch(P)
        sb = P.ShardedBackbone(_backbone(P), N_FRAMES)
        res = sb.run(P.Tensor4D(torch.from_numpy(x)), P.BinaryMask(mk))  # global host batch in
        torch.cuda.synchronize()
        merged = sb.index_lists(res)
        outs = [r.output.data.cpu().numpy() for r in res]
        q.put((rank, sb.lo, sb.hi, [m.tolist() for m in merged], outs, None))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, 0, 0, None, None, repr(e)))


def test_two_ranks_shard_one_batch_on_gpu(cuda_device):
    import torch

    import paper_1801_02108_b200 as P
    from oracle import sbnet_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    assert all(g[5] is None for g in got), [g[5] for g in got]
    # the single-process run of the whole batch
    x, mk = _batch(P)
    ref = P.run_backbone(_backbone(P), P.Tensor4D(torch.from_numpy(x).cuda()), P.BinaryMask(mk))
    assert [(g[1], g[2]) for g in got] == [P.shard_bounds(N_FRAMES, r, 2) for r in range(2)]
    for rank, lo, hi, merged, outs, _ in got:
        for s, r in enumerate(ref):
            assert merged[s] == r.indices.entries.tolist(), (rank, s)
            assert O.rel_err(outs[s], r.output.data[lo:hi].cpu().numpy()) <= 1e-5, (rank, s)
    assert sum(len(m) for m in got[0][3]) > 0
