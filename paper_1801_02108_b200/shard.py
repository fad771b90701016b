"""Batch sharding across GPUs: frames are independent, so N frames are
split into contiguous shards, one process per GPU, with NO collective on the hot path.

Each rank runs reduce_mask / the fused kernels on its own frames with local frame
indices.  Because index lists are ordered frame-major (reference `tiling.py:104`,
`:160`), concatenating the per-rank lists in rank order with the frame index shifted by
the shard offset reproduces the global `reduce_mask` output exactly; `merge_index_lists`
does that, and `gather_index_lists` is the optional off-hot-path verification collective
(all_gather over NCCL or gloo).
"""
from __future__ import annotations

import numpy as np


def shard_bounds(n_frames: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) frame range of `rank`; sizes differ by at most one frame."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(n_frames, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def merge_index_lists(parts, offsets) -> np.ndarray:
    """Concatenate per-rank (B_r, 3) lists (local frame indices) into the global list."""
    out = []
    for e, off in zip(parts, offsets):
        e = np.asarray(e, np.int64).reshape(-1, 3).copy()
        e[:, 0] += off
        out.append(e)
    return np.concatenate(out, axis=0) if out else np.zeros((0, 3), np.int64)


def gather_index_lists(local_entries: np.ndarray, n_frames: int, group=None) -> np.ndarray:
    """All-gather every rank's local list and merge (verification only; not timed)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")
    e = torch.as_tensor(np.asarray(local_entries, np.int64).reshape(-1, 3), device=dev)
    cnt = torch.tensor([e.shape[0]], device=dev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    cap = int(max(int(c.item()) for c in counts))
    pad = torch.zeros((max(cap, 1), 3), dtype=torch.int64, device=dev)
    pad[: e.shape[0]] = e
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    parts = [b[: int(c.item())].cpu().numpy() for b, c in zip(bufs, counts)]
    offsets = [shard_bounds(n_frames, r, world)[0] for r in range(world)]
    del rank
    return merge_index_lists(parts, offsets)
