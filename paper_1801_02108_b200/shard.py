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


def _rank_world(rank, world, group=None):
    if rank is not None and world is not None:
        return rank, world
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


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


class ShardedBackbone:
    """Batch-sharded `run_backbone` (config 5; reference `layers.py:346-353` is the per-rank
    unit of work): a global batch of `n_frames` frames is split into contiguous shards, one
    process per GPU; rank r runs the whole backbone on frames shard_bounds(n_frames, r,
    world) with local frame indices.  Nothing is exchanged on the hot path — frames are
    independent.  `index_lists` (verification only, off the hot path) all-gathers every
    stage's per-rank index list and merges them into the global reduce_mask output.

    rank / world default to the initialised torch.distributed process group (else 0 / 1).
    """

    def __init__(self, backbone, n_frames: int, rank: int | None = None, world: int | None = None,
                 group=None):
        self.backbone = backbone
        self.n_frames = n_frames
        self.group = group
        self.rank, self.world = _rank_world(rank, world, group)
        self.lo, self.hi = shard_bounds(n_frames, self.rank, self.world)

    @property
    def local_frames(self) -> range:
        """Global frame indices this rank owns."""
        return range(self.lo, self.hi)

    def run(self, x, base_mask, **kw):
        """run_backbone on this rank's shard of a GLOBAL batch (Tensor4D + BinaryMask with
        n_frames frames, host or device): the shard is sliced (a view) and moved to the
        current device; other ranks' frames are never touched."""
        from .tensor import Tensor4D
        from .tiling import BinaryMask
        if x.dims[0] != self.n_frames:
            raise ValueError(f"global batch has {x.dims[0]} frames, sharder expects {self.n_frames}")
        xs = Tensor4D.from_nhwc(x.nhwc()[self.lo:self.hi], x.layout)
        ms = None if base_mask is None else BinaryMask(base_mask.data[self.lo:self.hi], validate=False)
        return self.run_local(xs, ms, **kw)

    def run_local(self, x_shard, mask_shard, **kw):
        """run_backbone on frames already restricted to this rank's shard."""
        from .layers import run_backbone
        if x_shard.dims[0] != self.hi - self.lo:
            raise ValueError(f"shard has {x_shard.dims[0]} frames, rank {self.rank} owns {self.hi - self.lo}")
        return run_backbone(self.backbone, x_shard, mask_shard, **kw)

    def index_lists(self, results) -> list[np.ndarray]:
        """Global per-stage index lists (all_gather + merge in rank order)."""
        if self.world == 1:
            return [r.indices.entries for r in results]
        return [gather_index_lists(r.indices.entries, self.n_frames, self.group) for r in results]
