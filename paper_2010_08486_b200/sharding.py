"""Frame-index sharding over the GPUs of one box (one process per GPU).

The detector is a pure function of one frame (reference detector.py:309-314), so
frames are independent units: frame f is owned by rank f mod world_size, every
rank runs its own `Detector` on its own device with pinned H2D copies on its own
streams, and the per-frame blob arrays are gathered on the host in frame order.
There is no collective on the data path (no NCCL traffic proportional to the
frames); `torch.distributed` is only used to gather the small result records.
"""

from __future__ import annotations

import numpy as np

__all__ = ["owned_frames", "gather_frame_results", "ShardedRunner"]


def owned_frames(n_frames: int, rank: int, world_size: int) -> list[int]:
    """Indices of the frames rank `rank` processes (round-robin by frame index)."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError(f"bad rank {rank} / world size {world_size}")
    return list(range(rank, n_frames, world_size))


def gather_frame_results(local: dict, n_frames: int, dst: int = 0, group=None):
    """Host-side gather: `local` maps frame index -> picklable result (e.g. the
    structured record array).  Returns the frame-ordered list on rank `dst`, None
    elsewhere.  Works on any backend (gloo on CPU, nccl on GPUs)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [local[f] for f in range(n_frames)]
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bucket = [None] * world if rank == dst else None
    dist.gather_object(local, bucket, dst=dst, group=group)
    if rank != dst:
        return None
    merged = {}
    for part in bucket:
        overlap = set(merged) & set(part)
        if overlap:
            raise RuntimeError(f"frames {sorted(overlap)} were processed by two ranks")
        merged.update(part)
    missing = [f for f in range(n_frames) if f not in merged]
    if missing:
        raise RuntimeError(f"frames {missing} were not processed by any rank")
    return [merged[f] for f in range(n_frames)]


class ShardedRunner:
    """Runs `detect_fn(list_of_frames) -> list_of_results` on this rank's share of
    a frame sequence and gathers everything on rank 0.

    `detect_fn` is normally `Detector.run_batch`; tests inject a CPU stand-in so
    that the sharding logic is exercised with the gloo backend.
    """

    def __init__(self, detect_fn, rank: int | None = None, world_size: int | None = None):
        import torch.distributed as dist
        if rank is None or world_size is None:
            if dist.is_initialized():
                rank, world_size = dist.get_rank(), dist.get_world_size()
            else:
                rank, world_size = 0, 1
        self.detect_fn = detect_fn
        self.rank, self.world_size = rank, world_size

    def run(self, frame_source, n_frames: int, encode=lambda r: r):
        """frame_source(f) -> host frame f; only owned frames are materialised."""
        mine = owned_frames(n_frames, self.rank, self.world_size)
        frames = [frame_source(f) for f in mine]
        results = self.detect_fn(frames) if frames else []
        local = {f: encode(r) for f, r in zip(mine, results)}
        return gather_frame_results(local, n_frames)


def records_of(result) -> np.ndarray:
    """Compact picklable form of a DetectResult for the gather (structured records)."""
    return np.ascontiguousarray(result.blobs.records)
