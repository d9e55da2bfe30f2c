"""Host-side sharding of a reconstruction job over ranks (one process per GPU).

The path has no exchange step for one image: a batch of
independent frames (BASELINE.json configs[4], the real-time batch) is split
into contiguous frame ranges, one per rank, each reconstructed by its own plan
with no collective on the data path; a single image is replicated.  Timing
across ranks is the max of the per-rank device times.
"""
from __future__ import annotations


def frame_range(n_frames: int, rank: int, world: int):
    """Contiguous, balanced [lo, hi) frame range of ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_frames, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of ``value`` over the ranks of the default process group (or the
    value itself when not distributed)."""
    if dist is None or not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
