"""Multi-GPU host logic: batched independent tracks sharded over ranks.

North star (BASELINE.json): "A batch of independent tracks is sharded per GPU
with no communication."  One process per GPU; track i (global index) always
gets run seed `base_seed + i` and observes video `i % n_videos`, whatever
rank it lands on, so every track's trajectory is identical for any GPU count
(the per-track LCG stream is keyed by the seed, the fused kernel's results
do not depend on batching -- tests/test_gpu_fused.py).  The only collectives
are for timing/reporting (barrier, max of elapsed time, gather of
trajectories), none on the data path.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    first: int  # first global track index on this rank
    count: int  # tracks on this rank

    def seeds(self, base_seed: int) -> List[int]:
        return [base_seed + self.first + i for i in range(self.count)]

    def videos(self, n_videos: int) -> List[int]:
        return [(self.first + i) % n_videos for i in range(self.count)]


def shard_tracks(total_tracks: int, world: int, rank: int) -> Shard:
    """Contiguous block partition; the first `total % world` ranks get one extra."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if total_tracks < world:
        raise ValueError(f"{total_tracks} tracks cannot be spread over {world} ranks")
    q, r = divmod(total_tracks, world)
    first = rank * q + min(rank, r)
    return Shard(rank, world, first, q + (1 if rank < r else 0))


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (time-like metrics are the max over ranks)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    import torch

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_trajectories(local, dist=None, device=None):
    """All ranks' (tracks, F, 2) trajectories, concatenated in global track order."""
    import numpy as np

    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, np.asarray(local))
    return np.concatenate(out, axis=0)
