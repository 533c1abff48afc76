"""Multi-GPU plumbing: one process per GPU, environments sharded by contiguous
global index, one collective (the int64[8] episode statistics).

Environments are independent and every Philox counter uses the GLOBAL env
index (R#20), so shard r of G is bit-identical to the corresponding
slice of the unsharded batch and the step path needs no communication.  The
only exchange is the all-reduce of exact integer statistics (NCCL on GPUs,
gloo in the CPU tests) and the max-over-ranks of the timed region.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import torch
import torch.distributed as dist

from .navix import shard_range


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    n_total: int
    begin: int
    end: int

    @property
    def n(self) -> int:
        return self.end - self.begin


def env_rank_world():
    """(rank, world_size, local_rank) from the torchrun environment (defaults: 1 process)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def shard_for(n_total: int, rank: int, world: int) -> Shard:
    b, e = shard_range(n_total, rank, world)
    return Shard(rank, world, n_total, b, e)


def init_process_group(backend: str, device: torch.device | None = None):
    """Initialise the default group if WORLD_SIZE > 1 (torchrun sets MASTER_ADDR/PORT)."""
    rank, world, _ = env_rank_world()
    if world <= 1 or dist.is_initialized():
        return
    kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)


def all_reduce_stats(stats: torch.Tensor) -> torch.Tensor:
    """Sum the int64[8] episode statistics over ranks (exact, order independent)."""
    out = stats.clone()
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(out, op=dist.ReduceOp.SUM)
    return out


def max_over_ranks(x: float, device: torch.device | str = "cpu") -> float:
    """The slowest rank's time (the whole-box step time)."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_over_ranks(x: float, device: torch.device | str = "cpu") -> list[float]:
    """Every rank's value of x, in rank order (per-rank step times)."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return [float(x)]
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [float(v.item()) for v in out]


def mean_legacy_return(stats, max_steps: int, failure_reward: float = -1.0) -> float:
    """Mean episode return in minigrid reward mode from the reduced statistics
    (SURVEY §8c-7): (n_success - 0.9 * sum_success_step / T + failure_reward *
    n_failure) / episodes, evaluated once in binary64 so the reported value is
    identical for any G.  n_failure counts Dynamic-Obstacles collisions
    (reward -1, the default) and GoToDoor's toggle / done away from the target
    (reward 0: pass failure_reward=0)."""
    s = [int(v) for v in stats]
    if s[0] == 0:
        return 0.0
    return (s[2] - 0.9 * s[3] / max_steps + failure_reward * s[5]) / s[0]
