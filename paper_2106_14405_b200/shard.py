"""Environment sharding across GPUs.

Environments are independent, so data parallelism is a pure partition:
rank r owns global env ids [r*E, (r+1)*E).  Everything an env needs (layout
variant, initial state, action stream) is a function of its global id, so a
shard simulated on any rank -- or alone on one GPU -- is bit-identical.
The step path has no collective; ``reduce_window`` is the only
communication: one all_reduce of episode statistics and of the timing per
measurement window (NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np


def shard_env_ids(rank: int, world: int, envs_per_rank: int) -> np.ndarray:
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return np.arange(rank * envs_per_rank, (rank + 1) * envs_per_rank, dtype=np.int64)


def layout_of(global_ids: np.ndarray, n_layouts: int = 3) -> np.ndarray:
    return (np.asarray(global_ids) % n_layouts).astype(np.int32)


def reduce_window(stats: dict, times_ms: dict, device=None):
    """All-reduce a measurement window: SUM of episode stats, MAX of timings.

    Returns (stats, times) as plain floats; a no-op without an initialised
    process group."""
    import torch
    import torch.distributed as dist

    keys_s, keys_t = sorted(stats), sorted(times_ms)
    s = torch.tensor([float(stats[k]) for k in keys_s], dtype=torch.float64, device=device)
    t = torch.tensor([float(times_ms[k]) for k in keys_t], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return dict(zip(keys_s, s.cpu().tolist())), dict(zip(keys_t, t.cpu().tolist()))
