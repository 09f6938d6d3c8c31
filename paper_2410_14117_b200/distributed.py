"""Multi-GPU plumbing: one process per GPU, one contiguous env slab per rank.

The env step has no cross-env coupling (reference SPEC.md:347, engine.rs:4-5),
so sharding is data-parallel with no collective on the data path: rank r owns
global envs [offset_r, offset_r + n_r) and every counted RNG stream is keyed
by the GLOBAL env index (``batch.env_offset``), which makes a sharded run
bit-identical to the unsharded one (tests/test_oracle_golden.py,
tests/test_gpu_parity.py::test_sharding_invariance_on_device).

The only collective is the episode-statistics all-reduce: an f64[8] vector
(``STAT_NAMES``) reduced once per rollout window with ``torch.distributed``
(NCCL over NVLink on GPU tensors; gloo for the CPU tests).
"""

from __future__ import annotations

import copy

from .batch import STAT_NAMES


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slab of ``total`` envs for ``rank`` (sizes differ by at most one)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    base, extra = divmod(int(total), int(world))
    n = base + (1 if rank < extra else 0)
    offset = rank * base + min(rank, extra)
    return offset, n


def shard_config(cfg: dict, rank: int, world: int, *, weak: bool = True) -> dict:
    """Per-rank engine config.

    weak=True: every rank gets ``batch.num_envs`` envs (job size grows with N);
    weak=False: ``batch.num_envs`` is the job total, split into slabs.  Either
    way the global offset goes into ``batch.env_offset`` and a mixed-vehicle
    ``batch.vehicle_mix`` describes the whole job: under weak scaling the
    per-vehicle counts (given for one slab's worth of envs) are scaled to the
    grown job, so the vehicle proportions of the job are those of the config.
    """
    c = copy.deepcopy(cfg)
    b = c.setdefault("batch", {})
    n = int(b.get("num_envs", 64))
    base_off = int(b.get("env_offset", 0))
    if weak:
        off, cnt = rank * n, n
        mix = b.get("vehicle_mix")
        if mix:
            total = sum(int(x) for x in mix)
            if total != n:
                raise ValueError(f"batch.vehicle_mix sums to {total}, expected num_envs = {n}")
            b["vehicle_mix"] = [int(x) * world for x in mix]
    else:
        off, cnt = shard_range(n, rank, world)
    b["num_envs"] = cnt
    b["env_offset"] = base_off + off
    return c


def allreduce_stats(stats, group=None):
    """Sum an episode-statistics tensor over ranks in place (NCCL or gloo)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats


def summarize(stats) -> dict:
    """Named statistics plus derived means (mean reward per env-step, mean return)."""
    vals = [float(x) for x in (stats.tolist() if hasattr(stats, "tolist") else stats)]
    d = dict(zip(STAT_NAMES, vals))
    steps = max(d["env_steps"], 1.0)
    n_ep = d["done_truncation"] + d["done_divergence"] + d["done_failure"]
    d["mean_reward"] = d["sum_reward"] / steps
    d["episodes"] = n_ep
    d["mean_episode_return"] = d["sum_episode_return"] / n_ep if n_ep else float("nan")
    d["mean_episode_length"] = d["sum_episode_length"] / n_ep if n_ep else float("nan")
    return d


__all__ = ["shard_range", "shard_config", "allreduce_stats", "summarize"]
