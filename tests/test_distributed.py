"""N>1 path on CPU: world_size-2 gloo processes, sharded slabs, stats all-reduce.

Each rank runs its slab (global env offset) on the oracle -- the GPU engine's
checker, which is bit-identical to it on resets/terminations -- and all-reduces
the episode-statistics vector exactly as bench.py / the training loop do with
NCCL.  The reduced statistics and the concatenated slabs must equal the
single-process run of the whole job.
"""

from __future__ import annotations

import json
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2410_14117_b200 as uuv
from paper_2410_14117_b200.distributed import (allreduce_stats, shard_config, shard_range,
                                               summarize)

STEPS = 90


def _cfg(n):
    spec = uuv.TaskSpec(kind="helix", episode_len=40)
    return uuv.engine_config_dict([uuv.default_params(), uuv.bluerov2_params()], spec, n, 17,
                                  randomization=uuv.default_ranges(per_episode=True),
                                  vehicle_mix=[n // 3, n - n // 3])


def _run_slab(cfg):
    """Step a slab on the oracle; return (stats vector, final states)."""
    from oracle import oracle as orc
    b = orc.OracleBatch(cfg)
    off = cfg["batch"].get("env_offset", 0)
    act = orc.bench_actions(cfg["seed"], b.num_envs, b.action_dim, off)
    st = np.zeros(8)
    ret = np.zeros(b.num_envs)
    for _ in range(STEPS):
        o, r, d, q = b.step(act, with_reason=True)
        ret += r
        st[0] += r.sum()
        st[1] += (q == 0).sum()
        st[2] += (q == 1).sum()
        st[3] += (q == 2).sum()
        st[4] += ret[d].sum()
        st[6] += b.num_envs
        ret[d] = 0.0
    return st, b.states()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = shard_config(_cfg(total), rank, world, weak=False)
    st, states = _run_slab(cfg)
    t = torch.tensor(st, dtype=torch.float64)
    allreduce_stats(t)
    np.save(os.path.join(out_dir, f"states_{rank}.npy"), states)
    if rank == 0:
        np.save(os.path.join(out_dir, "stats.npy"), t.numpy())
        with open(os.path.join(out_dir, "cfg0.json"), "w") as f:
            json.dump(cfg, f)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_covers_job():
    for total, world in ((10, 3), (1 << 20, 8), (7, 7), (5, 2)):
        spans = [shard_range(total, r, world) for r in range(world)]
        assert spans[0][0] == 0
        for (o1, n1), (o2, _) in zip(spans, spans[1:]):
            assert o1 + n1 == o2
        assert sum(n for _, n in spans) == total


def test_shard_config_weak_and_strong():
    c = _cfg(100)
    w = shard_config(c, 3, 4, weak=True)
    assert w["batch"]["num_envs"] == 100 and w["batch"]["env_offset"] == 300
    # weak scaling: the job grows to 400 envs with the config's vehicle proportions
    assert w["batch"]["vehicle_mix"] == [4 * x for x in c["batch"]["vehicle_mix"]]
    s = shard_config(c, 3, 4, weak=False)
    assert s["batch"]["num_envs"] == 25 and s["batch"]["env_offset"] == 75
    assert s["batch"]["vehicle_mix"] == c["batch"]["vehicle_mix"]   # global mix kept


@pytest.mark.timeout(300)
def test_gloo_world2_sharded_stats_match_single_process():
    total, world = 96, 2
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, _free_port(), total, d), nprocs=world,
                           start_method="spawn")
        reduced = np.load(os.path.join(d, "stats.npy"))
        shard_states = np.concatenate([np.load(os.path.join(d, f"states_{r}.npy"))
                                       for r in range(world)])
    whole, whole_states = _run_slab(_cfg(total))
    # integer counts exact, float sums equal up to summation order
    assert np.array_equal(reduced[1:4], whole[1:4])
    assert reduced[6] == whole[6] == total * STEPS
    np.testing.assert_allclose(reduced[[0, 4]], whole[[0, 4]], rtol=1e-12)
    assert np.array_equal(shard_states, whole_states)
    s = summarize(torch.tensor(reduced))
    assert s["episodes"] == reduced[1] + reduced[2] + reduced[3] > 0


def _gpu_worker(rank, world, port, total, out_dir):
    """One rank = one B200EnvBatch slab on cuda:0 (independent slabs, no kernel
    waits on another rank); statistics all-reduced over gloo."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cfg = shard_config(_cfg(total), rank, world, weak=False)
    cfg["device"] = {"index": 0}
    env = uuv.B200EnvBatch(cfg)
    act = env.bench_actions_tensor()
    env.stats(clear=True)
    for _ in range(STEPS):
        env.step_tensors(act)
    torch.cuda.synchronize()
    st = env.stats_tensor().cpu()
    allreduce_stats(st)
    np.save(os.path.join(out_dir, f"states_{rank}.npy"), env.states())
    if rank == 0:
        np.save(os.path.join(out_dir, "stats.npy"), st.numpy())
    env.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(300)
def test_gloo_world2_b200_slabs_match_whole_batch():
    """Sharding invariance on the engine itself: two ranks' env slabs (global
    offsets, global vehicle mix) reproduce the unsharded B200 batch bit for bit,
    and the all-reduced episode statistics equal the whole batch's."""
    total, world = 6000, 2
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_gpu_worker, args=(world, _free_port(), total, d), nprocs=world,
                           start_method="spawn")
        reduced = np.load(os.path.join(d, "stats.npy"))
        shard_states = np.concatenate([np.load(os.path.join(d, f"states_{r}.npy"))
                                       for r in range(world)])
    cfg = _cfg(total)
    cfg["device"] = {"index": 0}
    whole = uuv.B200EnvBatch(cfg)
    act = whole.bench_actions_tensor()
    whole.stats(clear=True)
    for _ in range(STEPS):
        whole.step_tensors(act)
    torch.cuda.synchronize()
    ws = whole.stats_tensor().cpu().numpy()
    assert np.array_equal(shard_states, whole.states())
    names = uuv.STAT_NAMES
    for k, name in enumerate(names):
        if name in ("sum_reward", "sum_episode_return"):
            np.testing.assert_allclose(reduced[k], ws[k], rtol=1e-5)
        else:
            assert reduced[k] == ws[k], name
    assert reduced[names.index("env_steps")] == total * STEPS
    whole.close()
