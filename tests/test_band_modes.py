"""The fp64 band's ownership protocol gives one answer however
the work is scheduled: the concurrent band kernel on the side stream (default),
the band kernel after the step kernel on one stream, and the step kernel
launched first, with the fp64 vehicle constants in registers or read from the
kernel parameters; inside a CUDA graph as eagerly.  The engines free-run the same tumbling
workloads and must agree bit for bit -- states, observations, rewards,
terminations and the episode statistics -- while each runs hundreds of fp64
band steps.  A race between the two kernels (an env stepped twice, or not at
all) would break the equality at once.
"""

from __future__ import annotations

import numpy as np
import pytest

from tests.test_gpu_parity import _cfg

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_2410_14117_b200 as uuv  # noqa: E402

VARIANTS = {
    "side": {},
    "same_stream": {"band_stream": "same"},
    "step_first": {"band_order": "main_first"},
    "rege_on": {"band_rege": True},     # fp64 vehicle constants in registers (default <= 8,192 envs)
    "rege_off": {"band_rege": False},
}

WORKLOADS = {
    "c2_station_bluerov2": dict(vehicle="bluerov2", n=4096),
    "c5_mixed_pair": dict(mixed=True, n=131072, pair="on"),
    "c3_lemniscate_drep": dict(kind="lemniscate", dr="episode", episode_len=37, n=16384),
}


def _run(cfg, steps, graph):
    env = uuv.B200EnvBatch(cfg)
    act = env.bench_actions_tensor()
    out = None
    if graph:
        out = env.capture_graph(act, n_steps=1)   # the graph's own output buffers
        for _ in range(steps):
            env.replay_graph()
    else:
        for _ in range(steps):
            out = env.step_tensors(act)
    torch.cuda.synchronize()
    res = {"states": env.states(), "steps": env.step_counts(), "stats": env.stats()}
    if out is not None:
        obs, rew, done, reason = out
        res.update(obs=obs.cpu().numpy(), rew=rew.cpu().numpy(), done=done.cpu().numpy(),
                   reason=reason.cpu().numpy())
    env.close()
    return res


@pytest.mark.parametrize("name", list(WORKLOADS))
def test_band_schedules_agree_bit_for_bit(name):
    base = _cfg(**WORKLOADS[name])
    results = {}
    for v, dev in VARIANTS.items():
        cfg = {**base, "device": {**base["device"], **dev}}
        results[v] = _run(cfg, 260, graph=False)
    ref = results["side"]
    assert ref["stats"]["band64_steps"] > 100, "workload never entered the pitch band"
    for v, r in results.items():
        for k in ("states", "steps", "obs", "rew", "done", "reason"):
            assert np.array_equal(r[k], ref[k]), (v, k)
        for k in ("done_truncation", "done_divergence", "done_failure", "env_steps",
                  "band64_steps", "sum_episode_length"):
            assert r["stats"][k] == ref["stats"][k], (v, k, r["stats"][k], ref["stats"][k])
        # reward sums: fp32 warp partials, accumulated in a launch-order-dependent
        # order across the two kernels' slots -- equal to fp32 rounding
        assert abs(r["stats"]["sum_reward"] - ref["stats"]["sum_reward"]) <= \
            1e-6 * abs(ref["stats"]["sum_reward"]), v


def test_band_kernel_inside_a_cuda_graph_matches_eager():
    base = _cfg(vehicle="bluerov2", n=4096)
    eager = _run(base, 260, graph=False)
    graphed = _run(base, 260, graph=True)
    assert eager["stats"]["band64_steps"] > 100
    for k in ("states", "steps", "obs", "rew", "done", "reason"):
        assert np.array_equal(eager[k], graphed[k]), k
    assert eager["stats"]["band64_steps"] == graphed["stats"]["band64_steps"]
