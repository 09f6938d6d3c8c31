"""Small workload for compute-sanitizer (memcheck / racecheck / initcheck /
synccheck): every kernel family of the engine runs at least once --
the fp32 step (single + paired, station + tracking + DR, band kernel and its
tail), the persistent TMA-ring paired kernel, the host-ABI zero-copy (mapped)
and staged-copy steps, reset / observe / pack / PD kernels, the fp64 engine,
and the fused rollout (tcgen05 policy kernel, post, GAE).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2410_14117_b200 as uuv  # noqa: E402
from paper_2410_14117_b200 import rollout as R  # noqa: E402


def run():
    torch.cuda.set_device(0)
    mixed = [uuv.default_params(), uuv.bluerov2_params()]
    cases = [
        (uuv.TaskSpec(kind="station_keeping", episode_len=9), uuv.bluerov2_params(), None, 700, {}),
        (uuv.TaskSpec(kind="lemniscate", episode_len=7), uuv.default_params(),
         uuv.default_ranges(per_episode=True), 600, {}),
        (uuv.TaskSpec(kind="circle", episode_len=8), mixed, None, 1300, {"pair": "on"}),
        (uuv.TaskSpec(kind="station_keeping", episode_len=6), mixed, None, 2 * 128 * 148 + 300,
         {"pair": "on", "tma": True}),
    ]
    for spec, veh, ranges, n, dev in cases:
        kw = {"vehicle_mix": [n // 2, n - n // 2]} if isinstance(veh, list) else {}
        cfg = uuv.engine_config_dict(veh, spec, n, 3, 0, ranges, device=0, **kw)
        cfg["device"].update(dev)
        env = uuv.B200EnvBatch(cfg)
        act = env.bench_actions_tensor()
        s = env.states()
        s[: n // 3, 4] = 1.39            # pitch near the band: band kernel + tail paths
        s[: n // 3, 10] = 4.0
        env.set_states(s)
        for _ in range(12):
            env.step_tensors(act)
        env.observe_tensors()
        env.states_tensor()
        act_h = act.double().cpu().numpy()
        for _ in range(3):
            env.step(act_h)                   # host ABI (staged copy)
        env.use_pinned_host_buffers()
        for _ in range(3):
            env.step(act_h)                   # host ABI (zero-copy mapped)
        env.reset_all(5)
        env.stats(clear=True)
        env.close()
    # fp64 engine
    cfg = uuv.engine_config_dict(uuv.default_params(), uuv.TaskSpec(kind="helix", episode_len=5),
                                 300, 1, 0, uuv.default_ranges(per_episode=True),
                                 precision="fp64", device=0)
    env = uuv.B200EnvBatch(cfg)
    a = env.bench_actions_tensor()
    for _ in range(8):
        env.step_tensors(a)
    env.close()
    # fused rollout (tcgen05 policy kernel, normaliser post, GAE)
    env = uuv.batch_create(uuv.TaskSpec(kind="circle"), uuv.bluerov2_params(), None, 256, 1,
                           device=0)
    tc = R.TrainConfig(num_envs=256, horizon=3)
    pol = R.ActorCritic(env.obs_dim, env.action_dim, seed=0).cuda()
    norm = R.RunningNorm(env.obs_dim, "cuda")
    ro = R.Rollout(env, pol, norm, tc, use_graph=False)
    ro.reset(1)
    ro.collect()
    R.gae_fused(ro.rew_buf, ro.val_buf, ro.done_buf, ro.boot_value, 0.99, 0.95)
    torch.cuda.synchronize()
    env.close()
    print("sanitize workload done", flush=True)


if __name__ == "__main__":
    run()
