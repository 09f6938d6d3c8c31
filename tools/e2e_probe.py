"""Break the host-ABI step (e2e) time into its parts."""
import ctypes, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_2410_14117_b200 as uuv
from bench import build_config

cfg, _ = build_config(sys.argv[1] if len(sys.argv) > 1 else "c2", 0, "fp32")
env = uuv.B200EnvBatch(cfg)
n, A, D = env.num_envs, env.action_dim, env.obs_dim
act = torch.empty((n, A), dtype=torch.float64, pin_memory=True).numpy()
act[:] = uuv.bench_actions(env)
lib, h = env._lib, env._handle
P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
obs, rew, done = env._obs, env._rew, env._done


def t(fn, k=300):
    for _ in range(20):
        fn()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    return (time.perf_counter() - t0) / k * 1e6


print("pinned outputs:", isinstance(env._pinned, list))
print("raw uuvsim_step (C++: H2D+kernel+D2H+sync): %.1f us" %
      t(lambda: lib.uuvsim_step(h, P(act), act.size, P(obs), obs.size, P(rew), rew.size, P(done), done.size)))
print("B200EnvBatch.step (API, with copies):       %.1f us" % t(lambda: env.step(act)))
print("numpy copies only:                          %.1f us" % t(lambda: (obs.copy(), rew.copy(), done.astype(bool))))
pg_obs, pg_rew, pg_done = np.zeros_like(obs), np.zeros_like(rew), np.zeros_like(done)
pg_act = np.array(act)
print("raw uuvsim_step, pageable buffers:          %.1f us" %
      t(lambda: lib.uuvsim_step(h, P(pg_act), act.size, P(pg_obs), obs.size, P(pg_rew), rew.size, P(pg_done), done.size)))
print("device step (graph replay + sync):          %.1f us" % t(lambda: (env.replay_graph(), torch.cuda.synchronize())
                                                             if env.capture_graph(env.bench_actions_tensor(), 1) is None else None, 1) if False else "")
