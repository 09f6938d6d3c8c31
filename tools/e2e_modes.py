"""Host-ABI step (e2e) under device.host_io = copy vs mapped, per bench config.

    python tools/e2e_modes.py [c2 c3 ...]

For each config: raw ``uuvsim_step`` time with pinned f64 buffers, the
B200EnvBatch.step API time, and a bit-identity check of obs/rew/done between
the two modes over 50 steps.
"""
import ctypes
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_14117_b200 as uuv  # noqa: E402
from bench import build_config  # noqa: E402


def timeit(fn, k=300):
    for _ in range(20):
        fn()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    return (time.perf_counter() - t0) / k * 1e6


def run(name):
    res = {"config": name}
    outs = {}
    for mode in ("copy", "mapped"):
        cfg, _ = build_config(name, 0, "fp32")
        cfg["device"]["host_io"] = mode
        env = uuv.B200EnvBatch(cfg)
        env.use_pinned_host_buffers()
        n, a_dim = env.num_envs, env.action_dim
        act_t = torch.empty((n, a_dim), dtype=torch.float64, pin_memory=True)
        act = act_t.numpy()
        act[:] = uuv.bench_actions(env)
        lib, h = env._lib, env._handle
        P = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        obs, rew, done = env._obs, env._rew, env._done
        raw = timeit(lambda: lib.uuvsim_step(h, P(act), act.size, P(obs), obs.size, P(rew),
                                             rew.size, P(done), done.size))
        api = timeit(lambda: env.step(act))
        pg_act = np.array(act)
        pg = (np.zeros_like(obs), np.zeros_like(rew), np.zeros_like(done))
        pageable = timeit(lambda: lib.uuvsim_step(h, P(pg_act), act.size, P(pg[0]), obs.size,
                                                  P(pg[1]), rew.size, P(pg[2]), done.size), 100)
        env.reset_all(0)
        trace = []
        for _ in range(50):
            o, r, d = env.step(act)
            trace.append((o.copy(), r.copy(), d.copy()))
        outs[mode] = trace
        res[mode] = {"raw_us": raw, "api_us": api, "pageable_raw_us": pageable,
                     "raw_env_steps_per_s": n / (raw * 1e-6),
                     "api_env_steps_per_s": n / (api * 1e-6), "info_host_io": env.info["host_io"]}
        env.close()
    res["bit_identical"] = all(np.array_equal(x, y) for a, b in zip(outs["copy"], outs["mapped"])
                               for x, y in zip(a, b))
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    for c in (sys.argv[1:] or ["c2", "c4", "c3"]):
        run(c)
