"""Fixed cost of one host-ABI step vs batch size, per host_io mode.

    python tools/e2e_overhead.py
"""
import ctypes
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2410_14117_b200 as uuv  # noqa: E402


def main():
    for n in (32, 512, 4096, 16384):
        row = {"envs": n}
        for mode in ("copy", "mapped"):
            cfg = uuv.engine_config_dict(uuv.bluerov2_params(), uuv.TaskSpec(), n, 0, device=0)
            cfg["device"]["host_io"] = mode
            env = uuv.B200EnvBatch(cfg)
            act_t = torch.empty((n, env.action_dim), dtype=torch.float64, pin_memory=True)
            act = act_t.numpy()
            act[:] = uuv.bench_actions(env)
            lib, h = env._lib, env._handle
            P = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
            args = (h, P(act), act.size, P(env._obs), env._obs.size, P(env._rew), env._rew.size,
                    P(env._done), env._done.size)
            for _ in range(200):
                lib.uuvsim_step(*args)
            best = 1e9
            for _ in range(5):
                t0 = time.perf_counter()
                for _ in range(1000):
                    lib.uuvsim_step(*args)
                best = min(best, (time.perf_counter() - t0) * 1e3)
            row[mode + "_us"] = round(best, 2)
            t0 = time.perf_counter()
            for _ in range(1000):
                env.step(act)
            row[mode + "_api_us"] = round((time.perf_counter() - t0) * 1e3, 2)
            env.close()
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
