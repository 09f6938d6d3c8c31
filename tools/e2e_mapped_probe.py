"""Mapped host-ABI step at C2: cost of the pointer checks and of the kernel.

    python tools/e2e_mapped_probe.py [mapped|copy] [steps]
"""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2410_14117_b200 as uuv  # noqa: E402
from bench import build_config  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "mapped"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg, _ = build_config("c2", 0, "fp32")
cfg["device"]["host_io"] = mode
env = uuv.B200EnvBatch(cfg)
env.use_pinned_host_buffers()
act_t = torch.empty((env.num_envs, env.action_dim), dtype=torch.float64, pin_memory=True)
act = act_t.numpy()
act[:] = uuv.bench_actions(env)
lib, h = env._lib, env._handle
P = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
args = (h, P(act), act.size, P(env._obs), env._obs.size, P(env._rew), env._rew.size,
        P(env._done), env._done.size)
for _ in range(steps):
    lib.uuvsim_step(*args)
t0 = time.perf_counter()
for _ in range(1000):
    lib.uuvsim_step(*args)
print(mode, "raw us/step", (time.perf_counter() - t0) * 1e3)
cudart = ctypes.CDLL("libcudart.so.12") if False else None
try:
    from cuda.bindings import runtime as rt
except ImportError:
    from cuda import cudart as rt
ptr = act.ctypes.data
t0 = time.perf_counter()
for _ in range(1000):
    rt.cudaPointerGetAttributes(ptr)
print("cudaPointerGetAttributes (python binding) us", (time.perf_counter() - t0) * 1e3)
t0 = time.perf_counter()
for _ in range(1000):
    lib.uuvsim_spec(h, (ctypes.c_uint64 * 4)())
print("trivial ABI call us", (time.perf_counter() - t0) * 1e3)
