"""Host (numpy) counter RNG, bit-identical to the device one and to the
reference (pkg/src/uuvsim/rng.py:26-53).  Used only to build host-side bench
action matrices for the host-ABI path; the device path draws on the GPU."""

from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
PURPOSE_SALT = np.uint64(0x632BE59BD9B4E019)
PURPOSE_PARAMS, PURPOSE_RESET, PURPOSE_BENCH = 0, 1, 2


def mix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def draw_u64(seed, stream, purpose, counter) -> np.ndarray:
    with np.errstate(over="ignore"):
        h = mix64(np.asarray(seed, dtype=np.uint64))
        h = mix64(h ^ (np.asarray(stream, dtype=np.uint64) + GOLDEN))
        h = mix64(h ^ (np.asarray(purpose, dtype=np.uint64) + PURPOSE_SALT))
        return mix64(h ^ np.asarray(counter, dtype=np.uint64))


def u01(bits: np.ndarray) -> np.ndarray:
    return (bits >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def bench_actions(seed: int, num_envs: int, n_act: int, env_offset: int = 0) -> np.ndarray:
    e = np.arange(env_offset, env_offset + num_envs, dtype=np.uint64)[:, None]
    j = np.arange(n_act, dtype=np.uint64)[None, :]
    u = u01(draw_u64(np.uint64(int(seed) & (2**64 - 1)), e, PURPOSE_BENCH, j))
    return -1.0 + (1.0 - -1.0) * u
