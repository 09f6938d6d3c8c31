"""Drop-in proof on the GPU (SURVEY §4 test (6)): the reference's OWN ctypes
binding (``NativeEnvBatch``, reached through ``uuvsim.batch_create(...,
backend="native")`` with ``UUVSIM_CORE_LIB`` pointing at this repo's
libuuvsim_core.so) steps the B200 engine, and the result is compared with the
reference's pure-Python ``PyEnvBatch`` on the same seeds.

The reference package is imported from ``baseline/_ref`` (the offline install
this repo ships to the GPU box) or, in the build container,
from /root/reference/pkg/src.  Gate: termination masks bit-exact every step;
rewards and states within the documented free-running drift bound (2e-4,
DESIGN.md §6) for envs that never entered the pitch band; reset states equal
fp32 of the reference's fp64 draw.
"""

from __future__ import annotations

import importlib
import os
import sys
from pathlib import Path

import numpy as np
import pytest

from tests import parity as P

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2410_14117_b200" / "_lib" / "libuuvsim_core.so"


def _reference():
    for cand in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (cand / "uuvsim" / "__init__.py").is_file():
            os.environ["UUVSIM_CORE_LIB"] = str(LIB)
            if str(cand) not in sys.path:
                sys.path.insert(0, str(cand))
            mod = importlib.import_module("uuvsim")
            assert Path(mod.__file__).resolve().is_relative_to(cand.resolve())
            return mod
    pytest.skip("reference package not installed (baseline/_ref)")


@pytest.mark.parametrize("kind,dr,m,steps", [("station_keeping", False, 96, 60),
                                             ("lemniscate", True, 64, 45)])
def test_reference_native_binding_steps_b200_engine(kind, dr, m, steps):
    uuvsim = _reference()
    from uuvsim import _native
    _native._lib_cache.clear()
    assert _native.native_available(), "reference loader did not bind this library"
    spec = uuvsim.TaskSpec(kind=kind, episode_len=30 if dr else 600)
    base = uuvsim.default_params()
    ranges = None
    if dr:
        import dataclasses
        ranges = dataclasses.replace(uuvsim.default_ranges(), per_episode=True)
    nat = uuvsim.batch_create(spec, base, ranges, m, 7, threads=0, backend="native")
    py = uuvsim.batch_create(spec, base, ranges, m, 7, threads=0, backend="python")
    assert nat.backend == "native" and py.backend == "python"
    assert (nat.num_envs, nat.obs_dim, nat.action_dim) == (py.num_envs, py.obs_dim, py.action_dim)
    # reset: fp32 of the reference's fp64 draw, exactly
    assert np.array_equal(nat.states(), P.f32(py.states()))
    act = 0.3 * uuvsim.batch.bench_actions(py)
    ever_band = np.zeros(m, dtype=bool)
    n_dones = 0
    for t in range(steps):
        on, rn, dn = nat.step(act)
        op, rp, dp = py.step(act)
        assert np.array_equal(dn, dp), f"termination mask differs at step {t}"
        n_dones += int(dp.sum())
        sp = py.states()
        ever_band |= np.abs(sp[:, 4]) > P.PITCH_BAND
        keep = ~ever_band
        err = P.abs_err(nat.states()[keep], sp[keep], P.STATE_ANGLES)
        assert float(err.max()) < 2e-4, (t, float(err.max()))
        assert np.all(np.abs(rn[keep] - rp[keep]) < 2e-4)
    assert np.array_equal(nat.step_counts(), py.step_counts())
    if dr:
        assert n_dones >= m          # episode_len 30: every env reset (and redrew its DR record)
    nat.close()
