"""Host-side mirror of the reference interface (no GPU needed).

Vehicle data, TaskSpec / RandomizationRanges / VehicleParams validation and
the engine-config document must match what the reference produces for the
same inputs (tests/golden/engine_configs.json and vehicles.json were rendered
by the reference itself, tests/golden/make_golden.py).
"""

from __future__ import annotations

import json
import math
from pathlib import Path

import numpy as np
import pytest

import paper_2410_14117_b200 as uuv
from paper_2410_14117_b200 import _rng, vehicles
from paper_2410_14117_b200.batch import resolve_backend

GOLDEN = Path(__file__).resolve().parent / "golden"


def test_heavy_vehicle_equals_reference_document():
    ref = json.loads((GOLDEN / "vehicles.json").read_text())["bluerov2_heavy"]
    assert vehicles.bluerov2_heavy() == ref


def test_bluerov2_is_valid_six_thruster_vehicle():
    v = uuv.bluerov2_params()
    assert v.n_thrusters() == 6
    d = v.to_dict()
    assert d["weight"] == d["buoyancy"]          # neutrally buoyant like the Heavy file


@pytest.mark.parametrize("case", json.loads((GOLDEN / "engine_configs.json").read_text()))
def test_engine_config_matches_reference(case):
    spec = uuv.TaskSpec.from_dict(case["task_in"])
    rnd = case["randomization_in"]
    ranges = uuv.RandomizationRanges.from_dict(rnd) if rnd is not None else None
    mine = uuv.engine_config_dict(uuv.default_params(), spec, case["num_envs"], case["seed"],
                                  0, ranges)
    mine.pop("device")
    assert json.loads(json.dumps(mine)) == case["engine_config"]


def test_taskspec_target_angles_wrap_like_pose():
    t = uuv.TaskSpec(target=(0, 0, 2, 0.1, -7.0, math.pi))
    assert t.target[3] == 0.10000000000000009          # wrap(0.1) as in the reference
    assert -math.pi < t.target[4] <= math.pi
    assert t.target[5] == math.pi


@pytest.mark.parametrize("kw,msg", [
    (dict(kind="spiral"), "unknown task kind"),
    (dict(lookahead=0), "lookahead must be >= 1"),
    (dict(episode_len=0), "episode_len must be >= 1"),
    (dict(kind="circle", radius=0.0), "radius must be positive"),
    (dict(kind="lemniscate", scale=0.0), "scale must be positive"),
    (dict(control_dt=0.0), "control_dt must be positive"),
    (dict(n_substeps=0), "n_substeps must be >= 1"),
])
def test_taskspec_validation(kw, msg):
    with pytest.raises(ValueError, match=msg):
        uuv.TaskSpec(**kw)


def test_obs_dim():
    assert uuv.TaskSpec().obs_dim == 12
    assert uuv.TaskSpec(kind="circle", lookahead=4).obs_dim == 30


def test_ranges_validation():
    with pytest.raises(ValueError, match="range mass"):
        uuv.RandomizationRanges(mass=(0.0, 1.0))
    with pytest.raises(ValueError, match="rb_offset"):
        uuv.RandomizationRanges(rb_offset=-0.1)
    r = uuv.default_ranges(per_episode=True)
    assert uuv.RandomizationRanges.from_dict(r.to_dict()) == r


def test_vehicle_validation():
    d = vehicles.bluerov2_heavy()
    d["inertia"][0][1] = 0.5
    with pytest.raises(uuv.ParamsError, match="symmetric"):
        uuv.VehicleParams(d)
    d = vehicles.bluerov2_heavy()
    d.pop("mass")
    with pytest.raises(uuv.ParamsError, match="missing field"):
        uuv.VehicleParams(d)
    d = vehicles.bluerov2_heavy()
    d["damping_linear"][0][0] = -5.0
    with pytest.raises(uuv.ParamsError, match="positive semidefinite"):
        uuv.VehicleParams(d)


def test_host_bench_actions_match_oracle():
    from oracle import oracle as orc
    for seed, n, a, off in ((0, 64, 8, 0), (2**64 - 1, 33, 6, 1000)):
        assert np.array_equal(_rng.bench_actions(seed, n, a, off),
                              orc.bench_actions(seed, n, a, off))


def test_resolve_backend(monkeypatch):
    monkeypatch.delenv("UUVSIM_BACKEND", raising=False)
    assert resolve_backend() == "b200"
    assert resolve_backend("native") == "b200"
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        resolve_backend("python")
    monkeypatch.setenv("UUVSIM_BACKEND", "python")
    with pytest.raises(RuntimeError):
        resolve_backend()
    with pytest.raises(ValueError):
        resolve_backend("cuda")


def test_product_fails_loudly_without_library(monkeypatch, tmp_path):
    from paper_2410_14117_b200 import _core
    monkeypatch.setattr(_core, "_lib", None)
    monkeypatch.setenv("UUVSIM_B200_LIB", str(tmp_path / "missing.so"))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _core.load()
