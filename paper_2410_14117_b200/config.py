"""Host-side mirror of the reference's configuration types.

Same names, argument meaning and validation errors as the reference so that
callers of ``batch_create`` can switch packages unchanged:

* ``TaskSpec``            reference tasks.py:50-99 (target angles wrap like Pose)
* ``RandomizationRanges`` reference randomize.py:22-68, ``default_ranges`` :71-76
* ``VehicleParams``       reference vehicle.py:75-194 (document + validation)
* ``engine_config_dict``  reference config.py:135-154 (the JSON the engine parses)

These are plain host data; the physics lives in the CUDA engine.
"""

from __future__ import annotations

import copy
import json
import math
from dataclasses import dataclass, field

import numpy as np

from . import vehicles as _vehicles

STATION_KEEPING = "station_keeping"
CIRCLE = "circle"
HELIX = "helix"
LEMNISCATE = "lemniscate"
TASK_KINDS = (STATION_KEEPING, CIRCLE, HELIX, LEMNISCATE)
TRACKING_KINDS = (CIRCLE, HELIX, LEMNISCATE)
REASONS = ("truncation", "divergence", "failure")   # reference tasks.py:41-42


class ParamsError(ValueError):
    """Vehicle parameters violate an invariant (reference vehicle.py:31-32)."""


class ConfigError(ValueError):
    """Malformed or inconsistent run configuration (reference config.py:29-30)."""


def wrap_angle(a: float) -> float:
    """(-pi, pi] wrap with the reference's exact formula (dynamics.py:56-61)."""
    r = math.fmod(a + math.pi, 2.0 * math.pi)
    if r <= 0.0:
        r += 2.0 * math.pi
    return r - math.pi


@dataclass(frozen=True)
class TaskSpec:
    kind: str = STATION_KEEPING
    target: tuple = (0.0, 0.0, 2.0, 0.0, 0.0, 0.0)
    radius: float = 1.0
    angular_rate: float = 0.1
    climb_rate: float = 0.05
    scale: float = 2.0
    depth: float = 2.0
    center: tuple = (0.0, 0.0)
    lookahead: int = 5
    episode_len: int = 600
    control_dt: float = 0.05
    n_substeps: int = 10

    def __post_init__(self):
        if self.kind not in TASK_KINDS:
            raise ValueError(f"unknown task kind {self.kind!r}")
        if self.lookahead < 1:
            raise ValueError("lookahead must be >= 1")
        if self.episode_len < 1:
            raise ValueError("episode_len must be >= 1")
        if self.kind in (CIRCLE, HELIX) and not self.radius > 0.0:
            raise ValueError("radius must be positive")
        if self.kind == LEMNISCATE and not self.scale > 0.0:
            raise ValueError("scale must be positive")
        if not self.control_dt > 0.0:
            raise ValueError("control_dt must be positive")
        if self.n_substeps < 1:
            raise ValueError("n_substeps must be >= 1")
        t = [float(c) for c in self.target]
        if len(t) != 6:
            raise ValueError("target must be a 6-vector [x,y,z,phi,theta,psi]")
        t[3:6] = [wrap_angle(a) for a in t[3:6]]   # Pose.__post_init__ (dynamics.py:75-78)
        object.__setattr__(self, "target", tuple(t))
        object.__setattr__(self, "center", tuple(float(c) for c in self.center))

    @property
    def obs_dim(self) -> int:
        return 12 if self.kind == STATION_KEEPING else 6 * self.lookahead + 6

    def to_dict(self) -> dict:   # reference config.py:33-47
        return {"kind": self.kind, "target": list(self.target), "center": list(self.center),
                "radius": self.radius, "angular_rate": self.angular_rate,
                "climb_rate": self.climb_rate, "scale": self.scale, "depth": self.depth,
                "lookahead": self.lookahead, "episode_len": self.episode_len,
                "control_dt": self.control_dt, "n_substeps": self.n_substeps}

    @staticmethod
    def from_dict(d: dict) -> "TaskSpec":   # reference config.py:50-73
        kw = {}
        for name in ("kind", "radius", "angular_rate", "climb_rate", "scale", "depth",
                     "control_dt", "lookahead", "episode_len", "n_substeps"):
            if name in d:
                kw[name] = d[name]
        if "target" in d:
            if len(d["target"]) != 6:
                raise ConfigError("task.target must be a 6-vector [x,y,z,phi,theta,psi]")
            kw["target"] = tuple(d["target"])
        if "center" in d:
            kw["center"] = tuple(d["center"])
        try:
            return TaskSpec(**kw)
        except (TypeError, ValueError) as e:
            raise ConfigError(f"invalid task section: {e}") from e


@dataclass(frozen=True)
class RandomizationRanges:
    mass: tuple = (1.0, 1.0)
    added_mass: tuple = (1.0, 1.0)
    damping_linear: tuple = (1.0, 1.0)
    damping_quadratic: tuple = (1.0, 1.0)
    max_thrust: tuple = (1.0, 1.0)
    rb_offset: float = 0.0
    buoyancy_ratio: tuple = (1.0, 1.0)
    per_episode: bool = False

    def __post_init__(self):
        for name in ("mass", "added_mass", "damping_linear", "damping_quadratic",
                     "max_thrust", "buoyancy_ratio"):
            lo, hi = getattr(self, name)
            if not (0.0 < lo <= hi):
                raise ValueError(f"range {name} must satisfy 0 < lo <= hi")
            object.__setattr__(self, name, (float(lo), float(hi)))
        if self.rb_offset < 0.0:
            raise ValueError("rb_offset must be >= 0")

    def to_dict(self) -> dict:
        return {"mass": list(self.mass), "added_mass": list(self.added_mass),
                "damping_linear": list(self.damping_linear),
                "damping_quadratic": list(self.damping_quadratic),
                "max_thrust": list(self.max_thrust), "rb_offset": self.rb_offset,
                "buoyancy_ratio": list(self.buoyancy_ratio), "per_episode": self.per_episode}

    @staticmethod
    def from_dict(d: dict) -> "RandomizationRanges":
        kw = {k: tuple(d[k]) for k in ("mass", "added_mass", "damping_linear",
                                        "damping_quadratic", "max_thrust", "buoyancy_ratio")
              if k in d}
        if "rb_offset" in d:
            kw["rb_offset"] = float(d["rb_offset"])
        if "per_episode" in d:
            kw["per_episode"] = bool(d["per_episode"])
        return RandomizationRanges(**kw)


def default_ranges(per_episode: bool = False) -> RandomizationRanges:
    return RandomizationRanges(mass=(0.9, 1.1), added_mass=(0.8, 1.2),
                               damping_linear=(0.7, 1.3), damping_quadratic=(0.7, 1.3),
                               max_thrust=(0.9, 1.1), rb_offset=0.01,
                               buoyancy_ratio=(0.99, 1.01), per_episode=per_episode)


class VehicleParams:
    """A validated vehicle document (reference vehicle.py schema and _validate :114-137)."""

    def __init__(self, doc: dict):
        self._doc = copy.deepcopy(doc)
        self._validate()

    def _validate(self):
        d = self._doc
        try:
            mass = float(d["mass"])
            inertia = np.asarray(d["inertia"], dtype=np.float64)
            added = np.asarray(d["added_mass"], dtype=np.float64)
            dlin = np.asarray(d["damping_linear"], dtype=np.float64)
            dquad = np.asarray(d["damping_quadratic"], dtype=np.float64)
            rg, rb = np.asarray(d["r_g"], float), np.asarray(d["r_b"], float)
            w, b = float(d["weight"]), float(d["buoyancy"])
            th = d["thrusters"]
        except KeyError as e:
            raise ParamsError(f"vehicle parameter file is missing field {e}") from e
        if not mass > 0.0:
            raise ParamsError("mass must be positive")
        for name, mat, shape in (("inertia", inertia, (3, 3)), ("added_mass", added, (6, 6)),
                                 ("damping_linear", dlin, (6, 6))):
            if mat.shape != shape:
                raise ParamsError(f"{name} must have shape {shape}")
        for name, mat in (("inertia", inertia), ("added_mass", added)):
            if not np.allclose(mat, mat.T, atol=1e-9):
                raise ParamsError(f"{name} must be symmetric")
        if rg.shape != (3,) or rb.shape != (3,):
            raise ParamsError("r_g and r_b must be 3-vectors")
        if dquad.shape != (6,):
            raise ParamsError("damping_quadratic must be a 6-vector")
        if np.any(dquad < 0.0):
            raise ParamsError("damping_quadratic components must be >= 0")
        if w < 0.0 or b < 0.0:
            raise ParamsError("weight and buoyancy must be >= 0")
        if np.any(np.linalg.eigvalsh(inertia) <= 0.0):
            raise ParamsError("inertia must be positive definite")
        if np.any(np.linalg.eigvalsh(0.5 * (dlin + dlin.T)) < -1e-9):
            raise ParamsError("damping_linear must be positive semidefinite")
        if not 1 <= len(th) <= 8:
            raise ParamsError("the B200 engine supports 1..8 thrusters")
        for t in th:
            n = math.sqrt(sum(float(c) ** 2 for c in t["direction"]))
            if abs(n - 1.0) > 1e-9:
                raise ValueError(f"thruster direction must be unit norm, got {n!r}")
            if not float(t["max_thrust"]) > 0.0:
                raise ValueError("max_thrust must be positive")

    def n_thrusters(self) -> int:
        return len(self._doc["thrusters"])

    def to_dict(self) -> dict:
        return copy.deepcopy(self._doc)

    @staticmethod
    def from_dict(d: dict) -> "VehicleParams":
        return VehicleParams(d)


def load_params(path) -> VehicleParams:
    with open(path, "r", encoding="utf-8") as f:
        return VehicleParams(json.load(f))


def save_params(params: VehicleParams, path) -> None:
    with open(path, "w", encoding="utf-8") as f:
        json.dump(params.to_dict(), f, indent=2)
        f.write("\n")


def default_params() -> VehicleParams:
    """BlueROV2-Heavy defaults (reference vehicle.py:190-194)."""
    return VehicleParams(_vehicles.bluerov2_heavy())


def bluerov2_params() -> VehicleParams:
    """Standard 6-thruster BlueROV2 (authored here; absent from the reference)."""
    return VehicleParams(_vehicles.bluerov2())


def engine_config_dict(vehicle, task: TaskSpec, num_envs: int, seed: int, threads: int = 0,
                       randomization: RandomizationRanges | None = None, *,
                       precision: str = "fp32", device: int | None = None,
                       env_offset: int = 0, vehicle_mix=None, stats: bool = True) -> dict:
    """Engine JSON document (reference config.py:135-147) plus the B200 keys.

    ``vehicle`` is a VehicleParams / dict, or a list of them for mixed batches
    (then ``vehicle_mix`` gives contiguous GLOBAL env counts per vehicle).
    """
    batch = {"num_envs": int(num_envs), "threads": int(threads),
             "randomization": randomization.to_dict() if randomization else None}
    if env_offset:
        batch["env_offset"] = int(env_offset)
    d = {"seed": int(seed), "task": task.to_dict(), "batch": batch}
    if isinstance(vehicle, (list, tuple)):
        d["vehicles"] = [v.to_dict() if isinstance(v, VehicleParams) else dict(v)
                         for v in vehicle]
        if vehicle_mix is None:
            raise ConfigError("mixed vehicles need vehicle_mix")
        batch["vehicle_mix"] = [int(c) for c in vehicle_mix]
    else:
        d["vehicle"] = vehicle.to_dict() if isinstance(vehicle, VehicleParams) else dict(vehicle)
    dev = {"precision": precision, "stats": bool(stats)}
    if device is not None:
        dev["index"] = int(device)
    d["device"] = dev
    return d


def engine_config_json(*args, **kw) -> str:
    return json.dumps(engine_config_dict(*args, **kw))
