"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the C parity oracle.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs (cpu_baseline and
``--impl reference``) may import this module; it is the checker, never the
thing measured or shipped.

``OracleBatch`` mirrors the reference's ``PyEnvBatch`` (reference
pkg/src/uuvsim/batch.py:36-137) on top of ``uuv_oracle.c``, an fp64 C
restatement of the reference's flat kernels that is bit-identical to the
Python oracle (pinned by tests/golden/, see tests/test_oracle_golden.py).
It takes the same engine-config dict the reference's native engine parses
(reference config.py:135-154 / native/src/engine.rs:17-94), plus two optional
extensions shared with the B200 engine: ``vehicles`` (a list of vehicle docs)
with ``batch.vehicle_mix`` (contiguous per-vehicle env counts over the GLOBAL
env index) and ``batch.env_offset`` (global index of local env 0).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libuuv_oracle.so"

MAX_THR = 8
MAX_VEH = 4
KIND_CODES = {"station_keeping": 0, "circle": 1, "helix": 2, "lemniscate": 3}


class OrcVehicle(ctypes.Structure):
    _fields_ = [
        ("mass", ctypes.c_double), ("inertia", ctypes.c_double * 9),
        ("rg", ctypes.c_double * 3), ("rb", ctypes.c_double * 3),
        ("weight", ctypes.c_double), ("buoyancy", ctypes.c_double),
        ("added", ctypes.c_double * 36), ("dlin", ctypes.c_double * 36),
        ("dquad", ctypes.c_double * 6), ("n_thr", ctypes.c_int32),
        ("curve", ctypes.c_int32 * MAX_THR),
        ("pos", (ctypes.c_double * 3) * MAX_THR), ("dir", (ctypes.c_double * 3) * MAX_THR),
        ("kmax", ctypes.c_double * MAX_THR),
    ]


class OrcTask(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("lookahead", ctypes.c_int32),
        ("n_substeps", ctypes.c_int32), ("pad_", ctypes.c_int32),
        ("episode_len", ctypes.c_int64), ("target", ctypes.c_double * 6),
        ("cx", ctypes.c_double), ("cy", ctypes.c_double), ("radius", ctypes.c_double),
        ("omega", ctypes.c_double), ("climb", ctypes.c_double), ("scale", ctypes.c_double),
        ("depth", ctypes.c_double), ("control_dt", ctypes.c_double),
    ]


class OrcRanges(ctypes.Structure):
    _fields_ = [
        ("enabled", ctypes.c_int32), ("per_episode", ctypes.c_int32),
        ("mass", ctypes.c_double * 2), ("added", ctypes.c_double * 2),
        ("dlin", ctypes.c_double * 2), ("dquad", ctypes.c_double * 2),
        ("thrust", ctypes.c_double * 2), ("rb_offset", ctypes.c_double),
        ("ratio", ctypes.c_double * 2),
    ]


class OrcKParams(ctypes.Structure):
    _fields_ = [
        ("m_total", ctypes.c_double * 36), ("chol", ctypes.c_double * 36),
        ("dlin", ctypes.c_double * 36), ("dquad", ctypes.c_double * 6),
        ("weight", ctypes.c_double), ("buoyancy", ctypes.c_double),
        ("rg", ctypes.c_double * 3), ("rb", ctypes.c_double * 3),
        ("alloc", ctypes.c_double * (6 * MAX_THR)), ("kmax", ctypes.c_double * MAX_THR),
        ("curve", ctypes.c_int32 * MAX_THR), ("n_thr", ctypes.c_int32),
    ]


_lib = None


def build(force: bool = False) -> Path:
    """Compile the oracle with its committed Makefile (gcc, -ffp-contract=off)."""
    if force or not LIB_PATH.is_file():
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.is_file():
        build()
    L = ctypes.CDLL(str(LIB_PATH))
    u64, i64, i32, f64 = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    P = ctypes.POINTER
    vp = ctypes.c_void_p
    L.orc_mix64.restype = u64; L.orc_mix64.argtypes = [u64]
    L.orc_draw_u64.restype = u64; L.orc_draw_u64.argtypes = [u64, u64, u64, u64]
    L.orc_u01.restype = f64; L.orc_u01.argtypes = [u64]
    L.orc_wrap_angle.restype = f64; L.orc_wrap_angle.argtypes = [f64]
    L.orc_build_kernel.restype = i32; L.orc_build_kernel.argtypes = [P(OrcVehicle), P(OrcKParams)]
    L.orc_sample_params.restype = i32
    L.orc_sample_params.argtypes = [P(OrcVehicle), P(OrcRanges), u64, u64, P(u64), P(OrcKParams), vp]
    L.orc_wrench.restype = None; L.orc_wrench.argtypes = [P(OrcKParams), vp, vp]
    L.orc_substep.restype = i32; L.orc_substep.argtypes = [P(OrcKParams), vp, vp, f64, vp]
    L.orc_traj.restype = None; L.orc_traj.argtypes = [P(OrcTask), f64, vp]
    L.orc_observe.restype = None; L.orc_observe.argtypes = [P(OrcTask), vp, i64, vp]
    L.orc_env_step.restype = i32
    L.orc_env_step.argtypes = [P(OrcKParams), P(OrcTask), vp, i64, vp, P(i64), P(f64), P(f64)]
    L.orc_create.restype = vp
    L.orc_create.argtypes = [P(OrcVehicle), i32, vp, P(OrcTask), P(OrcRanges), i64, u64, u64,
                             i32, ctypes.c_char_p, i64]
    L.orc_destroy.restype = None; L.orc_destroy.argtypes = [vp]
    L.orc_set_threads.restype = None; L.orc_set_threads.argtypes = [vp, i32]
    L.orc_obs_dim.restype = i32; L.orc_obs_dim.argtypes = [vp]
    L.orc_reset.restype = None; L.orc_reset.argtypes = [vp, u64, vp]
    L.orc_step.restype = None; L.orc_step.argtypes = [vp, vp, vp, vp, vp, vp]
    for name in ("orc_get_states", "orc_set_states", "orc_get_steps", "orc_set_steps",
                 "orc_get_factors", "orc_observe_all"):
        getattr(L, name).restype = None
        getattr(L, name).argtypes = [vp, vp]
    L.orc_get_counters.restype = None; L.orc_get_counters.argtypes = [vp, vp, vp]
    L.orc_get_kparams.restype = None; L.orc_get_kparams.argtypes = [vp, i64, P(OrcKParams)]
    L.orc_bench_actions.restype = None; L.orc_bench_actions.argtypes = [u64, i64, i32, u64, vp]
    _lib = L
    return L


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------- config
def vehicle_struct(d: dict) -> OrcVehicle:
    """Vehicle doc (reference vehicle.py:3-12 schema) -> OrcVehicle."""
    v = OrcVehicle()
    v.mass = float(d["mass"])
    for i, row in enumerate(d["inertia"]):
        for j, x in enumerate(row):
            v.inertia[i * 3 + j] = float(x)
    for k in range(3):
        v.rg[k] = float(d["r_g"][k])
        v.rb[k] = float(d["r_b"][k])
    v.weight = float(d["weight"])
    v.buoyancy = float(d["buoyancy"])
    for i in range(6):
        for j in range(6):
            v.added[i * 6 + j] = float(d["added_mass"][i][j])
            v.dlin[i * 6 + j] = float(d["damping_linear"][i][j])
        v.dquad[i] = float(d["damping_quadratic"][i])
    th = d["thrusters"]
    if not 1 <= len(th) <= MAX_THR:
        raise ValueError(f"oracle supports 1..{MAX_THR} thrusters")
    v.n_thr = len(th)
    for i, t in enumerate(th):
        for k in range(3):
            v.pos[i][k] = float(t["position"][k])
            v.dir[i][k] = float(t["direction"][k])
        v.kmax[i] = float(t["max_thrust"])
        v.curve[i] = 0 if t.get("curve", "quadratic_signed") == "linear" else 1
    return v


def task_struct(d: dict) -> OrcTask:
    """Task section (reference engine.rs:365-404 defaults) -> OrcTask."""
    t = OrcTask()
    t.kind = KIND_CODES[d.get("kind", "station_keeping")]
    tg = d.get("target", [0.0, 0.0, 2.0, 0.0, 0.0, 0.0])
    for k in range(6):
        t.target[k] = float(tg[k])
    c = d.get("center", [0.0, 0.0])
    t.cx, t.cy = float(c[0]), float(c[1])
    t.radius = float(d.get("radius", 1.0))
    t.omega = float(d.get("angular_rate", 0.1))
    t.climb = float(d.get("climb_rate", 0.05))
    t.scale = float(d.get("scale", 2.0))
    t.depth = float(d.get("depth", 2.0))
    t.lookahead = int(d.get("lookahead", 5))
    t.episode_len = int(d.get("episode_len", 600))
    t.control_dt = float(d.get("control_dt", 0.05))
    t.n_substeps = int(d.get("n_substeps", 10))
    return t


def ranges_struct(d: dict | None) -> OrcRanges:
    r = OrcRanges()
    if d is None:
        r.enabled = 0
        return r
    r.enabled = 1
    r.per_episode = int(bool(d.get("per_episode", False)))
    for name, field in (("mass", "mass"), ("added_mass", "added"), ("damping_linear", "dlin"),
                        ("damping_quadratic", "dquad"), ("max_thrust", "thrust"),
                        ("buoyancy_ratio", "ratio")):
        lo, hi = d.get(name, [1.0, 1.0])
        getattr(r, field)[0] = float(lo)
        getattr(r, field)[1] = float(hi)
    r.rb_offset = float(d.get("rb_offset", 0.0))
    return r


def vehicle_ids(num_envs: int, env_offset: int, mix) -> np.ndarray:
    """Per-env vehicle index from contiguous global slabs (``batch.vehicle_mix``)."""
    if not mix:
        return np.zeros(num_envs, dtype=np.int32)
    bounds = np.cumsum(np.asarray(mix, dtype=np.int64))
    g = np.arange(env_offset, env_offset + num_envs, dtype=np.int64)
    vid = np.searchsorted(bounds, g, side="right")
    return np.minimum(vid, len(mix) - 1).astype(np.int32)


class OracleBatch:
    """CPU oracle batch with the reference PyEnvBatch protocol (batch.py:36-137)."""

    backend = "oracle"

    def __init__(self, cfg: dict, threads: int = 1):
        L = lib()
        self._lib = L
        vdocs = cfg.get("vehicles") or [cfg["vehicle"]]
        batch = cfg.get("batch", {}) or {}
        self.num_envs = int(batch.get("num_envs", 64))
        self.env_offset = int(batch.get("env_offset", 0))
        self.root_seed = int(cfg["seed"])
        self._veh = (OrcVehicle * MAX_VEH)(*[vehicle_struct(v) for v in vdocs])
        self._task = task_struct(cfg.get("task", {}) or {})
        self._ranges = ranges_struct(batch.get("randomization"))
        self.vid = vehicle_ids(self.num_envs, self.env_offset, batch.get("vehicle_mix"))
        self.action_dim = max(int(self._veh[i].n_thr) for i in range(len(vdocs)))
        err = ctypes.create_string_buffer(512)
        h = L.orc_create(self._veh, len(vdocs), _ptr(self.vid), ctypes.byref(self._task),
                         ctypes.byref(self._ranges), self.num_envs, self.root_seed & (2**64 - 1),
                         self.env_offset, self.action_dim, err, 512)
        if not h:
            raise ValueError(err.value.decode())
        self._h = h
        self.obs_dim = int(L.orc_obs_dim(h))
        self.episode_len = int(self._task.episode_len)
        self.threads = 1
        self.set_threads(threads)

    # -- reference protocol --------------------------------------------------
    def reset_all(self, seed: int) -> np.ndarray:
        obs = np.zeros((self.num_envs, self.obs_dim))
        self.root_seed = int(seed)
        self._lib.orc_reset(self._h, int(seed) & (2**64 - 1), _ptr(obs))
        return obs

    def step(self, actions, with_reason: bool = False):
        act = np.ascontiguousarray(actions, dtype=np.float64)
        if act.shape != (self.num_envs, self.action_dim):
            raise ValueError(f"actions must have shape {(self.num_envs, self.action_dim)}, "
                             f"got {act.shape}")
        obs = np.zeros((self.num_envs, self.obs_dim))
        rew = np.zeros(self.num_envs)
        done = np.zeros(self.num_envs, dtype=np.uint8)
        reason = np.zeros(self.num_envs, dtype=np.int8)
        self._lib.orc_step(self._h, _ptr(act), _ptr(obs), _ptr(rew), _ptr(done), _ptr(reason))
        if with_reason:
            return obs, rew, done.astype(bool), reason
        return obs, rew, done.astype(bool)

    def states(self) -> np.ndarray:
        out = np.zeros((self.num_envs, 12))
        self._lib.orc_get_states(self._h, _ptr(out))
        return out

    def set_states(self, s) -> None:
        s = np.ascontiguousarray(s, dtype=np.float64).reshape(self.num_envs, 12)
        self._lib.orc_set_states(self._h, _ptr(s))

    def step_counts(self) -> np.ndarray:
        out = np.zeros(self.num_envs, dtype=np.int64)
        self._lib.orc_get_steps(self._h, _ptr(out))
        return out

    def set_step_counts(self, steps) -> None:
        s = np.ascontiguousarray(steps, dtype=np.int64)
        self._lib.orc_set_steps(self._h, _ptr(s))

    def counters(self):
        rc = np.zeros(self.num_envs, dtype=np.uint64)
        pc = np.zeros(self.num_envs, dtype=np.uint64)
        self._lib.orc_get_counters(self._h, _ptr(rc), _ptr(pc))
        return rc, pc

    def factors(self) -> np.ndarray:
        out = np.zeros((self.num_envs, 9))
        self._lib.orc_get_factors(self._h, _ptr(out))
        return out

    def observe(self) -> np.ndarray:
        out = np.zeros((self.num_envs, self.obs_dim))
        self._lib.orc_observe_all(self._h, _ptr(out))
        return out

    def kparams(self, env: int) -> OrcKParams:
        kp = OrcKParams()
        self._lib.orc_get_kparams(self._h, int(env), ctypes.byref(kp))
        return kp

    def set_threads(self, n: int):
        n = int(n) if n else (os.cpu_count() or 1)
        self.threads = n
        self._lib.orc_set_threads(self._h, n)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.orc_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def bench_actions(seed: int, num_envs: int, n_act: int, env_offset: int = 0) -> np.ndarray:
    """Fixed U[-1,1] bench actions (reference batch.py:168-176), keyed by GLOBAL env index."""
    out = np.zeros((num_envs, n_act))
    lib().orc_bench_actions(int(seed) & (2**64 - 1), num_envs, n_act, env_offset, _ptr(out))
    return out


def wrap_angle(a: float) -> float:
    return float(lib().orc_wrap_angle(float(a)))


def draw_u64(seed, stream, purpose, counter) -> int:
    return int(lib().orc_draw_u64(seed & (2**64 - 1), stream, purpose, counter))


__all__ = ["OracleBatch", "bench_actions", "build", "lib", "vehicle_struct", "task_struct",
           "ranges_struct", "vehicle_ids", "wrap_angle", "draw_u64", "math"]
