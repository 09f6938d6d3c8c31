"""PD station/tracking baseline, batched on the device.

The reference validates its environments without learning through a PD
controller evaluated one env at a time on the host (reference
pkg/src/uuvsim/baseline.py:38-102, driven by ppo.py:211-242 ``evaluate``):

    err_body = R(phi, theta, psi)^T (r[0:3] - s[0:3])
    err_ang  = wrap(r[3:6] - s[3:6])                 wrap(a) = (a + pi) % 2pi - pi
    wrench   = kp * [err_body; err_ang] - kd * nu
    forces   = pinv(A) @ wrench                      A = allocation matrix, 6 x N
    throttle = f / kmax (linear) | copysign(sqrt(|f| / kmax), f) (quadratic_signed)
    clip to [-1, 1]

Here the same formula runs over the whole [M, 12] state slab as a handful of
batched torch ops on the env's device and stream, fed by the engine's device
state face (``B200EnvBatch.states_tensor``), so a closed-loop PD episode never
leaves HBM and can be captured in one CUDA graph together with the fused env
steps (the reference trajectory is a precomputed [episode_len, 6] device table;
each captured step reads its own row).  ``pd_baseline`` keeps the reference's
single-state numpy signature for drop-in use.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from .config import STATION_KEEPING, CIRCLE, HELIX, TaskSpec, VehicleParams

CURVE_LINEAR = "linear"
CURVE_QUADRATIC = "quadratic_signed"


@dataclass(frozen=True)
class PDGains:
    """Default gains and validation of reference baseline.py:21-31."""
    kp: tuple = (30.0, 30.0, 30.0, 6.0, 6.0, 6.0)
    kd: tuple = (28.0, 28.0, 28.0, 2.0, 2.0, 2.0)

    def __post_init__(self):
        for name in ("kp", "kd"):
            g = tuple(float(v) for v in getattr(self, name))
            if len(g) != 6 or not all(math.isfinite(v) for v in g):
                raise ValueError(f"{name} must be six finite gains")
            object.__setattr__(self, name, g)


def _doc(params) -> dict:
    return params.to_dict() if isinstance(params, VehicleParams) else dict(params)


def allocation_matrix(params) -> np.ndarray:
    """6 x N, columns [d; p x d] (reference thrusters.py:81-98)."""
    th = _doc(params)["thrusters"]
    a = np.zeros((6, len(th)))
    for i, t in enumerate(th):
        p = np.asarray(t["position"], dtype=np.float64)
        d = np.asarray(t["direction"], dtype=np.float64)
        a[0:3, i] = d
        a[3:6, i] = np.cross(p, d)
    return a


def thruster_table(params):
    """(kmax [N], quadratic [N] bool) of the vehicle's thrusters."""
    th = _doc(params)["thrusters"]
    kmax = np.array([float(t["max_thrust"]) for t in th])
    quad = np.array([t.get("curve", CURVE_QUADRATIC) != CURVE_LINEAR for t in th])
    return kmax, quad


def _rot_zyx(phi, theta, psi, xp):
    cphi, sphi = xp.cos(phi), xp.sin(phi)
    cth, sth = xp.cos(theta), xp.sin(theta)
    cpsi, spsi = xp.cos(psi), xp.sin(psi)
    return ((cpsi * cth, -spsi * cphi + cpsi * sth * sphi, spsi * sphi + cpsi * cphi * sth),
            (spsi * cth, cpsi * cphi + sphi * sth * spsi, -cpsi * sphi + sth * spsi * cphi),
            (-sth, cth * sphi, cth * cphi))


def pd_baseline(state, reference, gains: PDGains, params,
                alloc_pinv: np.ndarray | None = None) -> np.ndarray:
    """Single-state throttle vector, the reference's host signature
    (baseline.py:38-75); ``state``/``reference`` are 12-/6-arrays."""
    s = np.asarray(state, dtype=np.float64)
    r = np.asarray(reference, dtype=np.float64)
    out = pd_batch(torch.from_numpy(s[None]), torch.from_numpy(r), gains, params,
                   None if alloc_pinv is None else torch.from_numpy(np.asarray(alloc_pinv)))
    return out[0].numpy()


def pd_batch(states: torch.Tensor, reference: torch.Tensor, gains: PDGains, params,
             alloc_pinv: torch.Tensor | None = None, out: torch.Tensor | None = None):
    """Batched PD throttles [M, N] from states [M, 12] and a reference pose
    [6] or [M, 6], in the states' dtype/device (baseline.py:50-75)."""
    dt, dev = states.dtype, states.device
    if alloc_pinv is None:
        alloc_pinv = torch.from_numpy(np.linalg.pinv(allocation_matrix(params)))
    pinv = alloc_pinv.to(device=dev, dtype=dt)
    kmax, quad = thruster_table(params)
    kp = torch.tensor(gains.kp, dtype=dt, device=dev)
    kd = torch.tensor(gains.kd, dtype=dt, device=dev)
    kmax_t = torch.from_numpy(kmax).to(device=dev, dtype=dt)
    quad_t = torch.from_numpy(quad).to(device=dev)
    return _pd_core(states, reference.to(device=dev, dtype=dt), kp, kd, pinv, kmax_t, quad_t, out)


def _pd_core(s, r, kp, kd, pinv, kmax, quad, out=None):
    rot = _rot_zyx(s[:, 3], s[:, 4], s[:, 5], torch)
    ew = r[..., 0:3] - s[:, 0:3]
    # err_body = rot^T @ err_world: column j of rot dotted with the world error
    eb = [rot[0][j] * ew[:, 0] + rot[1][j] * ew[:, 1] + rot[2][j] * ew[:, 2] for j in range(3)]
    ea = torch.remainder(r[..., 3:6] - s[:, 3:6] + math.pi, 2.0 * math.pi) - math.pi
    err6 = torch.cat([torch.stack(eb, dim=1), ea], dim=1)
    wrench = kp * err6 - kd * s[:, 6:12]
    forces = wrench @ pinv.T
    thr = torch.where(quad, torch.copysign(torch.sqrt(forces.abs() / kmax), forces),
                      forces / kmax)
    if out is None:
        return thr.clamp(-1.0, 1.0)
    torch.clamp(thr, -1.0, 1.0, out=out)
    return out


def trajectory_table(spec: TaskSpec, steps: int, dtype=torch.float64, device="cpu", start=0):
    """Reference poses [steps, 6] at control steps start..start+steps-1
    (PDActor.reference, baseline.py:90-94, over tasks.py:132-153)."""
    t = torch.arange(start, start + steps, dtype=torch.float64) * spec.control_dt
    if spec.kind == STATION_KEEPING:
        tab = torch.tensor(spec.target, dtype=torch.float64).expand(steps, 6).clone()
    else:
        ang = spec.angular_rate * t
        ca, sa = torch.cos(ang), torch.sin(ang)
        cx, cy = spec.center
        zeros = torch.zeros_like(t)
        if spec.kind in (CIRCLE, HELIX):
            x, y = cx + spec.radius * ca, cy + spec.radius * sa
            z = spec.depth + (spec.climb_rate * t if spec.kind == HELIX else zeros)
            psi = torch.atan2(ca, -sa)
        else:   # lemniscate (Gerono)
            x, y = cx + spec.scale * ca, cy + spec.scale * (sa * ca)
            z = spec.depth + zeros
            psi = torch.atan2(ca * ca - sa * sa, -sa)
        tab = torch.stack([x, y, z, zeros, zeros, psi], dim=1)
    return tab.to(dtype=dtype, device=device)


class UuvPdGains(ctypes.Structure):
    """include/uuvsim.h UuvPdGains (per vehicle slot: pinv [8][6], kmax [8], curve)."""
    _fields_ = [("kp", ctypes.c_double * 6), ("kd", ctypes.c_double * 6),
                ("pinv", ((ctypes.c_double * 6) * 8) * 2), ("kmax", (ctypes.c_double * 8) * 2),
                ("quadratic", (ctypes.c_int32 * 8) * 2)]


@dataclass
class PDActor:
    """evaluate()-compatible PD controller tracking the task reference
    (baseline.py:78-102).  ``actor(obs, states, step)`` accepts numpy arrays
    (host, reference protocol) or torch tensors on any device."""

    spec: TaskSpec
    params: object
    gains: PDGains = field(default_factory=PDGains)

    def __post_init__(self):
        self._pinv = np.linalg.pinv(allocation_matrix(self.params))
        self._kmax, self._quad = thruster_table(self.params)
        self._cache = {}

    def engine_gains(self, params2=None) -> UuvPdGains:
        """Gains + allocation pseudo-inverse for the fused engine kernel; ``params2``
        gives the second vehicle of a mixed batch (default: the same vehicle)."""
        g = UuvPdGains()
        for j in range(6):
            g.kp[j], g.kd[j] = self.gains.kp[j], self.gains.kd[j]
        for slot, prm in enumerate((self.params, params2 if params2 is not None else self.params)):
            pinv = np.linalg.pinv(allocation_matrix(prm))
            kmax, quad = thruster_table(prm)
            for i in range(pinv.shape[0]):
                for j in range(6):
                    g.pinv[slot][i][j] = float(pinv[i, j])
                g.kmax[slot][i] = float(kmax[i])
                g.quadratic[slot][i] = int(bool(quad[i]))
        return g

    def reference(self, step: int) -> np.ndarray:
        return trajectory_table(self.spec, 1, start=int(step))[0].numpy()

    def _consts(self, dtype, device):
        key = (dtype, str(device))
        if key not in self._cache:
            def t(x):
                return torch.as_tensor(x).to(device=device, dtype=dtype)
            self._cache[key] = (t(self.gains.kp), t(self.gains.kd), t(self._pinv),
                                t(self._kmax), torch.as_tensor(self._quad).to(device))
        return self._cache[key]

    def act(self, states: torch.Tensor, reference: torch.Tensor, out=None) -> torch.Tensor:
        """Device form: states [M, 12], reference [6] / [M, 6] tensors."""
        kp, kd, pinv, kmax, quad = self._consts(states.dtype, states.device)
        return _pd_core(states, reference, kp, kd, pinv, kmax, quad, out)

    def __call__(self, obs, states, step):
        if isinstance(states, torch.Tensor):
            ref = torch.as_tensor(self.reference(step)).to(states.device, states.dtype)
            return self.act(states, ref)
        s = torch.from_numpy(np.asarray(states, dtype=np.float64))
        return self.act(s, torch.from_numpy(self.reference(step))).numpy()


@torch.no_grad()
def evaluate_pd(env, actor: PDActor, seed: int, steps: int | None = None,
                use_graph: bool = True) -> dict:
    """Closed-loop PD rollouts on the device (ppo.py:211-242 protocol): every
    env starts from ``reset_all(seed)``; per step the actor reads the device
    state slab, the reference pose at the shared step index, and steps the
    engine.  With ``use_graph`` the whole episode is one CUDA graph.

    Returns the reference metrics plus ``err0`` (per-env reset position
    error), ``per_step_error`` and ``final_error`` (per env, last step)."""
    spec = actor.spec
    steps = spec.episode_len if steps is None else int(steps)
    dev = torch.device("cuda", env.device_index)
    dt = env.dtype
    m, n = env.num_envs, env.action_dim
    table = trajectory_table(spec, steps, dtype=dt, device=dev)
    states = torch.empty((m, 12), dtype=dt, device=dev)
    act = torch.empty((m, n), dtype=dt, device=dev)
    errs = torch.empty((steps, m), dtype=dt, device=dev)
    dones = torch.empty((steps, m), dtype=torch.uint8, device=dev)

    fused = hasattr(env, "pd_actions_tensor")
    gains = actor.engine_gains() if fused else None

    def body(t):
        if fused:   # one kernel over the engine's state slab (uuvsim_dev_pd_actions)
            env.pd_actions_tensor(gains, table[t], out=act)
        else:
            env.states_tensor(out=states)
            actor.act(states, table[t], out=act)
        _o, r, d, _ = env.step_tensors(act)
        errs[t].copy_(r.neg())
        dones[t].copy_(d)

    graph = None
    if use_graph:
        # warm up once outside capture (lazy module loading, allocator), then
        # capture the whole episode; the env is reset after the warm-up step
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            env.reset_tensors(seed)
            body(0)
        torch.cuda.current_stream(dev).wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for t in range(steps):
                body(t)
    env.reset_tensors(seed)
    env.states_tensor(out=states)
    err0 = torch.linalg.vector_norm(table[0, 0:3] - states[:, 0:3], dim=1)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    if graph is not None:
        graph.replay()
    else:
        for t in range(steps):
            body(t)
    ev1.record()
    torch.cuda.synchronize(dev)
    errs64 = errs.double()
    return {"mean_pos_err_m": float(errs64.mean()), "max_pos_err_m": float(errs64.max()),
            "mean_return": float(-errs64.sum(0).mean()), "episodes": m, "seed": seed,
            "per_step_error": errs64.mean(1).cpu().numpy(),
            "err0": err0.double().cpu().numpy(), "final_error": errs64[-1].cpu().numpy(),
            "dones": dones.cpu().numpy(), "device_ms": ev0.elapsed_time(ev1)}


__all__ = ["PDGains", "PDActor", "UuvPdGains", "pd_baseline", "pd_batch", "allocation_matrix",
           "thruster_table", "trajectory_table", "evaluate_pd"]
