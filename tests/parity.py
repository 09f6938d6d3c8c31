"""Parity helpers shared by the GPU tests (fp32 tolerance contract of north_star).

Contract (BASELINE.json north_star):
* single step, teacher-forced from the oracle state: |a - b| <= 1e-6 + 1e-5 |b|
  per component, angles compared modulo 2 pi, over envs whose pitch stays in
  |theta| <= 1.4 rad at the start and end of the step (inside the Euler
  singularity band tan/sec(theta) amplify fp32 rounding; counted, not gated);
* reset / termination: done mask, reason, step counters and RNG counters
  bit-exact; reset states equal fp32(oracle fp64) exactly; divergence-radius
  ties (| |dp| - 10 | < 1e-4) are counted and excluded.
"""

from __future__ import annotations

import copy
import math

import numpy as np

ABS_TOL = 1e-6
REL_TOL = 1e-5
PITCH_BAND = 1.4
STATE_ANGLES = (3, 4, 5)


def angle_diff(a, b):
    d = np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)
    return np.abs(np.mod(d + math.pi, 2 * math.pi) - math.pi)


def obs_angle_cols(obs_dim: int):
    if obs_dim == 12:
        return [3, 4, 5]
    la = (obs_dim - 6) // 6
    return [6 * k + j for k in range(la) for j in (3, 4, 5)]


def abs_err(got, want, angle_cols=()):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    err = np.abs(got - want)
    for c in angle_cols:
        err[..., c] = angle_diff(got[..., c], want[..., c])
    return err


def within_tol(got, want, angle_cols=()):
    err = abs_err(got, want, angle_cols)
    return err <= ABS_TOL + REL_TOL * np.abs(np.asarray(want, dtype=np.float64))


def f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def with_device(cfg: dict, **dev) -> dict:
    c = copy.deepcopy(cfg)
    d = dict(c.get("device") or {})
    d.update(dev)
    c["device"] = d
    return c
