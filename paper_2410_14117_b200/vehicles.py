"""Built-in vehicle parameter sets (host-side data, SI units).

Documents follow the reference's vehicle-file schema (reference
pkg/src/uuvsim/vehicle.py:3-12): mass, inertia (3x3), r_g, r_b, weight,
buoyancy, added_mass (6x6), damping_linear (6x6), damping_quadratic (6),
thrusters [{position, direction, max_thrust, curve}].

* ``bluerov2_heavy()`` -- the reference's only shipped set (reference
  pkg/src/uuvsim/data/bluerov2_heavy.json, 8 vectored thrusters, 13.5 kg,
  W = B).  It is rebuilt here from its geometry; tests/test_host.py checks it
  equals the reference document value for value (tests/golden/vehicles.json).
* ``bluerov2()`` -- the standard 6-thruster BlueROV2, which the reference does
  NOT ship (reference SPEC.md:8).  Authored here as documented engineering
  defaults in the spirit of the Heavy file (its caveat applies: plausible,
  not calibrated): 11.5 kg, neutrally buoyant, 4 vectored horizontal
  thrusters at +-45 deg and 2 vertical thrusters on the lateral axis.
"""

from __future__ import annotations

import copy
import math

G = 9.81


def _diag6(d):
    return [[float(d[i]) if i == j else 0.0 for j in range(6)] for i in range(6)]


def _diag3(d):
    return [[float(d[i]) if i == j else 0.0 for j in range(3)] for i in range(3)]


def _thruster(pos, direction, kmax, curve="quadratic_signed"):
    return {"position": [float(c) for c in pos], "direction": [float(c) for c in direction],
            "max_thrust": float(kmax), "curve": curve}


def _vectored_horizontals(ax, ay, kmax):
    c = math.sqrt(2.0) / 2.0
    return [
        _thruster((ax, ay, 0.0), (c, c, 0.0), kmax),
        _thruster((ax, -ay, 0.0), (c, -c, 0.0), kmax),
        _thruster((-ax, ay, 0.0), (c, -c, 0.0), kmax),
        _thruster((-ax, -ay, 0.0), (c, c, 0.0), kmax),
    ]


def bluerov2_heavy() -> dict:
    """BlueROV2-Heavy-class defaults (8 thrusters); equals the reference data file."""
    k = 35.0
    vx, vy = 0.120, 0.218
    verticals = [_thruster((sx * vx, sy * vy, 0.0), (0.0, 0.0, -1.0), k)
                 for sx, sy in ((1, 1), (1, -1), (-1, 1), (-1, -1))]
    return {
        "mass": 13.5,
        "inertia": _diag3((0.26, 0.23, 0.37)),
        "r_g": [0.0, 0.0, 0.02],
        "r_b": [0.0, 0.0, 0.0],
        "weight": 132.435,
        "buoyancy": 132.435,
        "added_mass": _diag6((6.36, 7.12, 18.68, 0.189, 0.135, 0.222)),
        "damping_linear": _diag6((13.7, 6.0, 33.0, 0.6, 0.8, 0.9)),
        "damping_quadratic": [141.0, 217.0, 190.0, 1.19, 0.47, 1.5],
        "thrusters": _vectored_horizontals(0.156, 0.111, k) + verticals,
    }


def bluerov2() -> dict:
    """Standard BlueROV2 (6 thrusters), authored engineering defaults (not in the reference)."""
    k = 35.0
    mass = 11.5
    weight = mass * G
    verticals = [_thruster((0.0, 0.218, 0.0), (0.0, 0.0, -1.0), k),
                 _thruster((0.0, -0.218, 0.0), (0.0, 0.0, -1.0), k)]
    return {
        "mass": mass,
        "inertia": _diag3((0.16, 0.16, 0.16)),
        "r_g": [0.0, 0.0, 0.02],
        "r_b": [0.0, 0.0, 0.0],
        "weight": weight,
        "buoyancy": weight,
        "added_mass": _diag6((5.5, 12.7, 14.57, 0.12, 0.12, 0.12)),
        "damping_linear": _diag6((4.03, 6.22, 5.18, 0.07, 0.07, 0.07)),
        "damping_quadratic": [18.18, 21.66, 36.99, 1.55, 1.55, 1.55],
        "thrusters": _vectored_horizontals(0.156, 0.111, k) + verticals,
    }


VEHICLES = {"bluerov2_heavy": bluerov2_heavy, "bluerov2": bluerov2}


def get_vehicle(name: str) -> dict:
    try:
        return copy.deepcopy(VEHICLES[name]())
    except KeyError:
        raise ValueError(f"unknown vehicle {name!r}; known: {sorted(VEHICLES)}") from None
