"""Pin the C oracle to the reference: bit-exact against the golden fixtures.

The fixtures (tests/golden/*.json|npz) were produced by running the
reference's own Python PyEnvBatch / flat kernels (tests/golden/make_golden.py).
Passing here is what makes the oracle a trustworthy checker for the CUDA path.
"""

from __future__ import annotations

import ctypes
import hashlib
import json
import math
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as orc

GOLDEN = Path(__file__).resolve().parent / "golden"
ANCHORS = json.loads((GOLDEN / "anchors.json").read_text())
KAT = json.loads((GOLDEN / "kat.json").read_text())


def _replay(run):
    c = run["config"]
    b = orc.OracleBatch(c, threads=4)
    act = orc.bench_actions(c["seed"], b.num_envs, b.action_dim) * run["action_scale"]
    h = hashlib.sha256()
    obs0 = b.reset_all(c["seed"])
    h.update(obs0.tobytes())
    sum_rew, n_done = 0.0, 0
    for t in range(run["steps"]):
        if run["reseed_at"] is not None and t == run["reseed_at"]:
            h.update(b.reset_all(c["seed"] + 1).tobytes())
        obs, rew, done = b.step(act)
        h.update(obs.tobytes() + rew.tobytes() + done.tobytes())
        sum_rew += float(rew.sum())
        n_done += int(done.sum())
    rc, pc = b.counters()
    return {
        "sum_reward": sum_rew, "n_dones": n_done,
        "sum_step_counts": int(b.step_counts().sum()),
        "stream_sha256": h.hexdigest(),
        "states_sha256": hashlib.sha256(b.states().tobytes()).hexdigest(),
        "counters_sha256": hashlib.sha256(rc.tobytes() + pc.tobytes()).hexdigest(),
    }


@pytest.mark.parametrize("run", ANCHORS, ids=[r["name"] for r in ANCHORS])
def test_anchor_bit_exact(run):
    got = _replay(run)
    for key in ("n_dones", "sum_step_counts", "stream_sha256", "states_sha256",
                "counters_sha256"):
        assert got[key] == run[key], key
    assert got["sum_reward"] == run["sum_reward"]


def test_thread_count_independence():
    """engine.rs:4-5 / SPEC.md:347: results independent of the thread count."""
    run = next(r for r in ANCHORS if r["name"] == "lemniscate_drep_len37")
    c = run["config"]
    outs = []
    for threads in (1, 3, 8):
        b = orc.OracleBatch(c, threads=threads)
        act = orc.bench_actions(c["seed"], b.num_envs, b.action_dim)
        for _ in range(80):
            b.step(act)
        outs.append(b.states().tobytes())
    assert outs[0] == outs[1] == outs[2]


def test_traces_exact():
    tr = np.load(GOLDEN / "traces.npz")
    for prefix, name in (("lemniscate_", "trace_lemniscate"), ("station_", "trace_station")):
        run = next(r for r in ANCHORS if r["name"] == name)
        c = run["config"]
        b = orc.OracleBatch(c)
        act = orc.bench_actions(c["seed"], b.num_envs, b.action_dim)
        assert np.array_equal(b.reset_all(c["seed"]), tr[prefix + "obs"][0])
        for t in range(run["steps"]):
            obs, rew, done = b.step(act)
            assert np.array_equal(obs, tr[prefix + "obs"][t + 1])
            assert np.array_equal(rew, tr[prefix + "rew"][t])
            assert np.array_equal(done, tr[prefix + "done"][t])
            assert np.array_equal(b.states(), tr[prefix + "states"][t + 1])


def test_sharding_invariance():
    """Global env offsets: two half slabs == the whole batch, bit for bit."""
    run = next(r for r in ANCHORS if r["name"] == "helix_drep_len50")
    c = run["config"]
    whole = orc.OracleBatch(c)
    act = orc.bench_actions(c["seed"], whole.num_envs, whole.action_dim)
    n = whole.num_envs
    halves = []
    for off in (0, n // 2):
        ci = json.loads(json.dumps(c))
        ci["batch"]["num_envs"] = n // 2
        ci["batch"]["env_offset"] = off
        halves.append(orc.OracleBatch(ci))
    for _ in range(120):
        o, r, d = whole.step(act)
        parts = [h.step(act[i * (n // 2):(i + 1) * (n // 2)]) for i, h in enumerate(halves)]
        assert np.array_equal(o, np.concatenate([p[0] for p in parts]))
        assert np.array_equal(d, np.concatenate([p[2] for p in parts]))
    assert np.array_equal(whole.states(), np.concatenate([h.states() for h in halves]))


def test_kat_rng_and_wrap():
    L = orc.lib()
    for z, want in KAT["mix64"]:
        assert L.orc_mix64(z) == want
    for s, st, p, c, want in KAT["draw_u64"]:
        assert L.orc_draw_u64(s, st, p, c) == want
    for b, want in KAT["u01"]:
        assert L.orc_u01(b) == want
    for a, want in KAT["wrap_angle"]:
        assert L.orc_wrap_angle(a) == want


def test_kat_kernel_params():
    from paper_2410_14117_b200.vehicles import bluerov2, bluerov2_heavy
    L = orc.lib()
    for name, doc in (("bluerov2_heavy", bluerov2_heavy()), ("bluerov2", bluerov2())):
        kp = orc.OrcKParams()
        assert L.orc_build_kernel(ctypes.byref(orc.vehicle_struct(doc)), ctypes.byref(kp)) == 0
        want = KAT["kernel"][name]
        assert list(kp.m_total) == want["m_total"]
        assert list(kp.chol) == want["chol"]
        n = kp.n_thr
        assert list(kp.alloc)[:6 * n] == want["alloc"]


def test_kat_sample_params():
    from paper_2410_14117_b200.vehicles import bluerov2_heavy
    L = orc.lib()
    base = orc.vehicle_struct(bluerov2_heavy())
    r = orc.ranges_struct({"mass": [0.9, 1.1], "added_mass": [0.8, 1.2],
                           "damping_linear": [0.7, 1.3], "damping_quadratic": [0.7, 1.3],
                           "max_thrust": [0.9, 1.1], "rb_offset": 0.01,
                           "buoyancy_ratio": [0.99, 1.01]})
    for sp in KAT["sample_params"]:
        kp = orc.OrcKParams()
        ctr = ctypes.c_uint64(0)
        fac = np.zeros(9)
        rc = L.orc_sample_params(ctypes.byref(base), ctypes.byref(r), 0, sp["env"],
                                 ctypes.byref(ctr), ctypes.byref(kp),
                                 fac.ctypes.data_as(ctypes.c_void_p))
        assert rc == 0 and ctr.value == sp["counter"] == 9
        assert list(kp.m_total) == sp["m_total"]
        assert list(kp.chol) == sp["chol"]
        assert kp.weight == sp["weight"] and kp.buoyancy == sp["buoyancy"]
        assert list(kp.rb) == sp["r_b"]
        assert list(kp.kmax)[:8] == sp["max_thrust"]
        assert list(kp.dquad) == sp["damping_quadratic"]


def test_kat_wrench_substep_traj_observe():
    from paper_2410_14117_b200.vehicles import bluerov2_heavy
    L = orc.lib()
    kp = orc.OrcKParams()
    L.orc_build_kernel(ctypes.byref(orc.vehicle_struct(bluerov2_heavy())), ctypes.byref(kp))
    for a, want in KAT["wrench"]:
        a = np.array(a)
        tau = np.zeros(6)
        L.orc_wrench(ctypes.byref(kp), a.ctypes.data_as(ctypes.c_void_p),
                     tau.ctypes.data_as(ctypes.c_void_p))
        assert tau.tolist() == want
    for s, tau, want, fail in KAT["substep"]:
        s, tau = np.array(s), np.array(tau)
        out = np.zeros(12)
        f = L.orc_substep(ctypes.byref(kp), s.ctypes.data_as(ctypes.c_void_p),
                          tau.ctypes.data_as(ctypes.c_void_p), 0.005,
                          out.ctypes.data_as(ctypes.c_void_p))
        assert f == fail
        assert out.tolist() == want
    for kind, t, want in KAT["traj"]:
        task = orc.task_struct({"kind": kind})
        out = np.zeros(4)
        L.orc_traj(ctypes.byref(task), t, out.ctypes.data_as(ctypes.c_void_p))
        assert out.tolist() == want
    for kind, s, step, want in KAT["observe"]:
        task = orc.task_struct({"kind": kind})
        s = np.array(s)
        out = np.zeros(len(want))
        L.orc_observe(ctypes.byref(task), s.ctypes.data_as(ctypes.c_void_p), step,
                      out.ctypes.data_as(ctypes.c_void_p))
        assert out.tolist() == want


def test_spec_known_answers():
    """SURVEY §4 known answers (with the SPEC.md:230 sign erratum: the code wins)."""
    spec = KAT["spec"]
    np.testing.assert_allclose(spec["kinematic_psi_half_pi"], [0, 1, 0, 0, 0, 0], atol=1e-15)
    assert spec["thrust_force_quadratic"] == -10.0
    assert math.isclose(spec["pose_error_yaw"][5], 0.28318530717958623, rel_tol=1e-12)
    assert spec["reward_345"] == -5.0
    assert spec["circle_t0"][:3] == [1.0, 0.0, 2.0]
    assert math.isclose(spec["circle_t0"][3], math.pi / 2)
    assert orc.wrap_angle(-math.pi) == orc.wrap_angle(math.pi) == orc.wrap_angle(3 * math.pi)
