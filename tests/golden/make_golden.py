"""Generate the golden fixtures by running the REFERENCE's own Python oracle.

Run in the build container (the reference exists only there):

    python tests/golden/make_golden.py

It imports ``uuvsim`` from /root/reference/pkg/src (read-only), drives its
PyEnvBatch (reference pkg/src/uuvsim/batch.py:36-137) and flat kernels, and
writes small fixtures next to this file:

* ``anchors.json``  -- per-run digests (sum of rewards, dones, step counts,
  sha256 of the obs/reward/done stream and of the final states/counters) for
  the SURVEY Appendix-C runs plus tracking / per-episode-DR / BlueROV2 /
  reseed variants;
* ``traces.npz``    -- full per-step arrays of two short runs;
* ``kat.json``      -- scalar known answers (RNG, wrap_angle, kernel params,
  sample_params, wrench, substep, trajectory, observe) incl. SPEC.md examples;
* ``vehicles.json`` -- the reference's Heavy vehicle document.

Nothing on the GPU box reads /root/reference; tests only read these files.
"""

from __future__ import annotations

import hashlib
import json
import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import uuvsim  # noqa: E402  (reference)
from uuvsim import rng as rrng  # noqa: E402
from uuvsim import batch as rbatch  # noqa: E402
from uuvsim import config as rconfig  # noqa: E402
from uuvsim import dynamics as rdyn  # noqa: E402
from uuvsim import tasks as rtasks  # noqa: E402
from uuvsim import thrusters as rthr  # noqa: E402
from uuvsim.randomize import RandomizationRanges, default_ranges, sample_params  # noqa: E402
from uuvsim.vehicle import VehicleParams, default_params  # noqa: E402

from paper_2410_14117_b200.vehicles import bluerov2  # noqa: E402

HEAVY = default_params().to_dict()
BLUEROV2 = bluerov2()
DR = default_ranges().to_dict()
DR_EP = dict(DR, per_episode=True)


def cfg(vehicle, task, num_envs, seed, randomization=None):
    return {"seed": seed, "vehicle": vehicle, "task": task,
            "batch": {"num_envs": num_envs, "threads": 0, "randomization": randomization}}


def make_ref_batch(c):
    """Build the reference PyEnvBatch; also return the normalised engine config.

    The stored config is what the reference itself would hand its native
    engine (config.engine_config_dict; e.g. target angles pass through
    Pose.__post_init__'s wrap), so JSON-level consumers see identical inputs.
    """
    veh = VehicleParams.from_dict(c["vehicle"])
    task = rconfig.task_from_dict(c["task"])
    rnd = c["batch"]["randomization"]
    ranges = RandomizationRanges.from_dict(rnd) if rnd is not None else None
    b = rbatch.PyEnvBatch(task, veh, ranges, c["batch"]["num_envs"], c["seed"])
    norm = rconfig.engine_config_dict(veh, task, c["batch"]["num_envs"], c["seed"], 0, ranges)
    return b, norm


def run(name, c, steps, action_scale=1.0, reseed_at=None, trace=False):
    b, c = make_ref_batch(c)
    act = rbatch.bench_actions(b) * action_scale
    h = hashlib.sha256()
    obs0 = b.reset_all(c["seed"])
    h.update(obs0.tobytes())
    sum_rew = 0.0
    n_done = 0
    tr = {"obs": [obs0], "rew": [], "done": [], "states": [b.states()]}
    for t in range(steps):
        if reseed_at is not None and t == reseed_at:
            o = b.reset_all(c["seed"] + 1)
            h.update(o.tobytes())
        obs, rew, done = b.step(act)
        h.update(obs.tobytes() + rew.tobytes() + done.tobytes())
        sum_rew += float(rew.sum())
        n_done += int(done.sum())
        if trace:
            tr["obs"].append(obs); tr["rew"].append(rew); tr["done"].append(done)
            tr["states"].append(b.states())
    states = b.states()
    rc = np.array([s.counter for s in b._reset_streams], dtype=np.uint64)
    pc = np.array([s.counter for s in b._param_streams], dtype=np.uint64)
    out = {
        "name": name, "config": c, "steps": steps, "action_scale": action_scale,
        "reseed_at": reseed_at,
        "sum_reward": sum_rew, "n_dones": n_done,
        "sum_step_counts": int(b.step_counts().sum()),
        "stream_sha256": h.hexdigest(),
        "states_sha256": hashlib.sha256(states.tobytes()).hexdigest(),
        "counters_sha256": hashlib.sha256(rc.tobytes() + pc.tobytes()).hexdigest(),
    }
    print(f"{name}: sum_rew={sum_rew:.12e} dones={n_done} stream={out['stream_sha256'][:16]}")
    if trace:
        return out, {k: np.array(v) for k, v in tr.items()}
    return out, None


def kats():
    k = {}
    k["draw_u64"] = [[s, st, p, c, rrng.draw_u64(s, st, p, c)]
                     for s, st, p, c in [(0, 0, 0, 0), (0, 17, 1, 5), (12345, 3, 2, 7),
                                         (2**64 - 1, 2**40, 1, 123456789), (7, 65535, 0, 8)]]
    k["mix64"] = [[z, rrng.mix64(z)] for z in (0, 1, 2**63, 2**64 - 1, 0x1234567890ABCDEF)]
    k["u01"] = [[b, rrng.u01(b)] for b in (0, 1 << 11, 2**64 - 1, 0xDEADBEEFCAFEBABE)]
    k["wrap_angle"] = [[a, rdyn.wrap_angle(a)] for a in
                       (0.0, 0.1, -math.pi, math.pi, 3 * math.pi, -3 * math.pi, 1e-300, 7.5,
                        -7.5, 100.0, -1e6, 2 * math.pi, math.pi + 1e-15)]
    kernels = {}
    for nm, doc in (("bluerov2_heavy", HEAVY), ("bluerov2", BLUEROV2)):
        kp = VehicleParams.from_dict(doc).kernel()
        kernels[nm] = {"m_total": list(kp.m_total), "chol": list(kp.chol),
                       "alloc": list(kp.alloc)}
    k["kernel"] = kernels
    # sample_params: factors are recovered from the kernel params
    sp = []
    for env in (0, 1, 63, 1000):
        st = rrng.Stream(0, env, rrng.PURPOSE_PARAMS)
        p = sample_params(default_params(), default_ranges(), st)
        kp = p.kernel()
        sp.append({"env": env, "counter": st.counter, "m_total": list(kp.m_total),
                   "chol": list(kp.chol), "weight": kp.weight, "buoyancy": kp.buoyancy,
                   "r_b": list(kp.r_b), "max_thrust": list(kp.max_thrust),
                   "damping_quadratic": list(kp.damping_quadratic)})
    k["sample_params"] = sp
    # wrench / substep / trajectory / observe on seeded random inputs
    r = np.random.default_rng(1234)
    kp = default_params().kernel()
    wr = []
    for _ in range(8):
        a = (r.uniform(-1.5, 1.5, 8)).tolist()
        wr.append([a, rthr._wrench_flat(kp.alloc, kp.max_thrust, kp.curve_codes, a)])
    k["wrench"] = wr
    ss = []
    for _ in range(16):
        s = r.uniform(-1, 1, 12)
        s[3:6] = r.uniform(-3, 3, 3)
        s[4] = r.uniform(-1.4, 1.4)
        tau = r.uniform(-50, 50, 6)
        out, fail, _ = rdyn._substep_flat(kp, s.tolist(), tau.tolist(), 0.005)
        ss.append([s.tolist(), tau.tolist(), list(out), fail])
    k["substep"] = ss
    tj = []
    for kind in ("circle", "helix", "lemniscate"):
        spec = rtasks.TaskSpec(kind=kind)
        kt = spec.kernel()
        for t in (0.0, 0.05, 1.0, 15.7, 29.95):
            tj.append([kind, t, list(rtasks._traj_flat(kt, t))])
    k["traj"] = tj
    ob = []
    for kind in ("station_keeping", "circle", "lemniscate"):
        spec = rtasks.TaskSpec(kind=kind)
        s = r.uniform(-2, 2, 12)
        s[3:6] = r.uniform(-3, 3, 3)
        ob.append([kind, s.tolist(), 7, rtasks._observe_flat(spec.kernel(), s.tolist(), 7)])
    k["observe"] = ob
    # SPEC known answers, values as the reference code returns them
    k["spec"] = {
        "kinematic_psi_half_pi": rdyn.kinematic_transform(
            rdyn.Pose(psi=math.pi / 2), rdyn.BodyVelocity(u=1.0)).tolist(),
        "thrust_force_quadratic": rthr.thrust_force(-0.5, 40.0, "quadratic_signed"),
        "pose_error_yaw": rtasks.pose_error(rdyn.Pose(psi=3.0), rdyn.Pose(psi=-3.0)).tolist(),
        "reward_345": rtasks.reward(rtasks.TaskSpec(target=rdyn.Pose(3.0, 4.0, 0.0)),
                                    rdyn.State(), 0),
        "circle_t0": list(rtasks._traj_flat(rtasks.TaskSpec(kind="circle").kernel(), 0.0)),
    }
    return k


def main():
    runs = []
    traces = {}
    heavy_station = {"kind": "station_keeping"}
    runs.append(run("c1_station_nodr_T1000", cfg(HEAVY, heavy_station, 64, 0), 1000)[0])
    runs.append(run("station_dr_T1000", cfg(HEAVY, heavy_station, 64, 0, DR), 1000)[0])
    runs.append(run("circle_dr_T300", cfg(HEAVY, {"kind": "circle"}, 64, 0, DR), 300)[0])
    runs.append(run("helix_drep_len50", cfg(HEAVY, {"kind": "helix", "episode_len": 50}, 32, 3,
                                            DR_EP), 200)[0])
    runs.append(run("lemniscate_drep_len37", cfg(HEAVY, {"kind": "lemniscate", "episode_len": 37},
                                                 32, 11, DR_EP), 200)[0])
    runs.append(run("bluerov2_station_T600", cfg(BLUEROV2, heavy_station, 48, 5), 600)[0])
    runs.append(run("bluerov2_circle_drep_len41",
                    cfg(BLUEROV2, {"kind": "circle", "episode_len": 41, "lookahead": 3}, 24, 9,
                        DR_EP), 150)[0])
    runs.append(run("station_reseed", cfg(HEAVY, heavy_station, 16, 2), 100, reseed_at=40)[0])
    runs.append(run("station_half_actions_substeps4",
                    cfg(HEAVY, {"kind": "station_keeping", "n_substeps": 4, "control_dt": 0.04,
                                "target": [1.0, -2.0, 3.0, 0.1, -0.2, 2.5]}, 16, 21),
                    300, action_scale=0.5)[0])
    a, tr = run("trace_lemniscate", cfg(HEAVY, {"kind": "lemniscate", "episode_len": 23}, 6, 4,
                                        DR_EP), 60, trace=True)
    runs.append(a)
    for k2, v in tr.items():
        traces["lemniscate_" + k2] = v
    a, tr = run("trace_station", cfg(HEAVY, heavy_station, 5, 0), 40, trace=True)
    runs.append(a)
    for k2, v in tr.items():
        traces["station_" + k2] = v

    (HERE / "anchors.json").write_text(json.dumps(runs, indent=1) + "\n")
    np.savez_compressed(HERE / "traces.npz", **traces)
    (HERE / "kat.json").write_text(json.dumps(kats(), indent=1) + "\n")
    (HERE / "vehicles.json").write_text(json.dumps({"bluerov2_heavy": HEAVY}, indent=1) + "\n")
    # engine-config documents the reference renders for its native engine
    ecs = []
    for task_in, rnd_in, n, seed in (
            ({"kind": "station_keeping", "target": [1.0, -2.0, 3.0, 0.1, -0.2, 7.0]}, None, 8, 3),
            ({"kind": "lemniscate", "lookahead": 3, "episode_len": 99, "scale": 2.5},
             dict(DR_EP), 64, 2**63 + 5),
            ({"kind": "helix", "center": [1.5, -0.5], "radius": 2.0, "climb_rate": 0.1,
              "control_dt": 0.04, "n_substeps": 8}, {"mass": [0.8, 1.2]}, 5, 0)):
        veh = VehicleParams.from_dict(HEAVY)
        task = rconfig.task_from_dict(task_in)
        ranges = RandomizationRanges.from_dict(rnd_in) if rnd_in is not None else None
        ecs.append({"task_in": task_in, "randomization_in": rnd_in, "num_envs": n, "seed": seed,
                    "engine_config": rconfig.engine_config_dict(veh, task, n, seed, 0, ranges)})
    (HERE / "engine_configs.json").write_text(json.dumps(ecs, indent=1) + "\n")
    print("wrote", HERE)


if __name__ == "__main__":
    main()
