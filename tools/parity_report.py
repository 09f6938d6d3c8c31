"""Parity report: error statistics of the B200 engine against the C oracle.

    python tools/parity_report.py [--out gpurun_out/parity.json]

For each config: teacher-forced single-step errors (per state component, max
abs / max scaled-by-tolerance, counts outside tolerance with their input
pitch), and free-rollout drift over 100 steps.  Used to derive the documented
bounds in DESIGN.md; the pass/fail gates live in tests/test_gpu_parity.py.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2410_14117_b200 as uuv  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from tests import parity as P  # noqa: E402
from tests.test_gpu_parity import CONFIGS, _cfg  # noqa: E402


def teacher_forced(cfg, steps=24, warm=300):
    """Strict protocol (tests/test_gpu_parity.py::test_single_step_teacher_forced):
    both sides free-run ``warm`` steps, then each step starts from the SAME
    fp32-rounded state on the GPU and the oracle; every env with |theta_in| <=
    1.4 is compared (no exceptions)."""
    gpu = uuv.B200EnvBatch(cfg)
    ref = orc.OracleBatch(cfg, threads=0)
    act = orc.bench_actions(cfg["seed"], ref.num_envs, ref.action_dim)
    for _ in range(warm):
        gpu.step_ex(act)
        ref.step(act)
    rc_g, pc_g = gpu.counters()
    rc_r, pc_r = ref.counters()
    synced = (rc_g == rc_r) & (pc_g == pc_r)
    gpu.stats(clear=True)
    worst = np.zeros(12)
    worst_scaled = np.zeros(12)
    outs = []
    n_done_mismatch = n_gate = n_band = n_ties = 0
    for t in range(steps):
        s_in = P.f32(ref.states())
        ref.set_states(s_in)
        gpu.set_states(s_in)
        gpu.set_step_counts(ref.step_counts())
        og, rg, dg, qg = gpu.step_ex(act)
        orr, rr, dr, qr = ref.step(act, with_reason=True)
        sg, sr = gpu.states(), ref.states()
        gate = (np.abs(s_in[:, 4]) <= P.PITCH_BAND) & synced
        tie = np.abs(-rr - 10.0) < 1e-4
        n_ties += int((gate & tie).sum())
        n_band += int((~gate).sum())
        ok = gate & ~tie
        n_done_mismatch += int((dg[ok] != dr[ok]).sum())
        live = ok & ~dr
        n_gate += int(live.sum())
        err = P.abs_err(sg[live], sr[live], P.STATE_ANGLES)
        scaled = err / (P.ABS_TOL + P.REL_TOL * np.abs(sr[live]))
        if err.size:
            worst = np.maximum(worst, err.max(axis=0))
            worst_scaled = np.maximum(worst_scaled, scaled.max(axis=0))
        idx = np.argwhere(scaled > 1.0)
        for e_, c_ in idx[:20]:
            env = np.flatnonzero(live)[e_]
            outs.append({"t": t, "env": int(env), "comp": int(c_),
                         "theta_in": float(s_in[env, 4]), "got": float(sg[env, c_]),
                         "want": float(sr[env, c_]), "err": float(err[e_, c_]),
                         "in": s_in[env].tolist()})
    b64 = gpu.stats()["band64_steps"]
    gpu.close()
    return {"max_abs_err": worst.tolist(), "max_err_over_tol": worst_scaled.tolist(),
            "n_outside": len(outs), "outside": outs[:20], "done_mismatch": n_done_mismatch,
            "gated_env_steps": n_gate, "excluded_theta_in_band": n_band, "divergence_ties": n_ties,
            "fp64_band_env_steps": b64, "env_steps": steps * ref.num_envs, "warm": warm}


def rollout(cfg, steps=100, scale=0.3):
    gpu = uuv.B200EnvBatch(cfg)
    ref = orc.OracleBatch(cfg, threads=0)
    act = scale * orc.bench_actions(cfg["seed"], ref.num_envs, ref.action_dim)
    ever = np.zeros(ref.num_envs, dtype=bool)
    drift = []
    mism = 0
    for t in range(steps):
        og, rg, dg = gpu.step(act)
        orr, rr, dr = ref.step(act)
        mism += int((dg != dr).sum())
        sr = ref.states()
        ever |= np.abs(sr[:, 4]) > P.PITCH_BAND
        err = P.abs_err(gpu.states(), sr, P.STATE_ANGLES)
        drift.append(float(err[~ever].max()) if (~ever).any() else 0.0)
    gpu.close()
    return {"drift_by_step": drift[::10] + [drift[-1]], "max_drift": max(drift),
            "n_band_envs": int(ever.sum()), "done_mismatch": mism}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/parity.json")
    ap.add_argument("--configs", default=",".join(CONFIGS))
    ap.add_argument("--envs", type=int, default=0, help="override num_envs of every config")
    ap.add_argument("--tf-steps", type=int, default=24)
    ap.add_argument("--warm", type=int, default=300)
    ap.add_argument("--md", default="", help="also write a markdown summary here")
    args = ap.parse_args()
    rep = {}
    for name in args.configs.split(","):
        kw = dict(CONFIGS[name])
        if args.envs:
            kw["n"] = args.envs
        cfg = _cfg(**kw)
        rep[name] = {"num_envs": cfg["batch"]["num_envs"],
                     "teacher_forced": teacher_forced(cfg, args.tf_steps, args.warm),
                     "rollout_0.3": rollout(cfg)}
        tf = rep[name]["teacher_forced"]
        print(name, "tf max_err/tol", np.round(tf["max_err_over_tol"], 3).tolist(),
              "outside", tf["n_outside"], "rollout drift", rep[name]["rollout_0.3"]["max_drift"],
              flush=True)
    for prec_name, prec in (("fp64_lemniscate", "fp64"),):
        cfg = _cfg(kind="lemniscate", dr="episode", episode_len=37, n=2048, precision=prec)
        rep[prec_name] = {"rollout_0.3": rollout(cfg, 150), "rollout_1.0": rollout(cfg, 150, 1.0)}
        print(prec_name, rep[prec_name]["rollout_0.3"]["max_drift"],
              rep[prec_name]["rollout_1.0"]["max_drift"], flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(rep, indent=1))
    if args.md:
        names = ("x", "y", "z", "phi", "theta", "psi", "u", "v", "w", "p", "q", "r")
        lines = ["# Parity report (B200 fp32 engine vs the C oracle, strict protocol)", "",
                 f"Both sides free-run {args.warm} steps under bench actions, then each of "
                 f"{args.tf_steps} steps starts the GPU and the oracle from the SAME fp32-rounded",
                 "state.  Every env with |theta_in| <= 1.4 rad is gated (the contract's only",
                 "exclusion), tolerance 1e-6 + 1e-5|b| per component (angles mod 2 pi);",
                 "divergence-radius ties (| |dp| - 10 | < 1e-4) are counted.  fp64 band env-steps:",
                 "steps the engine ran in fp64 because the pitch could leave the band.",
                 "Free rollouts at 0.3 x bench actions for the drift bound.", "",
                 "| config | envs | gated env-steps | worst err / tol (component) | outside tol | done mismatch | |theta_in| > 1.4 | fp64 band | ties | 100-step drift |",
                 "|---|---|---|---|---|---|---|---|---|---|"]
        for name, r in rep.items():
            if "teacher_forced" not in r:
                continue
            tf, ro = r["teacher_forced"], r["rollout_0.3"]
            w = int(np.argmax(tf["max_err_over_tol"]))
            lines.append(f"| {name} | {r['num_envs']} | {tf['gated_env_steps']} | "
                         f"{max(tf['max_err_over_tol']):.3f} ({names[w]}) | {tf['n_outside']} | "
                         f"{tf['done_mismatch'] + ro['done_mismatch']} | "
                         f"{tf['excluded_theta_in_band']} | {int(tf['fp64_band_env_steps'])} | "
                         f"{tf['divergence_ties']} | {ro['max_drift']:.2e} |")
        for name, r in rep.items():
            if "teacher_forced" in r:
                continue
            lines.append("")
            lines.append(f"{name}: fp64 engine, 150-step rollouts: max drift "
                         f"{r['rollout_0.3']['max_drift']:.2e} (0.3 x bench actions), "
                         f"{r['rollout_1.0']['max_drift']:.2e} (full bench actions)")
        Path(args.md).write_text("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
