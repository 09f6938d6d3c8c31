"""Closed-loop PD report: device PD + fused step vs the C oracle + fp64 PD.

    python tools/pd_report.py [--envs 2048] [--big 1048576]

Prints one JSON line per case with the max relative drift of the mean
per-step error, done-mask equality, and the device closed-loop throughput
(one CUDA graph per 600-step episode) at --big envs.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2410_14117_b200 as uuv  # noqa: E402
from paper_2410_14117_b200 import baseline as B  # noqa: E402
from tests.test_baseline import _consts, _oracle_closed_loop  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=2048)
    ap.add_argument("--big", type=int, default=1 << 20)
    a = ap.parse_args()
    for kind, veh, dr, prec in (("station_keeping", "heavy", False, "fp32"),
                                ("circle", "bluerov2", True, "fp32"),
                                ("lemniscate", "heavy", True, "fp32"),
                                ("station_keeping", "heavy", False, "fp64")):
        spec = uuv.TaskSpec(kind=kind)
        params = uuv.default_params() if veh == "heavy" else uuv.bluerov2_params()
        ranges = uuv.default_ranges(per_episode=True) if dr else None
        cfg = uuv.engine_config_dict(params, spec, a.envs, 11, 0, ranges, precision=prec, device=0)
        tab = B.trajectory_table(spec, 600).numpy()
        _s0, errs, dones, _ = _oracle_closed_loop(cfg, 600, 11, _consts(params), tab)
        env = uuv.B200EnvBatch(cfg, 11)
        out = B.evaluate_pd(env, B.PDActor(spec, params), 11, 600)
        env.close()
        ref = errs.mean(1)
        drift = np.abs(out["per_step_error"] - ref) / np.maximum(np.abs(ref), 1e-12)
        print(json.dumps({"case": f"{kind}/{veh}/{'dr' if dr else 'nodr'}/{prec}",
                          "envs": a.envs, "max_rel_drift_mean_err": float(drift.max()),
                          "dones_equal": bool(np.array_equal(out["dones"].astype(bool), dones)),
                          "final_mean_err_gpu": float(out["per_step_error"][-1]),
                          "final_mean_err_oracle": float(ref[-1])}), flush=True)
    # device closed-loop throughput at scale
    spec = uuv.TaskSpec()
    params = uuv.default_params()
    env = uuv.batch_create(spec, params, None, a.big, 3, device=0)
    actor = B.PDActor(spec, params)
    B.evaluate_pd(env, actor, 3, 50)                    # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = B.evaluate_pd(env, actor, 3, 600)
    wall = time.perf_counter() - t0
    env.close()
    print(json.dumps({"case": "pd_closed_loop_throughput", "envs": a.big, "steps": 600,
                      "wall_s_incl_capture": wall,
                      "env_steps_per_s_incl_capture": a.big * 600 / wall,
                      "device_ms_episode": out["device_ms"],
                      "env_steps_per_s_device": a.big * 600 / (out["device_ms"] * 1e-3),
                      "spec_pass": bool(np.all(out["final_error"] < 0.3 * out["err0"]))}))


if __name__ == "__main__":
    main()
