"""Config C4: PPO on the device rollout loop (graph-captured collection).

    python tools/train_c4.py [--task circle] [--envs 16384] [--steps 5e6] [--eval-every 5]

Prints one JSON line per iteration and a summary: collection env-steps/s
(policy + env step inside one CUDA graph per horizon), update time, and the
deterministic evaluation error (reference ppo.py:211-242 metric).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2410_14117_b200 as uuv  # noqa: E402
from paper_2410_14117_b200 import rollout as R  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--task", default="circle")
    ap.add_argument("--vehicle", default="bluerov2")
    ap.add_argument("--envs", type=int, default=16384)
    ap.add_argument("--horizon", type=int, default=64)
    ap.add_argument("--steps", type=float, default=5e6)
    ap.add_argument("--minibatch", type=int, default=65536)
    ap.add_argument("--epochs", type=int, default=4)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--dr", action="store_true")
    ap.add_argument("--eval-every", type=int, default=5)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--unfused", action="store_true", help="framework-op policy path")
    ap.add_argument("--eager-update", action="store_true", help="no CUDA graph for the PPO step")
    a = ap.parse_args()
    base = uuv.bluerov2_params() if a.vehicle == "bluerov2" else uuv.default_params()

    def make(n, seed):
        return uuv.batch_create(uuv.TaskSpec(kind=a.task), base,
                                uuv.default_ranges(per_episode=True) if a.dr else None,
                                n, seed, device=0)

    cfg = R.TrainConfig(num_envs=a.envs, horizon=a.horizon, total_env_steps=int(a.steps),
                        minibatch=a.minibatch, epochs=a.epochs, lr=a.lr)
    t0 = time.perf_counter()
    out = R.train(make, cfg, use_graph=not a.no_graph, eval_every=a.eval_every,
                  log_cb=lambda r: print(json.dumps(r), flush=True),
                  fused=False if a.unfused else None,
                  graph_update=False if a.eager_update else None)
    wall = time.perf_counter() - t0
    final = R.evaluate(out["policy"], out["normalizer"], make, 1024, 1000, 600)
    print(json.dumps({"summary": True, "task": a.task, "envs": a.envs, "env_steps": out["env_steps"],
                      "wall_s": wall, "collect_env_steps_per_sec": out["collect_env_steps_per_sec"],
                      "update_s_per_iter": out["update_s_per_iter"], "final_eval": final}))


if __name__ == "__main__":
    main()
