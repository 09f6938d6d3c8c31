"""C4 rollout loop: time per horizon (graph) and, under ncu, the per-kernel split.

    python tools/c4_loop_probe.py [--eager] [--reps 5]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2410_14117_b200 as uuv  # noqa: E402
from paper_2410_14117_b200 import rollout as R  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--eager", action="store_true")
    ap.add_argument("--unfused", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--horizon", type=int, default=64)
    ap.add_argument("--no-pdl", action="store_true")
    a = ap.parse_args()
    env = uuv.batch_create(uuv.TaskSpec(kind="circle"), uuv.bluerov2_params(), None, 16384, 0,
                           device=0)
    cfg = R.TrainConfig(num_envs=16384, horizon=a.horizon)
    pol = R.ActorCritic(env.obs_dim, env.action_dim).cuda()
    ro = R.Rollout(env, pol, R.RunningNorm(env.obs_dim, "cuda"), cfg, use_graph=not a.eager,
                   fused=not a.unfused, pdl=not a.no_pdl)
    ro.reset(0)
    ro.collect()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.reps):
        ro.collect()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) * 1e3 / (a.reps * a.horizon)
    print(f"us per env-step batch {us:.2f}  env-steps/s {16384 / us * 1e6:.3e}")


if __name__ == "__main__":
    main()
