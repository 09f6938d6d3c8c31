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


def breakdown(ro, env, horizon=64, reps=5):
    """Incremental device cost of each launch of a fused collection step: graphs of
    `horizon` steps with all three launches, without post, without the policy,
    and the env step alone (CUDA-event time of graph replays)."""
    F = ro.fused
    F.prepare()
    obs0 = ro.env_obs

    def make(policy, step, post, norm=True, copy=True):
        def body():
            for t in range(horizon):
                if policy:
                    F.act(obs0, nobs=ro.obs_buf[t], raw=ro.act_buf[t], act=ro.act_in,
                          logp=ro.logp_buf[t], value=ro.val_buf[t])
                if step:
                    _, r, d, _ = env.step_tensors(ro.act_in)
                if post:
                    cp = copy and step
                    F.post(r if cp else None, d if cp else None, ro.rew_buf[t],
                           ro.done_buf[t], update_norm=norm)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            body()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            body()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e3 / (reps * horizon)

    full = make(True, True, True)
    no_post = make(True, True, False)
    no_pol = make(False, True, True)
    step = make(False, True, False)
    pol = make(True, False, False)
    sp_nonorm = make(False, True, True, norm=False)
    sp_nocopy = make(False, True, True, copy=False)
    sp_bare = make(False, True, True, norm=False, copy=False)
    print(f"all three {full:.2f} us/step | policy+step {no_post:.2f} | step+post {no_pol:.2f} "
          f"| step alone {step:.2f} | policy alone {pol:.2f} | step+post(no norm) "
          f"{sp_nonorm:.2f} | step+post(no copy) {sp_nocopy:.2f} | step+post(counter only) "
          f"{sp_bare:.2f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--eager", action="store_true")
    ap.add_argument("--unfused", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--horizon", type=int, default=64)
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--breakdown", action="store_true",
                    help="eager fused step with events around each launch (warm kernel times)")
    a = ap.parse_args()
    env = uuv.batch_create(uuv.TaskSpec(kind="circle"), uuv.bluerov2_params(), None, 16384, 0,
                           device=0)
    cfg = R.TrainConfig(num_envs=16384, horizon=a.horizon)
    pol = R.ActorCritic(env.obs_dim, env.action_dim).cuda()
    ro = R.Rollout(env, pol, R.RunningNorm(env.obs_dim, "cuda"), cfg, use_graph=not a.eager,
                   fused=not a.unfused, pdl=not a.no_pdl)
    ro.reset(0)
    if a.breakdown:
        breakdown(ro, env)
        return
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
