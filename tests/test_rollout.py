"""Device PPO rollout loop.

CPU: GAE and the running normaliser against restatements of the reference
formulas (reference ppo.py:112-130, nets.py:168-192).  GPU: graph-captured
collection == eager collection, and a short training run that must reduce the
station-keeping error of the untrained policy.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2410_14117_b200 import rollout as R


def _gae_reference(rewards, values, dones, boot, gamma, lam):
    """ppo.py:112-130 over (env, time) numpy arrays."""
    m, t_len = rewards.shape
    adv = np.zeros((m, t_len))
    last = np.zeros(m)
    for t in range(t_len - 1, -1, -1):
        nonterminal = 1.0 - dones[:, t]
        nv = boot if t == t_len - 1 else values[:, t + 1]
        delta = rewards[:, t] + gamma * nv * nonterminal - values[:, t]
        last = delta + gamma * lam * nonterminal * last
        adv[:, t] = last
    return adv, adv + values


def test_gae_matches_reference_formula():
    rng = np.random.default_rng(0)
    m, t = 37, 23
    r, v = rng.normal(size=(m, t)), rng.normal(size=(m, t))
    d = (rng.random((m, t)) < 0.1).astype(float)
    b = rng.normal(size=m)
    want_a, want_r = _gae_reference(r, v, d, b, 0.99, 0.95)
    got_a, got_r = R.gae(torch.tensor(r.T), torch.tensor(v.T), torch.tensor(d.T),
                         torch.tensor(b), 0.99, 0.95)
    np.testing.assert_allclose(got_a.numpy().T, want_a, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(got_r.numpy().T, want_r, rtol=1e-12, atol=1e-12)


def test_running_norm_matches_reference_formula():
    rng = np.random.default_rng(1)
    dim = 12
    mean, var, count = np.zeros(dim), np.ones(dim), 1e-4     # nets.py:171-175
    rn = R.RunningNorm(dim, "cpu")
    for _ in range(5):
        batch = rng.normal(2.0, 3.0, size=(64, dim))
        b_mean, b_var, n = batch.mean(0), batch.var(0), batch.shape[0]
        delta = b_mean - mean
        tot = count + n
        mean = mean + delta * (n / tot)
        var = (var * count + b_var * n + delta * delta * (count * n / tot)) / tot
        count = tot
        rn.update(torch.tensor(batch, dtype=torch.float32))
    np.testing.assert_allclose(rn.mean.numpy(), mean, rtol=1e-6)
    np.testing.assert_allclose(rn.var.numpy(), var, rtol=1e-6)
    x = torch.tensor(rng.normal(0, 100, size=(4, dim)), dtype=torch.float32)
    z = rn.normalize(x).numpy()
    assert np.all(np.abs(z) <= 10.0)


def test_policy_shapes_and_log_prob():
    pol = R.ActorCritic(12, 6, hidden=64, seed=0)
    obs = torch.randn(5, 12)
    mean, value = pol(obs)
    assert mean.shape == (5, 6) and value.shape == (5,)
    assert torch.all(mean.abs() <= 1.0)
    a = mean + 0.3
    lp = pol.log_prob(a, mean)
    std = torch.exp(pol.log_std)
    want = torch.distributions.Normal(mean, std).log_prob(a).sum(-1)
    torch.testing.assert_close(lp, want)


def _make_env(kind="station_keeping", dr=False):
    import paper_2410_14117_b200 as uuv

    def make(n, seed):
        spec = uuv.TaskSpec(kind=kind)
        ranges = uuv.default_ranges(per_episode=True) if dr else None
        return uuv.batch_create(spec, uuv.bluerov2_params(), ranges, n, seed, device=0)
    return make


@pytest.mark.gpu
def test_graph_collect_equals_eager():
    make = _make_env("circle")
    cfg = R.TrainConfig(num_envs=2048, horizon=16, init_log_std=-40.0)
    outs = []
    for use_graph in (False, True):
        env = make(cfg.num_envs, 3)
        pol = R.ActorCritic(env.obs_dim, env.action_dim, seed=1, init_log_std=-40.0).cuda()
        norm = R.RunningNorm(env.obs_dim, "cuda")
        ro = R.Rollout(env, pol, norm, cfg, use_graph=use_graph)
        ro.reset(3)
        ro.collect()
        if use_graph:        # first call warmed up + captured + replayed: restart in place
            env.reset_all(3)
            norm.mean.zero_()
            norm.var.fill_(1.0)
            norm.count.fill_(1e-4)
            ro.reset(3)
            ro.collect()
        torch.cuda.synchronize()
        outs.append([b.clone() for b in (ro.obs_buf, ro.rew_buf, ro.done_buf, ro.val_buf)])
        env.close()
    for a, b in zip(*outs):
        torch.testing.assert_close(a, b, rtol=1e-5, atol=1e-5)


@pytest.mark.gpu
def test_short_training_reduces_station_error():
    make = _make_env("station_keeping")
    # the reference's own PPO settings (ppo.py:33-50): 1024 envs x 64, minibatch 4096
    cfg = R.TrainConfig(num_envs=1024, horizon=64, total_env_steps=1024 * 64 * 20,
                        minibatch=4096, epochs=4, lr=3e-4)
    env0 = make(8, 0)
    pol0 = R.ActorCritic(env0.obs_dim, env0.action_dim, seed=0).cuda()
    env0.close()
    before = R.evaluate(pol0, R.RunningNorm(12, "cuda"), make, 256, 1000, 200)
    out = R.train(make, cfg)
    after = R.evaluate(out["policy"], out["normalizer"], make, 256, 1000, 200)
    assert np.isfinite(out["metrics"][-1]["loss"])
    assert after["mean_pos_err_m"] < 0.8 * before["mean_pos_err_m"], (before, after)
    assert out["collect_env_steps_per_sec"] > 2e6
