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


# ---------------------------------------------------------------- fused kernels ---

def _random_policy(obs_dim, act_dim, seed):
    pol = R.ActorCritic(obs_dim, act_dim, seed=seed).cuda()
    g = torch.Generator(device="cuda").manual_seed(seed)
    with torch.no_grad():
        for prm in pol.parameters():     # non-trivial biases / weights / log-std
            prm.add_(0.1 * torch.randn(prm.shape, device="cuda", generator=g))
    return pol


@pytest.mark.gpu
@pytest.mark.parametrize("tc", [False, True], ids=["cuda_cores", "tcgen05"])
@pytest.mark.parametrize("obs_dim,act_dim", [(12, 6), (36, 8), (24, 6), (30, 3), (18, 1)])
def test_fused_policy_matches_torch(obs_dim, act_dim, tc):
    from paper_2410_14117_b200.rl_fused import FusedActorCritic
    M = 1000
    pol = _random_policy(obs_dim, act_dim, 3)
    norm = R.RunningNorm(obs_dim, "cuda")
    g = torch.Generator(device="cuda").manual_seed(5)
    norm.mean.copy_(torch.randn(obs_dim, device="cuda", generator=g, dtype=torch.float64))
    norm.var.copy_(torch.rand(obs_dim, device="cuda", generator=g, dtype=torch.float64) + 0.1)
    norm.count.fill_(123.0)
    obs = 3.0 * torch.randn((M, obs_dim), device="cuda", generator=g)
    ref_norm = R.RunningNorm(obs_dim, "cuda")
    ref_norm.mean.copy_(norm.mean); ref_norm.var.copy_(norm.var); ref_norm.count.copy_(norm.count)
    F = FusedActorCritic(pol, norm, M, tensor_cores=tc)
    F.prepare()
    nobs = torch.empty((M, obs_dim), device="cuda")
    raw = torch.empty((M, act_dim), device="cuda")
    act = torch.empty_like(raw)
    logp = torch.empty(M, device="cuda")
    value = torch.empty(M, device="cuda")
    F.act(obs, nobs=nobs, raw=raw, act=act, logp=logp, value=value, sample=False)
    F.post()
    torch.cuda.synchronize()
    with torch.no_grad():
        want_nobs = ref_norm.normalize(obs)
        mean, v = pol(want_nobs)
        want_logp = pol.log_prob(mean, mean)
    ref_norm.update(obs)
    torch.testing.assert_close(nobs, want_nobs, rtol=1e-6, atol=1e-6)
    torch.testing.assert_close(raw, mean, rtol=1e-5, atol=1e-5)
    torch.testing.assert_close(act, mean.clamp(-1, 1), rtol=1e-5, atol=1e-5)
    torch.testing.assert_close(value, v, rtol=1e-5, atol=1e-5)
    torch.testing.assert_close(logp, want_logp, rtol=1e-6, atol=1e-5)
    torch.testing.assert_close(norm.mean, ref_norm.mean, rtol=1e-10, atol=1e-12)
    torch.testing.assert_close(norm.var, ref_norm.var, rtol=1e-9, atol=1e-12)
    torch.testing.assert_close(norm.count, ref_norm.count)
    assert int(F.noise_ctr.item()) == 1


@pytest.mark.gpu
def test_fused_noise_is_standard_normal_and_logp_consistent():
    from paper_2410_14117_b200.rl_fused import FusedActorCritic
    M, D, A = 16384, 12, 6
    pol = _random_policy(D, A, 1)
    with torch.no_grad():
        pol.log_std.zero_()
    norm = R.RunningNorm(D, "cuda")
    F = FusedActorCritic(pol, norm, M, seed=11)
    F.prepare()
    obs = torch.randn((M, D), device="cuda")
    raw = torch.empty((M, A), device="cuda")
    raw2 = torch.empty_like(raw)
    logp = torch.empty(M, device="cuda")
    F.act(obs, raw=raw, logp=logp, update_norm=False)
    F.post(update_norm=False)
    F.act(obs, raw=raw2, update_norm=False)
    torch.cuda.synchronize()
    with torch.no_grad():
        mean, _ = pol(norm.normalize(obs))
        eps = (raw - mean).double()
        want_logp = pol.log_prob(raw, mean)
    assert abs(float(eps.mean())) < 0.01
    assert 0.97 < float(eps.var()) < 1.03
    assert abs(float((eps ** 3).mean())) < 0.05            # symmetric
    assert 2.85 < float((eps ** 4).mean()) < 3.15           # Gaussian kurtosis
    torch.testing.assert_close(logp, want_logp, rtol=1e-5, atol=1e-4)
    assert not torch.equal(raw, raw2)                       # the counter advanced


@pytest.mark.gpu
def test_fused_collect_matches_framework_collect():
    make = _make_env("circle")
    cfg = R.TrainConfig(num_envs=2048, horizon=16, init_log_std=-40.0)
    outs = []
    for fused in (False, True):
        env = make(cfg.num_envs, 3)
        pol = R.ActorCritic(env.obs_dim, env.action_dim, seed=1, init_log_std=-40.0).cuda()
        norm = R.RunningNorm(env.obs_dim, "cuda")
        ro = R.Rollout(env, pol, norm, cfg, use_graph=False, fused=fused)
        ro.reset(3)
        ro.collect()
        torch.cuda.synchronize()
        outs.append([b.clone() for b in (ro.obs_buf, ro.rew_buf, ro.done_buf, ro.val_buf,
                                         ro.boot_value, norm.mean, norm.var)])
        env.close()
    for a, b in zip(*outs):
        torch.testing.assert_close(a.double(), b.double(), rtol=1e-4, atol=1e-4)


@pytest.mark.gpu
@pytest.mark.parametrize("use_graph", [False, True], ids=["eager", "graph"])
def test_programmatic_launch_is_bit_identical(use_graph):
    """The fused rollout with programmatic dependent launches (policy / step /
    post waiting in griddepcontrol instead of stream order) produces exactly the
    buffers of the plain launches: sampled actions, rewards, terminations,
    normaliser statistics."""
    make = _make_env("circle", dr=True)
    cfg = R.TrainConfig(num_envs=3000, horizon=24)
    outs = []
    for pdl in (False, True):
        env = make(cfg.num_envs, 5)
        pol = _random_policy(env.obs_dim, env.action_dim, 4)
        norm = R.RunningNorm(env.obs_dim, "cuda")
        ro = R.Rollout(env, pol, norm, cfg, use_graph=use_graph, fused=True, pdl=pdl)
        assert ro.fused.pdl == pdl
        ro.reset(5)
        ro.collect()
        ro.collect()        # graph: warm-up + capture + replay, then a second replay
        torch.cuda.synchronize()
        outs.append([b.clone() for b in (ro.obs_buf, ro.act_buf, ro.logp_buf, ro.rew_buf,
                                         ro.done_buf, ro.val_buf, ro.boot_value, norm.mean,
                                         norm.var, norm.count, ro.fused.noise_ctr)])
        env.close()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.gpu
def test_gae_fused_matches_reference():
    g = torch.Generator(device="cuda").manual_seed(2)
    T, M = 37, 1000
    r = torch.randn((T, M), device="cuda", generator=g)
    v = torch.randn((T, M), device="cuda", generator=g)
    d = (torch.rand((T, M), device="cuda", generator=g) < 0.1).float()
    b = torch.randn(M, device="cuda", generator=g)
    want_a, want_r = R.gae(r, v, d, b, 0.99, 0.95)
    got_a, got_r = R.gae_fused(r, v, d, b, 0.99, 0.95)
    torch.testing.assert_close(got_a, want_a, rtol=1e-5, atol=1e-5)
    torch.testing.assert_close(got_r, want_r, rtol=1e-5, atol=1e-5)


@pytest.mark.gpu
def test_graphed_update_equals_eager_update():
    make = _make_env("circle")
    cfg = R.TrainConfig(num_envs=1024, horizon=16, minibatch=4096, epochs=2, lr=3e-4)
    env = make(cfg.num_envs, 4)
    pol0 = R.ActorCritic(env.obs_dim, env.action_dim, seed=2).cuda()
    norm = R.RunningNorm(env.obs_dim, "cuda")
    ro = R.Rollout(env, pol0, norm, cfg, use_graph=False)
    ro.reset(4)
    ro.collect()
    results = []
    for graphed in (False, True):
        pol = R.ActorCritic(env.obs_dim, env.action_dim, seed=2).cuda()
        pol.load_state_dict(pol0.state_dict())
        opt = torch.optim.Adam(pol.parameters(), lr=cfg.lr, eps=1e-8, capturable=graphed)
        step = (R.GraphedMinibatchStep(pol, opt, cfg, cfg.minibatch, env.obs_dim,
                                       env.action_dim, torch.device("cuda")) if graphed else None)
        ro.policy = pol
        losses = []
        for it in range(3):   # covers warm-up, capture and replays
            gen = torch.Generator(device="cuda").manual_seed(9 + it)
            losses.append(R.ppo_update(pol, opt, ro, cfg, gen, step)["loss"])
        torch.cuda.synchronize()
        results.append((losses, [p.detach().clone() for p in pol.parameters()]))
    env.close()
    (l0, p0), (l1, p1) = results
    np.testing.assert_allclose(l1, l0, rtol=1e-4, atol=1e-5)
    # Adam moves every weight by ~lr per step whatever the gradient's size, so the
    # fp32 rounding differences of the fused GAE / capturable Adam can flip the
    # sign of near-zero gradients: parameters agree to a few learning rates
    for a, b in zip(p0, p1):
        torch.testing.assert_close(b, a, rtol=0, atol=10 * cfg.lr)
