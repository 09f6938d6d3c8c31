"""Device PPO rollout loop over the B200 step.

The reference trains with a numpy actor-critic on the host (reference
pkg/src/uuvsim/ppo.py:263-338, nets.py:31-192): every control step crosses the
C ABI with f64 host buffers.  Here the policy, the observation normaliser, the
Gaussian sampling, the rollout buffer and GAE live on the GPU next to the env
slab, and one rollout horizon -- ``horizon`` x (normalise -> policy -> sample ->
fused env step -> store) -- is captured as ONE CUDA graph and replayed.  The
PPO update runs eagerly with torch autograd.

Semantics kept from the reference:
* architecture (nets.py:31-55): separate actor / critic trunks, two tanh hidden
  layers of ``hidden``, tanh mean head, scalar value head, state-independent
  log-std; orthogonal init with gains sqrt(2) / 0.01 / 1;
* RunningNorm (nets.py:168-192): parallel-variance update, clip 10, count 1e-4;
* GAE (ppo.py:112-130) with ``done`` terminal; advantages normalised once per
  update (ppo.py:176); clipped surrogate + value loss - entropy (ppo.py:133-170);
* actions are sampled raw and clipped to [-1, 1] before the step (ppo.py:308-310).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import torch
from torch import nn

LOG_2PI = math.log(2.0 * math.pi)


@dataclass
class TrainConfig:
    """Reference TrainConfig (ppo.py:33-65) with GPU-sized defaults."""
    seed: int = 0
    total_env_steps: int = 5_000_000
    num_envs: int = 16384
    horizon: int = 64
    minibatch: int = 65536
    epochs: int = 4
    gamma: float = 0.99
    lam: float = 0.95
    clip: float = 0.2
    lr: float = 3e-4
    entropy_coef: float = 0.0
    value_coef: float = 0.5
    hidden: int = 64
    init_log_std: float = -0.5

    def __post_init__(self):
        if not (0.0 < self.gamma <= 1.0):
            raise ValueError("gamma must be in (0, 1]")
        if not (0.0 <= self.lam <= 1.0):
            raise ValueError("lam must be in [0, 1]")
        if not self.clip > 0.0:
            raise ValueError("clip must be positive")


def _orthogonal_(w: torch.Tensor, gain: float, gen: torch.Generator) -> None:
    rows, cols = w.shape
    a = torch.randn(max(rows, cols), min(rows, cols), generator=gen, dtype=torch.float64)
    q, r = torch.linalg.qr(a)
    q = q * torch.sign(torch.diagonal(r))
    q = q.T if rows < cols else q
    with torch.no_grad():
        w.copy_((gain * q[:rows, :cols]).to(w.dtype))


class ActorCritic(nn.Module):
    """Gaussian policy (tanh mean) + independent value critic (nets.py:31-71)."""

    def __init__(self, obs_dim: int, act_dim: int, hidden: int = 64, seed: int = 0,
                 init_log_std: float = -0.5):
        super().__init__()
        self.a1, self.a2, self.am = (nn.Linear(obs_dim, hidden), nn.Linear(hidden, hidden),
                                     nn.Linear(hidden, act_dim))
        self.c1, self.c2, self.cv = (nn.Linear(obs_dim, hidden), nn.Linear(hidden, hidden),
                                     nn.Linear(hidden, 1))
        self.log_std = nn.Parameter(torch.full((act_dim,), float(init_log_std)))
        gen = torch.Generator().manual_seed(seed)
        g = math.sqrt(2.0)
        for lin, gain in ((self.a1, g), (self.a2, g), (self.am, 0.01), (self.c1, g),
                          (self.c2, g), (self.cv, 1.0)):
            _orthogonal_(lin.weight, gain, gen)
            nn.init.zeros_(lin.bias)

    def forward(self, obs: torch.Tensor):
        mean = torch.tanh(self.am(torch.tanh(self.a2(torch.tanh(self.a1(obs))))))
        value = self.cv(torch.tanh(self.c2(torch.tanh(self.c1(obs)))))[:, 0]
        return mean, value

    def log_prob(self, actions: torch.Tensor, mean: torch.Tensor) -> torch.Tensor:
        z = (actions - mean) * torch.exp(-self.log_std)
        return (-0.5 * z * z - self.log_std - 0.5 * LOG_2PI).sum(-1)

    def entropy(self) -> torch.Tensor:
        return (self.log_std + 0.5 * (1.0 + LOG_2PI)).sum()


class RunningNorm:
    """Running mean/variance normaliser on the device (nets.py:168-192)."""

    def __init__(self, dim: int, device, clip: float = 10.0):
        self.mean = torch.zeros(dim, device=device, dtype=torch.float64)
        self.var = torch.ones(dim, device=device, dtype=torch.float64)
        self.count = torch.full((), 1e-4, device=device, dtype=torch.float64)
        self.clip = clip

    def update(self, batch: torch.Tensor) -> None:   # in place: graph-capturable
        b = batch.to(torch.float64)
        b_mean = b.mean(0)
        b_var = b.var(0, unbiased=False)
        n = float(b.shape[0])
        delta = b_mean - self.mean
        tot = self.count + n
        m2 = self.var * self.count + b_var * n + delta * delta * (self.count * n / tot)
        self.mean.add_(delta * (n / tot))
        self.var.copy_(m2 / tot)
        self.count.copy_(tot)

    def normalize(self, obs: torch.Tensor) -> torch.Tensor:
        z = (obs.to(torch.float64) - self.mean) / torch.sqrt(self.var + 1e-8)
        return z.clamp(-self.clip, self.clip).to(obs.dtype)


def gae(rewards, values, dones, bootstrap_value, gamma: float, lam: float):
    """GAE over [T, M] tensors (ppo.py:112-130): done_t is terminal."""
    t_len = rewards.shape[0]
    adv = torch.empty_like(rewards)
    last = torch.zeros_like(bootstrap_value)
    for t in range(t_len - 1, -1, -1):
        nonterminal = 1.0 - dones[t]
        next_value = bootstrap_value if t == t_len - 1 else values[t + 1]
        delta = rewards[t] + gamma * next_value * nonterminal - values[t]
        last = delta + gamma * lam * nonterminal * last
        adv[t] = last
    return adv, adv + values


class Rollout:
    """Horizon buffers + the graph-captured collection loop for one env slab."""

    def __init__(self, env, policy: ActorCritic, norm: RunningNorm, cfg: TrainConfig,
                 use_graph: bool = True, fused: bool | None = None, pdl: bool = True):
        self.env, self.policy, self.norm, self.cfg = env, policy, norm, cfg
        dev = torch.device("cuda", env.device_index)
        T, M = cfg.horizon, env.num_envs
        f = torch.float32
        self.obs_buf = torch.zeros((T, M, env.obs_dim), device=dev, dtype=f)
        self.act_buf = torch.zeros((T, M, env.action_dim), device=dev, dtype=f)
        self.logp_buf = torch.zeros((T, M), device=dev, dtype=f)
        self.rew_buf = torch.zeros((T, M), device=dev, dtype=f)
        self.val_buf = torch.zeros((T, M), device=dev, dtype=f)
        self.done_buf = torch.zeros((T, M), device=dev, dtype=f)
        self.obs = torch.zeros((M, env.obs_dim), device=dev, dtype=f)   # current obs
        self.act_in = torch.zeros((M, env.action_dim), device=dev, dtype=f)
        self.boot_value = torch.zeros(M, device=dev, dtype=f)
        self.graph = None
        self.use_graph = use_graph
        # fused path (csrc/rl_kernels.cu): policy + sampling + normaliser in one kernel
        # and one small post kernel around each env step, instead of ~40 framework kernels
        if fused is None:
            fused = env.obs_dim <= 36 and env.action_dim <= 8 and policy.a1.weight.shape[0] == 64
        self.fused = None
        if fused:
            from .rl_fused import FusedActorCritic
            # pdl: policy / step / post launched as programmatic dependents, so
            # each kernel's CTAs are resident before its predecessor finishes
            self.fused = FusedActorCritic(policy, norm, M, seed=cfg.seed + 7,
                                          env_offset=getattr(env, "env_offset", 0), pdl=pdl)
        self.env_obs = None

    def reset(self, seed: int):
        self.env_obs = self.env.reset_tensors(seed)
        self.obs.copy_(self.env_obs)

    @torch.no_grad()
    def _collect(self):
        if self.fused is not None:
            self._collect_fused()
            return
        pol, norm, env = self.policy, self.norm, self.env
        std = torch.exp(pol.log_std)
        for t in range(self.cfg.horizon):
            nobs = norm.normalize(self.obs)
            norm.update(self.obs)
            mean, value = pol(nobs)
            raw = mean + std * torch.randn_like(mean)
            self.act_in.copy_(raw.clamp(-1.0, 1.0))
            o, r, d, _ = env.step_tensors(self.act_in)
            self.obs_buf[t].copy_(nobs)
            self.act_buf[t].copy_(raw)
            self.logp_buf[t].copy_(pol.log_prob(raw, mean))
            self.val_buf[t].copy_(value)
            self.rew_buf[t].copy_(r)
            self.done_buf[t].copy_(d)
            self.obs.copy_(o)
        self.boot_value.copy_(pol(norm.normalize(self.obs))[1])

    @torch.no_grad()
    def _collect_fused(self):
        F, env = self.fused, self.env
        obs = self.env_obs
        F.prepare()   # parameters changed since the last horizon (PPO update)
        pdl = F.pdl and hasattr(env, "set_pdl")
        # the step writes reward and fp32 done straight into the horizon buffers,
        # and the normaliser merge (which needs only the policy's partial sums)
        # runs on a side stream beside the step: two launches on the critical path
        # per step instead of three
        direct = hasattr(env, "set_done_f32")
        cur = torch.cuda.current_stream()
        side = self._side_stream() if direct else None
        if pdl:
            env.set_pdl(True)
        try:
            for t in range(self.cfg.horizon):
                F.act(obs, nobs=self.obs_buf[t], raw=self.act_buf[t], act=self.act_in,
                      logp=self.logp_buf[t], value=self.val_buf[t])
                if direct:
                    side.wait_stream(cur)
                    with torch.cuda.stream(side):
                        F.post()
                    env.set_done_f32(self.done_buf[t])
                    obs, r, d, _ = env.step_tensors(self.act_in, rew_out=self.rew_buf[t])
                    cur.wait_stream(side)
                else:
                    obs, r, d, _ = env.step_tensors(self.act_in)
                    F.post(r, d, self.rew_buf[t], self.done_buf[t])
            F.act(obs, value=self.boot_value, sample=False, update_norm=False, value_only=True)
        finally:
            if pdl:
                env.set_pdl(False)
            if direct:
                env.set_done_f32(None)
        self.env_obs = obs

    def _side_stream(self):
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=torch.device("cuda", self.env.device_index))
        return self._side

    def collect(self):
        """One horizon; the first call with use_graph captures it as a CUDA graph."""
        if not self.use_graph:
            self._collect()
            return
        if self.graph is None:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):   # warm-up outside capture (allocator, cuBLAS)
                self._collect()
            torch.cuda.current_stream().wait_stream(s)
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                self._collect()
        self.graph.replay()


def gae_fused(rewards, values, dones, bootstrap_value, gamma: float, lam: float):
    """gae() as one kernel (csrc/rl_kernels.cu k_gae: a thread per env walks the
    horizon backwards) instead of ~6 framework ops per time step."""
    import ctypes
    from . import _core
    lib = _core.load()
    T, M = rewards.shape
    for t in (rewards, values, dones, bootstrap_value):
        if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
            raise ValueError("gae_fused needs contiguous fp32 CUDA tensors")
    adv, ret = torch.empty_like(rewards), torch.empty_like(rewards)
    _core.check(lib, lib.uuvsim_rl_gae(
        rewards.data_ptr(), values.data_ptr(), dones.data_ptr(), bootstrap_value.data_ptr(),
        T, M, ctypes.c_float(gamma), ctypes.c_float(lam), adv.data_ptr(), ret.data_ptr(),
        torch.cuda.current_stream().cuda_stream))
    return adv, ret


class GraphedMinibatchStep:
    """One PPO minibatch step -- forward, clipped surrogate + value loss, backward,
    Adam -- captured as a CUDA graph on static minibatch buffers (ppo.py:133-196).
    The shuffled minibatch rows are gathered into the static buffers eagerly;
    the first three steps run eagerly on a side stream to allocate optimizer
    state, the fourth is captured, and every later one is a replay."""

    WARMUP = 3

    def __init__(self, policy: ActorCritic, opt, cfg: TrainConfig, mb: int, obs_dim: int,
                 act_dim: int, dev):
        self.policy, self.opt, self.cfg = policy, opt, cfg
        f = torch.float32
        self.obs = torch.zeros((mb, obs_dim), device=dev, dtype=f)
        self.act = torch.zeros((mb, act_dim), device=dev, dtype=f)
        self.logp_old = torch.zeros(mb, device=dev, dtype=f)
        self.adv = torch.zeros(mb, device=dev, dtype=f)
        self.ret = torch.zeros(mb, device=dev, dtype=f)
        self.agg = torch.zeros(5, device=dev, dtype=torch.float64)
        self.graph = None
        self.steps = 0
        self.side = torch.cuda.Stream(device=dev)

    def _body(self):
        pol, cfg = self.policy, self.cfg
        mean, value = pol(self.obs)
        logp = pol.log_prob(self.act, mean)
        ratio = torch.exp(logp - self.logp_old)
        s1 = ratio * self.adv
        s2 = ratio.clamp(1.0 - cfg.clip, 1.0 + cfg.clip) * self.adv
        surrogate = -torch.minimum(s1, s2).mean()
        value_loss = ((value - self.ret) ** 2).mean()
        loss = surrogate + cfg.value_coef * value_loss - cfg.entropy_coef * pol.entropy()
        self.opt.zero_grad(set_to_none=False)
        loss.backward()
        self.opt.step()
        with torch.no_grad():
            self.agg.add_(torch.stack([
                loss.detach(), surrogate.detach(), value_loss.detach(),
                (self.logp_old - logp).mean().detach(),
                ((ratio - 1.0).abs() > cfg.clip).float().mean()]).double())

    def __call__(self):
        if self.graph is not None:
            self.graph.replay()
        elif self.steps < self.WARMUP:
            self.side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(self.side):
                self._body()
            torch.cuda.current_stream().wait_stream(self.side)
        else:
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                self._body()
            self.graph.replay()
        self.steps += 1


def ppo_update(policy: ActorCritic, opt, ro: Rollout, cfg: TrainConfig,
               gen: torch.Generator, step: GraphedMinibatchStep | None = None) -> dict:
    """Shuffled minibatch epochs (ppo.py:173-196) with torch autograd; with ``step``
    each minibatch is one replay of a captured graph (see GraphedMinibatchStep)."""
    if step is not None:
        return _ppo_update_graphed(policy, ro, cfg, gen, step)
    adv, ret = gae(ro.rew_buf, ro.val_buf, ro.done_buf, ro.boot_value, cfg.gamma, cfg.lam)
    obs = ro.obs_buf.reshape(-1, ro.obs_buf.shape[-1])
    act = ro.act_buf.reshape(-1, ro.act_buf.shape[-1])
    logp_old = ro.logp_buf.reshape(-1)
    adv = adv.reshape(-1)
    ret = ret.reshape(-1)
    adv = (adv - adv.mean()) / (adv.std(unbiased=False) + 1e-8)
    n = obs.shape[0]
    mb = min(cfg.minibatch, n)
    agg = {"loss": 0.0, "policy_loss": 0.0, "value_loss": 0.0, "approx_kl": 0.0,
           "clip_fraction": 0.0}
    count = 0
    for _ in range(cfg.epochs):
        order = torch.randperm(n, device=obs.device, generator=gen)
        for lo in range(0, n, mb):
            idx = order[lo:lo + mb]
            mean, value = policy(obs[idx])
            logp = policy.log_prob(act[idx], mean)
            ratio = torch.exp(logp - logp_old[idx])
            s1 = ratio * adv[idx]
            s2 = ratio.clamp(1.0 - cfg.clip, 1.0 + cfg.clip) * adv[idx]
            surrogate = -torch.minimum(s1, s2).mean()
            value_loss = ((value - ret[idx]) ** 2).mean()
            loss = surrogate + cfg.value_coef * value_loss - cfg.entropy_coef * policy.entropy()
            opt.zero_grad(set_to_none=True)
            loss.backward()
            opt.step()
            with torch.no_grad():
                agg["loss"] += loss.detach()
                agg["policy_loss"] += surrogate.detach()
                agg["value_loss"] += value_loss.detach()
                agg["approx_kl"] += (logp_old[idx] - logp).mean().detach()
                agg["clip_fraction"] += ((ratio - 1.0).abs() > cfg.clip).float().mean()
            count += 1
    out = {k: float(v) / count for k, v in agg.items()}
    if not math.isfinite(out["loss"]):
        raise RuntimeError("non-finite PPO loss")
    return out


def _ppo_update_graphed(policy, ro: Rollout, cfg: TrainConfig, gen, step: GraphedMinibatchStep):
    adv, ret = gae_fused(ro.rew_buf, ro.val_buf, ro.done_buf, ro.boot_value, cfg.gamma, cfg.lam)
    obs = ro.obs_buf.reshape(-1, ro.obs_buf.shape[-1])
    act = ro.act_buf.reshape(-1, ro.act_buf.shape[-1])
    logp_old = ro.logp_buf.reshape(-1)
    adv = adv.reshape(-1)
    ret = ret.reshape(-1)
    adv = (adv - adv.mean()) / (adv.std(unbiased=False) + 1e-8)
    n = obs.shape[0]
    mb = step.obs.shape[0]
    step.agg.zero_()
    count = 0
    for _ in range(cfg.epochs):
        order = torch.randperm(n, device=obs.device, generator=gen)
        for lo in range(0, n - mb + 1, mb):   # full minibatches (static graph shapes)
            idx = order[lo:lo + mb]
            torch.index_select(obs, 0, idx, out=step.obs)
            torch.index_select(act, 0, idx, out=step.act)
            torch.index_select(logp_old, 0, idx, out=step.logp_old)
            torch.index_select(adv, 0, idx, out=step.adv)
            torch.index_select(ret, 0, idx, out=step.ret)
            step()
            count += 1
    vals = (step.agg / max(count, 1)).tolist()
    out = dict(zip(("loss", "policy_loss", "value_loss", "approx_kl", "clip_fraction"), vals))
    if not math.isfinite(out["loss"]):
        raise RuntimeError("non-finite PPO loss")
    return out


@torch.no_grad()
def evaluate(policy: ActorCritic, norm: RunningNorm, make_env, episodes: int, seed: int,
             episode_len: int) -> dict:
    """Deterministic mean-action rollouts (ppo.py:211-242): position error per step."""
    env = make_env(episodes, seed)
    obs = env.reset_tensors(seed).clone()
    err = torch.zeros(episode_len, device=obs.device, dtype=torch.float64)
    ret = torch.zeros(episodes, device=obs.device, dtype=torch.float64)
    act = torch.zeros((episodes, env.action_dim), device=obs.device, dtype=torch.float32)
    for t in range(episode_len):
        mean, _ = policy(norm.normalize(obs))
        act.copy_(mean.clamp(-1.0, 1.0))
        o, r, d, _ = env.step_tensors(act)
        err[t] = (-r.double()).mean()
        ret += r.double()
        obs = o.clone()
    env.close()
    return {"mean_pos_err_m": float(err.mean()), "final_pos_err_m": float(err[-1]),
            "mean_return": float(ret.mean()), "episodes": episodes}


def train(make_env, cfg: TrainConfig, use_graph: bool = True, log_cb=None,
          eval_every: int = 0, eval_episodes: int = 256, episode_len: int = 600,
          fused: bool | None = None, graph_update: bool | None = None) -> dict:
    """collect -> GAE -> PPO update until cfg.total_env_steps (ppo.py:245-338)."""
    env = make_env(cfg.num_envs, cfg.seed)
    dev = torch.device("cuda", env.device_index)
    policy = ActorCritic(env.obs_dim, env.action_dim, cfg.hidden, cfg.seed,
                         cfg.init_log_std).to(dev)
    n_samples = cfg.num_envs * cfg.horizon
    if graph_update is None:   # graphed minibatch steps need full, equal minibatches
        graph_update = use_graph and n_samples % min(cfg.minibatch, n_samples) == 0
    opt = torch.optim.Adam(policy.parameters(), lr=cfg.lr, eps=1e-8,
                           capturable=bool(graph_update))
    step = (GraphedMinibatchStep(policy, opt, cfg, min(cfg.minibatch, n_samples), env.obs_dim,
                                 env.action_dim, dev) if graph_update else None)
    norm = RunningNorm(env.obs_dim, dev)
    torch.manual_seed(cfg.seed + 1)
    gen = torch.Generator(device=dev).manual_seed(cfg.seed + 2)
    ro = Rollout(env, policy, norm, cfg, use_graph, fused=fused)
    ro.reset(cfg.seed)
    env_steps, it = 0, 0
    t_collect = t_update = 0.0
    metrics = []
    while env_steps < cfg.total_env_steps:
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        ro.collect()
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        losses = ppo_update(policy, opt, ro, cfg, gen, step)
        torch.cuda.synchronize(dev)
        t2 = time.perf_counter()
        if it > 0:   # the first horizon includes graph capture
            t_collect += t1 - t0
        if it > 0:   # the first update includes warm-up + graph capture
            t_update += t2 - t1
        env_steps += cfg.num_envs * cfg.horizon
        it += 1
        rec = {"iteration": it, "env_steps": env_steps, **losses}
        if eval_every and it % eval_every == 0:
            rec.update(evaluate(policy, norm, make_env, eval_episodes, cfg.seed + 1000,
                                episode_len))
        metrics.append(rec)
        if log_cb:
            log_cb(rec)
    timed_steps = max(it - 1, 1) * cfg.num_envs * cfg.horizon
    env.close()
    return {"policy": policy, "normalizer": norm, "metrics": metrics, "env_steps": env_steps,
            "collect_env_steps_per_sec": timed_steps / max(t_collect, 1e-12),
            "update_s_per_iter": t_update / max(it - 1, 1)}


__all__ = ["TrainConfig", "ActorCritic", "RunningNorm", "gae", "gae_fused", "Rollout",
           "GraphedMinibatchStep", "ppo_update", "evaluate", "train"]
