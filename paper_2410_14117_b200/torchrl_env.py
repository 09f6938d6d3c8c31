"""RL-library adapters over the device face.

The reference's batch API folds every episode end into one ``done`` flag and
returns the POST-reset observation for finished envs (reference
pkg/src/uuvsim/batch.py:106-119); the reason code that tells a time-limit
truncation (0) from a divergence (1) or an integration failure (2) exists but
is not exported (tasks.py:41-42, 205).  Value bootstrapping in TorchRL /
Gymnasium-style loops needs both: ``terminated`` vs ``truncated`` and the
TERMINAL observation of an auto-reset env.

``VecEnv`` provides them on the device, with no extra pass over the slab: the
fused step kernel already writes the reason code, and with a registered
terminal-observation buffer (``uuvsim_dev_set_final_obs``) it also writes the
pre-reset observation of every finished env -- a branch taken by ~1/episode_len
of the envs per step.

``make_torchrl_env`` wraps a VecEnv as a TorchRL ``EnvBase`` when torchrl is
importable (it is not installed in this image, so that class is import-gated).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .batch import B200EnvBatch

REASON_TRUNCATED, REASON_DIVERGED, REASON_FAILED = 0, 1, 2


@dataclass
class StepOut:
    """One vector step.  All tensors live on the env's device; ``obs`` /
    ``final_obs`` / ``reward`` are reused buffers (clone to keep them)."""
    obs: torch.Tensor          # [M, D] post-reset for finished envs (reference semantics)
    next_obs: torch.Tensor     # [M, D] terminal obs for finished envs, else == obs
    reward: torch.Tensor       # [M]
    terminated: torch.Tensor   # [M] bool: divergence or integration failure
    truncated: torch.Tensor    # [M] bool: episode_len reached
    done: torch.Tensor         # [M] bool: terminated | truncated
    reason: torch.Tensor       # [M] int8: -1 running, 0 truncated, 1 diverged, 2 failed


class VecEnv:
    """Device vector env with the terminated/truncated split and terminal
    observations (Gymnasium vector ``final_obs`` semantics)."""

    def __init__(self, batch: B200EnvBatch):
        self.batch = batch
        self.num_envs, self.obs_dim, self.action_dim = (batch.num_envs, batch.obs_dim,
                                                        batch.action_dim)
        self.device = torch.device("cuda", batch.device_index)
        self.dtype = batch.dtype
        self.final_obs = torch.zeros((self.num_envs, self.obs_dim), dtype=self.dtype,
                                     device=self.device)
        batch.set_final_obs(self.final_obs)   # the batch keeps it alive while registered
        self._next = torch.empty_like(self.final_obs)
        self._term = torch.empty(self.num_envs, dtype=torch.bool, device=self.device)
        self._trunc = torch.empty_like(self._term)
        self._done = torch.empty_like(self._term)

    def reset(self, seed: int | None = None) -> torch.Tensor:
        return self.batch.reset_tensors(seed)

    def step(self, actions: torch.Tensor) -> StepOut:
        obs, rew, done, reason = self.batch.step_tensors(actions)
        torch.ge(reason, REASON_DIVERGED, out=self._term)
        torch.eq(reason, REASON_TRUNCATED, out=self._trunc)
        torch.ne(done, 0, out=self._done)
        torch.where(self._done[:, None], self.final_obs, obs, out=self._next)
        return StepOut(obs, self._next, rew, self._term, self._trunc, self._done, reason)

    def states(self) -> torch.Tensor:
        return self.batch.states_tensor()

    def close(self):
        if getattr(self.batch, "_open", False):
            self.batch.set_final_obs(None)
        self.batch.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def make_vec_env(spec, params, ranges=None, num_envs: int = 4096, seed: int = 0,
                 device: int = 0, **kw) -> VecEnv:
    from .batch import batch_create
    return VecEnv(batch_create(spec, params, ranges, num_envs, seed, device=device, **kw))


def _specs():
    """TorchRL spec classes across the 0.4 -> 0.6 renames."""
    import torchrl.data as D
    comp = getattr(D, "Composite", None) or D.CompositeSpec
    unb = getattr(D, "Unbounded", None) or D.UnboundedContinuousTensorSpec
    bnd = getattr(D, "Bounded", None) or D.BoundedTensorSpec
    cat = getattr(D, "Categorical", None) or D.DiscreteTensorSpec
    return comp, unb, bnd, cat


def make_torchrl_env(vec: VecEnv, seed: int = 0):
    """TorchRL ``EnvBase`` over a VecEnv (batch_size [M]).

    ``_step`` reports the TERMINAL observation under ``next`` with
    ``terminated`` / ``truncated`` / ``done``; the engine has already reset the
    finished envs, so the collector's partial ``_reset`` (``"_reset"`` mask)
    just hands back the cached post-reset observations.
    """
    try:
        from tensordict import TensorDict
        from torchrl.envs import EnvBase
    except ImportError as e:   # torchrl is optional (absent from this image)
        raise ImportError("make_torchrl_env needs torchrl and tensordict installed") from e
    comp, unb, bnd, cat = _specs()
    m, d, n = vec.num_envs, vec.obs_dim, vec.action_dim

    class UUVTorchRLEnv(EnvBase):
        batch_locked = True

        def __init__(self):
            super().__init__(device=vec.device, batch_size=torch.Size([m]))
            self.vec = vec
            self._seed = int(seed)
            self._post_reset = None
            self.observation_spec = comp(observation=unb(shape=(m, d), dtype=vec.dtype,
                                                         device=vec.device), shape=(m,))
            self.action_spec = bnd(low=-1.0, high=1.0, shape=(m, n), dtype=vec.dtype,
                                   device=vec.device)
            self.reward_spec = unb(shape=(m, 1), dtype=vec.dtype, device=vec.device)
            flag = dict(n=2, shape=(m, 1), dtype=torch.bool, device=vec.device)
            self.done_spec = comp(done=cat(**flag), terminated=cat(**flag),
                                  truncated=cat(**flag), shape=(m,))

        def _flags(self, done=None, term=None, trunc=None):
            z = torch.zeros((m, 1), dtype=torch.bool, device=vec.device)
            return {"done": z if done is None else done[:, None].clone(),
                    "terminated": z if term is None else term[:, None].clone(),
                    "truncated": z if trunc is None else trunc[:, None].clone()}

        def _reset(self, tensordict=None, **kw):
            mask = None if tensordict is None else tensordict.get("_reset", None)
            if mask is None or self._post_reset is None:
                obs = vec.reset(self._seed).clone()
            else:   # auto-reset already happened inside the fused step
                obs = self._post_reset
            return TensorDict({"observation": obs, **self._flags()}, batch_size=[m],
                              device=vec.device)

        def _step(self, tensordict):
            out = vec.step(tensordict.get("action").to(vec.dtype).contiguous())
            self._post_reset = out.obs.clone()
            return TensorDict({"observation": out.next_obs.clone(),
                               "reward": out.reward[:, None].clone(),
                               **self._flags(out.done, out.terminated, out.truncated)},
                              batch_size=[m], device=vec.device)

        def _set_seed(self, s):
            self._seed = int(s or 0)
            return s

    return UUVTorchRLEnv()


__all__ = ["VecEnv", "StepOut", "make_vec_env", "make_torchrl_env", "REASON_TRUNCATED",
           "REASON_DIVERGED", "REASON_FAILED"]
