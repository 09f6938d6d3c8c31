"""ctypes face of the fused rollout-loop kernels (include/uuvsim_rl.h).

``FusedActorCritic`` binds an ``rollout.ActorCritic`` + ``RunningNorm`` (their
tensors are read in place, so optimizer updates are seen by captured graphs) and
exposes the two launches of one collection step:

    act(obs, t)   normalise + actor-critic + Gaussian sample + clamp + log-prob
                  (+ normaliser partial sums), outputs into the horizon buffers
    post(rew, done, t)   merge the normaliser update, copy reward/done, advance
                  the noise counter
"""

from __future__ import annotations

import ctypes

import torch

from . import _core

_f = ctypes.c_void_p


class PolicyArgs(ctypes.Structure):
    _fields_ = [("num_envs", ctypes.c_uint64), ("obs_dim", ctypes.c_uint32),
                ("act_dim", ctypes.c_uint32), ("hidden", ctypes.c_uint32),
                ("flags", ctypes.c_uint32), ("seed", ctypes.c_uint64),
                ("env_offset", ctypes.c_uint64), ("noise_ctr", _f), ("obs", _f),
                ("norm_mean", _f), ("norm_var", _f), ("norm_clip", ctypes.c_double),
                ("a1w", _f), ("a1b", _f), ("a2w", _f), ("a2b", _f), ("amw", _f), ("amb", _f),
                ("c1w", _f), ("c1b", _f), ("c2w", _f), ("c2b", _f), ("cvw", _f), ("cvb", _f),
                ("log_std", _f), ("nobs_out", _f), ("raw_out", _f), ("act_out", _f),
                ("logp_out", _f), ("value_out", _f), ("stats_part", _f), ("wimage", _f)]


class PostArgs(ctypes.Structure):
    _fields_ = [("num_envs", ctypes.c_uint64), ("obs_dim", ctypes.c_uint32),
                ("n_part", ctypes.c_uint32), ("stats_part", _f), ("norm_mean", _f),
                ("norm_var", _f), ("norm_count", _f), ("rew_in", _f), ("done_in", _f),
                ("rew_out", _f), ("done_out", _f), ("noise_ctr", _f),
                ("flags", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


SAMPLE, NORM_STATS, VALUE_ONLY, PDL = 1, 2, 4, 8


def _p(t):
    return None if t is None else t.data_ptr()


class FusedActorCritic:
    def __init__(self, policy, norm, num_envs: int, seed: int = 0, env_offset: int = 0,
                 tensor_cores: bool = True, pdl: bool = False):
        self.lib = _core.load()
        # programmatic dependent launch of the policy / post kernels (tensor-core
        # path): their CTAs start while the previous kernel of the step finishes
        self.pdl = bool(pdl) and tensor_cores
        self.policy, self.norm = policy, norm
        self.M = int(num_envs)
        self.D = policy.a1.weight.shape[1]
        self.A = policy.am.weight.shape[0]
        self.H = policy.a1.weight.shape[0]
        if self.H != 64 or self.D > 36 or self.A > 8:
            raise ValueError("fused policy kernel supports hidden 64, obs_dim <= 36, act_dim <= 8")
        for prm in policy.parameters():
            if prm.dtype != torch.float32 or not prm.is_cuda or not prm.is_contiguous():
                raise ValueError("fused policy kernel needs contiguous fp32 CUDA parameters")
        dev = policy.a1.weight.device
        self.seed, self.env_offset = int(seed), int(env_offset)
        self.noise_ctr = torch.zeros(1, dtype=torch.int64, device=dev)
        rows = int(self.lib.uuvsim_rl_policy_blocks(self.M))
        self.stats_part = torch.zeros(rows * 2 * self.D, dtype=torch.float64, device=dev)
        # rows the policy launch writes: one per 128-env CTA on the tensor cores,
        # one per 64-env block on the CUDA cores
        self.n_part = (self.M + 127) // 128 if tensor_cores else rows
        # tcgen05 path: weights split to 3xTF32 in the UMMA layout by prepare()
        self.image = None
        if tensor_cores:
            nb = int(self.lib.uuvsim_rl_image_bytes(self.D))
            self.image = torch.zeros(nb, dtype=torch.uint8, device=dev)

    def _args(self, obs, flags, nobs=None, raw=None, act=None, logp=None, value=None):
        pol, nm = self.policy, self.norm
        return PolicyArgs(
            self.M, self.D, self.A, self.H, flags, self.seed & (2**64 - 1), self.env_offset,
            _p(self.noise_ctr), _p(obs), _p(nm.mean), _p(nm.var), float(nm.clip),
            _p(pol.a1.weight), _p(pol.a1.bias), _p(pol.a2.weight), _p(pol.a2.bias),
            _p(pol.am.weight), _p(pol.am.bias), _p(pol.c1.weight), _p(pol.c1.bias),
            _p(pol.c2.weight), _p(pol.c2.bias), _p(pol.cv.weight), _p(pol.cv.bias),
            _p(pol.log_std), _p(nobs), _p(raw), _p(act), _p(logp), _p(value),
            _p(self.stats_part), _p(self.image))

    def prepare(self):
        """(Re)build the tensor-core weight image from the current parameters --
        once per horizon (stream-ordered, graph-capturable)."""
        if self.image is None:
            return
        a = self._args(None, 0)
        _core.check(self.lib, self.lib.uuvsim_rl_prepare(
            ctypes.byref(a), self.image.data_ptr(), self.image.numel(),
            torch.cuda.current_stream().cuda_stream))

    def act(self, obs, nobs=None, raw=None, act=None, logp=None, value=None,
            sample: bool = True, update_norm: bool = True, value_only: bool = False):
        flags = (SAMPLE if sample else 0) | (NORM_STATS if update_norm else 0) | \
                (VALUE_ONLY if value_only else 0) | (PDL if self.pdl else 0)
        a = self._args(obs, flags, nobs, raw, act, logp, value)
        _core.check(self.lib, self.lib.uuvsim_rl_policy_act(
            ctypes.byref(a), torch.cuda.current_stream().cuda_stream))

    def post(self, rew=None, done=None, rew_out=None, done_out=None, update_norm: bool = True):
        nm = self.norm
        # programmatic launch only behind the env step on the same stream (a bare
        # statistics merge runs on a side stream of the collection graph)
        pdl = self.pdl and rew is not None
        a = PostArgs(self.M, self.D, self.n_part if update_norm else 0, _p(self.stats_part),
                     _p(nm.mean), _p(nm.var), _p(nm.count), _p(rew), _p(done), _p(rew_out),
                     _p(done_out), _p(self.noise_ctr), 1 if pdl else 0, 0)
        _core.check(self.lib, self.lib.uuvsim_rl_post(
            ctypes.byref(a), torch.cuda.current_stream().cuda_stream))


__all__ = ["FusedActorCritic", "PolicyArgs", "PostArgs"]
