"""Batched environments on the B200 engine -- the reference's batch API, GPU-backed.

``batch_create`` / ``B200EnvBatch`` keep the duck-typed protocol every caller
of the reference uses (reference pkg/src/uuvsim/batch.py:36-137,
_native.py:122-213): attributes ``backend, num_envs, obs_dim, action_dim,
episode_len, root_seed, threads``; ``reset_all(seed)``, ``step(actions) ->
(obs, rew, done)``, ``states()``, ``step_counts()``, ``set_threads(n)``,
``close()`` and the context manager.  Those host-f64 calls go through the C
ABI v1 (``uuvsim_step`` with host buffers, copies included).

The same handle also exposes the device face for GPU-resident training loops:
``reset_tensors`` / ``step_tensors`` take and return CUDA tensors (zero-copy,
launched on the current torch stream, capturable by ``torch.cuda.graph``),
and ``capture_graph`` / ``replay_graph`` run K steps as one native CUDA graph.
"""

from __future__ import annotations

import ctypes
import json
import sys
import os
import time

import numpy as np

from . import _core
from .config import (ConfigError, RandomizationRanges, TaskSpec, VehicleParams,
                     engine_config_dict)

STAT_NAMES = ("sum_reward", "done_truncation", "done_divergence", "done_failure",
              "sum_episode_return", "sum_episode_length", "env_steps", "resample_rejected",
              "band64_steps")


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class B200EnvBatch:
    """M environments resident on one GPU, stepped by the fused sm_100a kernel."""

    backend = "b200"
    _fast = None   # C fast path of step_ex (set with the pinned output pool)

    def __init__(self, config: dict | str, root_seed: int | None = None, threads: int = 0,
                 pinned: bool = True):
        lib = _core.load()
        self._lib = lib
        text = config if isinstance(config, str) else json.dumps(config)
        cfg = json.loads(text)
        handle = ctypes.c_uint64(0)
        _core.check(lib, lib.uuvsim_create(text.encode("utf-8"), ctypes.byref(handle)))
        self._handle = handle.value
        self._open = True
        self._registered = {}   # device buffers the engine writes into (kept alive here)
        spec = (ctypes.c_uint64 * 4)()
        _core.check(lib, lib.uuvsim_spec(self._handle, spec))
        self.num_envs, self.obs_dim, self.action_dim, self.episode_len = (int(x) for x in spec)
        self.root_seed = int(cfg["seed"] if root_seed is None else root_seed)
        self.threads = int(threads)
        self.env_offset = int((cfg.get("batch") or {}).get("env_offset", 0))
        self.info = json.loads(self._info())
        self.precision = self.info["precision"]
        self.device_index = int(self.info["device"])
        self._obs = np.zeros((self.num_envs, self.obs_dim))
        self._rew = np.zeros(self.num_envs)
        self._done = np.zeros(self.num_envs, dtype=np.uint8)
        self._reason = np.zeros(self.num_envs, dtype=np.int8)
        if pinned:   # page-locked output staging: the D2H copies DMA straight in
            try:
                self.use_pinned_host_buffers()
            except Exception:
                pass
        self._t = None          # device tensors (lazy)
        self._bufptrs = None
        if self.root_seed != int(cfg["seed"]):
            self.reset_all(self.root_seed)
        # else: the engine reset every env with the config seed at create; skipping
        # the host reset keeps a device-face-only batch free of host-ABI staging

    # -------------------------------------------------------------- reference protocol
    def reset_all(self, seed: int) -> np.ndarray:
        self._require_open()
        self.root_seed = int(seed)
        _core.check(self._lib, self._lib.uuvsim_reset(self._handle, int(seed) & (2**64 - 1),
                                                      _ptr(self._obs), self._obs.size))
        return self._obs.copy()

    def step(self, actions):
        obs, rew, done, _ = self.step_ex(actions)
        return obs, rew, done

    def step_ex(self, actions):
        """step() plus the termination reason per env (-1, 0 trunc, 1 div, 2 fail)."""
        self._require_open()
        fast = self._fast
        if fast is not None:
            # C fast path (csrc/hostcall.c): float64 C-contiguous [M, A] actions straight
            # into uuvsim_step_ex, outputs into a pooled block (anything else returns
            # -100 and takes the general path below)
            arrs, ptrs = self._free_block()
            rc = fast(self._handle, actions, self.num_envs, self.action_dim, ptrs)
            if rc == 0:
                return arrs[0], arrs[1], arrs[2], arrs[3]
            if rc != -100:
                _core.check(self._lib, rc)
        act = np.ascontiguousarray(actions, dtype=np.float64)
        if act.shape != (self.num_envs, self.action_dim):
            raise ValueError(f"actions must have shape {(self.num_envs, self.action_dim)}, "
                             f"got {act.shape}")
        if getattr(self, "_pool", None) is not None:
            # outputs land in a page-locked block the engine writes directly
            # (zero-copy or one DMA); the returned arrays ARE that block, so no
            # host copy.  A block is reused only once the caller holds none of
            # its arrays (reference semantics: every step returns fresh arrays)
            arrs, ptrs = self._free_block()
            _core.check(self._lib, self._lib.uuvsim_step_ex(
                self._handle, act.ctypes.data, act.size, *ptrs))
            # a fresh tuple: holding it must count as holding the arrays
            return arrs[0], arrs[1], arrs[2], arrs[3]
        if getattr(self, "_bufptrs", None) is None:   # fixed output buffers: marshal once
            self._bufptrs = (self._obs.ctypes.data, self._obs.size, self._rew.ctypes.data,
                             self._rew.size, self._done.ctypes.data, self._done.size,
                             self._reason.ctypes.data, self._reason.size)
        _core.check(self._lib, self._lib.uuvsim_step_ex(
            self._handle, act.ctypes.data, act.size, *self._bufptrs))
        return (self._obs.copy(), self._rew.copy(), self._done.astype(bool),
                self._reason.copy())

    def states(self) -> np.ndarray:
        self._require_open()
        out = np.zeros((self.num_envs, 12))
        _core.check(self._lib, self._lib.uuvsim_states(self._handle, _ptr(out), out.size))
        return out

    def step_counts(self) -> np.ndarray:
        self._require_open()
        out = np.zeros(self.num_envs, dtype=np.int64)
        _core.check(self._lib, self._lib.uuvsim_step_counts(self._handle, _ptr(out), out.size))
        return out

    def set_threads(self, n: int):
        self._require_open()
        _core.check(self._lib, self._lib.uuvsim_set_threads(self._handle, int(n)))
        self.threads = int(n)

    def close(self):
        if getattr(self, "_open", False):
            self._lib.uuvsim_destroy(self._handle)
            self._open = False
            self._registered = {}

    def _require_open(self):
        if not self._open:
            raise RuntimeError("batch has been closed")

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def use_pinned_host_buffers(self) -> None:
        """Back the host-ABI output arrays with page-locked memory (faster DMA)."""
        import torch
        n = self.num_envs
        self._pinned = [torch.empty((n, self.obs_dim), dtype=torch.float64, pin_memory=True),
                        torch.empty(n, dtype=torch.float64, pin_memory=True),
                        torch.empty(n, dtype=torch.uint8, pin_memory=True),
                        torch.empty(n, dtype=torch.int8, pin_memory=True)]
        self._obs, self._rew, self._done, self._reason = (t.numpy() for t in self._pinned)
        self._bufptrs = None
        # step outputs: pool of pinned blocks [obs f64 | rew f64 | done u8 | reason i8]
        self._pool = []
        self._torch = torch
        self._fast = _fast_step(self._lib)

    def _new_block(self):
        n, d = self.num_envs, self.obs_dim
        o_rew = n * d * 8
        o_done = o_rew + n * 8
        o_rsn = o_done + n
        t = self._torch.empty(o_rsn + n, dtype=self._torch.uint8, pin_memory=True)
        blk = t.numpy()
        base = blk.ctypes.data
        arrs = (blk[:o_rew].view(np.float64).reshape(n, d), blk[o_rew:o_done].view(np.float64),
                blk[o_done:o_rsn].view(np.bool_), blk[o_rsn:o_rsn + n].view(np.int8))
        ptrs = (base, n * d, base + o_rew, n, base + o_done, n, base + o_rsn, n)
        return [t, blk, (arrs, ptrs), None]

    _POOL_MAX = 8

    def _free_block(self):
        """A pool block the caller holds no array (or sub-view) of."""
        for entry in self._pool:
            if _pool_refs(entry) == entry[3]:
                return entry[2]
        entry = self._new_block()
        entry[3] = _pool_refs(entry)     # reference counts while only the pool holds it
        if len(self._pool) < self._POOL_MAX:
            self._pool.append(entry)
        return entry[2]

    # -------------------------------------------------------------- inspection / resume
    def set_states(self, states) -> None:
        self._require_open()
        s = np.ascontiguousarray(states, dtype=np.float64).reshape(self.num_envs, 12)
        _core.check(self._lib, self._lib.uuvsim_set_states(self._handle, _ptr(s), s.size))

    def set_step_counts(self, steps) -> None:
        self._require_open()
        s = np.ascontiguousarray(steps, dtype=np.int64)
        _core.check(self._lib, self._lib.uuvsim_set_step_counts(self._handle, _ptr(s), s.size))

    def counters(self):
        rc = np.zeros(self.num_envs, dtype=np.uint64)
        pc = np.zeros(self.num_envs, dtype=np.uint64)
        _core.check(self._lib, self._lib.uuvsim_counters(self._handle, _ptr(rc), _ptr(pc),
                                                         self.num_envs))
        return rc, pc

    def dr_factors(self) -> np.ndarray:
        out = np.zeros((self.num_envs, 10))
        _core.check(self._lib, self._lib.uuvsim_dr_factors(self._handle, _ptr(out), out.size))
        return out

    def wrench(self, actions) -> np.ndarray:
        """Body wrench tau [N, 6] of every env for the given actions (the step
        kernel's thruster map, reference thrusters.py:97-119)."""
        act = np.ascontiguousarray(actions, dtype=np.float64)
        if act.shape != (self.num_envs, self.action_dim):
            raise ValueError(f"actions must have shape {(self.num_envs, self.action_dim)}")
        out = np.zeros((self.num_envs, 6))
        _core.check(self._lib, self._lib.uuvsim_wrench(self._handle, _ptr(act), act.size,
                                                       _ptr(out), out.size))
        return out

    def stats(self, clear: bool = False) -> dict:
        out = np.zeros(len(STAT_NAMES))
        _core.check(self._lib, self._lib.uuvsim_stats(self._handle, _ptr(out), len(STAT_NAMES), int(clear)))
        return dict(zip(STAT_NAMES, out.tolist()))

    def _info(self) -> str:
        buf = ctypes.create_string_buffer(8192)
        n = self._lib.uuvsim_info(self._handle, buf, 8192)
        if n < 0:
            _core.check(self._lib, int(-n))
        return buf.raw[:n].decode()

    def synchronize(self):
        _core.check(self._lib, self._lib.uuvsim_synchronize(self._handle))

    # -------------------------------------------------------------- device face (torch)
    def _tensors(self):
        if self._t is None:
            import torch
            dev = torch.device("cuda", self.device_index)
            n = self.num_envs
            dt = self.dtype
            self._t = {
                "obs": torch.zeros((n, self.obs_dim), dtype=dt, device=dev),
                "rew": torch.zeros(n, dtype=dt, device=dev),
                "done": torch.zeros(n, dtype=torch.uint8, device=dev),
                "reason": torch.zeros(n, dtype=torch.int8, device=dev),
                "stats": torch.zeros(len(STAT_NAMES), dtype=torch.float64, device=dev),
            }
        return self._t

    @property
    def dtype(self):
        """torch dtype of the device face: float32 (fp32 engine) or float64 (fp64)."""
        import torch
        return torch.float64 if self.precision == "fp64" else torch.float32

    @staticmethod
    def _stream(stream=None) -> int:
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        return int(s.cuda_stream)

    def _check_actions(self, actions):
        import torch
        if (not isinstance(actions, torch.Tensor) or actions.dtype != self.dtype
                or not actions.is_cuda or actions.device.index != self.device_index
                or tuple(actions.shape) != (self.num_envs, self.action_dim)
                or not actions.is_contiguous()):
            raise ValueError(f"actions must be a contiguous {self.dtype} CUDA tensor of shape "
                             f"{(self.num_envs, self.action_dim)} on cuda:{self.device_index}")

    def reset_tensors(self, seed: int | None = None, stream=None):
        """reset_all on the device; returns the (reused) obs tensor [M, obs_dim] f32."""
        self._require_open()
        t = self._tensors()
        if seed is not None:
            self.root_seed = int(seed)
        _core.check(self._lib, self._lib.uuvsim_dev_reset(
            self._handle, self.root_seed & (2**64 - 1), t["obs"].data_ptr(), t["obs"].numel(),
            self._stream(stream)))
        return t["obs"]

    def step_tensors(self, actions, stream=None, rew_out=None):
        """One fused step on device tensors -> (obs, rew, done u8, reason i8) (reused).

        Element dtype is ``self.dtype`` (float32 for the default fp32 engine).
        ``rew_out``: a caller tensor of num_envs elements the reward goes to
        instead (e.g. a rollout buffer row); it is returned as ``rew``."""
        self._require_open()
        self._check_actions(actions)
        t = self._tensors()
        rew = t["rew"]
        if rew_out is not None:
            if (rew_out.dtype != rew.dtype or rew_out.numel() != rew.numel() or
                    not rew_out.is_contiguous() or rew_out.device != rew.device):
                raise ValueError(f"rew_out must be a contiguous {rew.dtype} tensor of "
                                 f"{rew.numel()} elements on {rew.device}")
            rew = rew_out
        _core.check(self._lib, self._lib.uuvsim_dev_step(
            self._handle, actions.data_ptr(), actions.numel(), t["obs"].data_ptr(),
            t["obs"].numel(), rew.data_ptr(), rew.numel(), t["done"].data_ptr(),
            t["done"].numel(), t["reason"].data_ptr(), t["reason"].numel(),
            self._stream(stream)))
        return t["obs"], rew, t["done"], t["reason"]

    def set_done_f32(self, buf) -> None:
        """Register (tensor) or clear (None) a float32 [num_envs] device buffer
        later device-face steps also write done into as 0.0 / 1.0
        (uuvsim_dev_set_done_f32).  The batch keeps a reference to the tensor
        while it is registered: the engine writes into its memory."""
        self._require_open()
        if buf is None:
            _core.check(self._lib, self._lib.uuvsim_dev_set_done_f32(self._handle, None, 0))
            self._registered.pop("done_f32", None)
            return
        import torch
        if buf.dtype != torch.float32 or not buf.is_cuda or not buf.is_contiguous():
            raise ValueError("done buffer must be a contiguous float32 CUDA tensor")
        _core.check(self._lib, self._lib.uuvsim_dev_set_done_f32(
            self._handle, buf.data_ptr(), buf.numel()))
        self._registered["done_f32"] = buf

    def set_final_obs(self, buf) -> None:
        """Register (tensor) or clear (None) a [num_envs, obs_dim] device buffer the
        step writes finished envs' TERMINAL observations into
        (uuvsim_dev_set_final_obs); referenced by the batch while registered."""
        self._require_open()
        if buf is None:
            _core.check(self._lib, self._lib.uuvsim_dev_set_final_obs(self._handle, None, 0))
            self._registered.pop("final_obs", None)
            return
        if (buf.dtype != self.dtype or not buf.is_cuda or not buf.is_contiguous() or
                buf.numel() != self.num_envs * self.obs_dim):
            raise ValueError(f"final_obs must be a contiguous {self.dtype} CUDA tensor of "
                             f"{self.num_envs * self.obs_dim} elements")
        _core.check(self._lib, self._lib.uuvsim_dev_set_final_obs(
            self._handle, buf.data_ptr(), buf.numel()))
        self._registered["final_obs"] = buf

    def set_pdl(self, on: bool = True) -> None:
        """Launch later device-face steps as programmatic dependents of the previous
        kernel on the stream (include/uuvsim.h uuvsim_dev_set_pdl); results unchanged."""
        self._require_open()
        _core.check(self._lib, self._lib.uuvsim_dev_set_pdl(self._handle, 1 if on else 0))

    def observe_tensors(self, stream=None):
        t = self._tensors()
        _core.check(self._lib, self._lib.uuvsim_dev_observe(
            self._handle, t["obs"].data_ptr(), t["obs"].numel(), self._stream(stream)))
        return t["obs"]

    def snapshot(self) -> bytes:
        """Exact checkpoint of the slab (states, counters, RNG counters, DR records)."""
        self._require_open()
        n = ctypes.c_uint64(0)
        _core.check(self._lib, self._lib.uuvsim_snapshot_size(self._handle, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        _core.check(self._lib, self._lib.uuvsim_snapshot(self._handle, buf, n.value))
        return buf.raw

    def restore(self, blob: bytes) -> None:
        """Load a snapshot taken from an engine of the same configuration; the
        next steps continue bit-for-bit.  Returns no observation (call
        ``observe_tensors`` or step)."""
        self._require_open()
        _core.check(self._lib, self._lib.uuvsim_restore(self._handle, blob, len(blob)))
        self.root_seed = int.from_bytes(blob[32:40], "little")   # SnapHeader.root_seed

    def pd_actions_tensor(self, gains, reference, out=None, stream=None):
        """PD-baseline throttles [M, action_dim] for the current states, one kernel
        (uuvsim_dev_pd_actions); ``gains`` from ``baseline.PDActor.engine_gains()``,
        ``reference`` a device tensor of 6 (engine precision)."""
        import ctypes
        import torch
        if out is None:
            out = torch.empty((self.num_envs, self.action_dim), dtype=self.dtype,
                              device=torch.device("cuda", self.device_index))
        _core.check(self._lib, self._lib.uuvsim_dev_pd_actions(
            self._handle, ctypes.byref(gains), reference.data_ptr(), out.data_ptr(), out.numel(),
            self._stream(stream)))
        return out

    def states_tensor(self, out=None, stream=None):
        """Raw states [M, 12] on the device (engine precision), e.g. for PD control."""
        import torch
        if out is None:
            out = torch.empty((self.num_envs, 12), dtype=self.dtype,
                              device=torch.device("cuda", self.device_index))
        _core.check(self._lib, self._lib.uuvsim_dev_states(self._handle, out.data_ptr(),
                                                           out.numel(), self._stream(stream)))
        return out

    def bench_actions_tensor(self, stream=None):
        """Fixed U[-1,1] bench actions (reference batch.py:168-176) generated on device."""
        import torch
        out = torch.empty((self.num_envs, self.action_dim), dtype=self.dtype,
                          device=torch.device("cuda", self.device_index))
        _core.check(self._lib, self._lib.uuvsim_dev_bench_actions(
            self._handle, out.data_ptr(), out.numel(), self._stream(stream)))
        return out

    def stats_tensor(self, clear: bool = False, stream=None):
        """Episode statistics reduced on device into an f64[8] tensor (NCCL-ready)."""
        t = self._tensors()
        _core.check(self._lib, self._lib.uuvsim_dev_stats(
            self._handle, t["stats"].data_ptr(), len(STAT_NAMES), int(clear), self._stream(stream)))
        return t["stats"]

    def capture_graph(self, actions, n_steps: int = 1):
        """Capture ``n_steps`` device steps on fixed buffers into a native CUDA graph."""
        self._check_actions(actions)
        t = self._tensors()
        import torch
        torch.cuda.synchronize(self.device_index)
        _core.check(self._lib, self._lib.uuvsim_dev_graph_capture(
            self._handle, actions.data_ptr(), t["obs"].data_ptr(), t["rew"].data_ptr(),
            t["done"].data_ptr(), t["reason"].data_ptr(), int(n_steps)))
        self._graph_actions = actions   # keep the captured buffer alive
        return t["obs"], t["rew"], t["done"], t["reason"]

    def replay_graph(self, stream=None):
        _core.check(self._lib, self._lib.uuvsim_dev_graph_launch(self._handle,
                                                                 self._stream(stream)))


def resolve_backend(backend: str | None = None) -> str:
    """explicit arg > UUVSIM_BACKEND > b200 (reference batch.py:140-153); no CPU fallback."""
    choice = backend or os.environ.get("UUVSIM_BACKEND") or ""
    if choice in ("", "auto", "b200", "native"):
        return "b200"
    if choice == "python":
        raise RuntimeError("this package is the B200 engine; the pure-Python backend lives in "
                           "the reference package (there is no CPU fallback here)")
    raise ValueError(f"unknown backend {choice!r}")


_FAST = {}


def _fast_step(lib):
    """hostcall.step_ex bound to this library's uuvsim_step_ex, or None (module
    not built, or a second library in the process: the ctypes path is used)."""
    addr = ctypes.cast(lib.uuvsim_step_ex, ctypes.c_void_p).value
    if addr not in _FAST:
        fn = None
        if not _FAST:   # the module holds one function pointer
            try:
                from . import _hostcall
                _hostcall.bind(addr)
                fn = _hostcall.step_ex
            except ImportError:
                fn = None
        _FAST[addr] = fn
    return _FAST[addr]


def _pool_refs(entry):
    """Reference counts of a pool block and of each array handed out from it:
    a returned array the caller keeps raises its own count, any slice / view of
    it raises the block's (numpy collapses view bases onto the block)."""
    arrs = entry[2][0]
    return (sys.getrefcount(entry[1]), sys.getrefcount(arrs[0]), sys.getrefcount(arrs[1]),
            sys.getrefcount(arrs[2]), sys.getrefcount(arrs[3]))


def batch_create(spec: TaskSpec, base, ranges: RandomizationRanges | None, num_envs: int,
                 root_seed: int, threads: int = 0, backend: str | None = None, *,
                 precision: str = "fp32", device: int | None = None, env_offset: int = 0,
                 vehicle_mix=None, stats: bool = True) -> B200EnvBatch:
    """Create M environments on the GPU (reference batch.py:156-165 signature)."""
    resolve_backend(backend)
    if num_envs < 1:
        raise ValueError("num_envs must be >= 1")
    if device is None:
        try:
            import torch
            device = torch.cuda.current_device() if torch.cuda.is_available() else None
        except Exception:
            device = None
    cfg = engine_config_dict(base, spec, num_envs, root_seed, threads, ranges,
                             precision=precision, device=device, env_offset=env_offset,
                             vehicle_mix=vehicle_mix, stats=stats)
    return B200EnvBatch(cfg, root_seed, threads=threads)


def bench_actions(batch) -> np.ndarray:
    """Fixed U[-1,1] action matrix (reference batch.py:168-176), host f64."""
    from ._rng import bench_actions as _ba
    return _ba(batch.root_seed, batch.num_envs, batch.action_dim,
               getattr(batch, "env_offset", 0))


def bench_throughput(batch, n_steps: int, threads: int | None = None) -> dict:
    """Step n_steps times under fixed random actions, timed (reference batch.py:179-197)."""
    if n_steps < 1:
        raise ValueError("n_steps must be >= 1")
    if threads is not None:
        batch.set_threads(threads)
    actions = bench_actions(batch)
    t0 = time.perf_counter()
    for _ in range(n_steps):
        batch.step(actions)
    wall = time.perf_counter() - t0
    return {"env_steps_per_sec": batch.num_envs * n_steps / wall, "wall_time_s": wall,
            "n_steps": n_steps, "num_envs": batch.num_envs, "threads": batch.threads,
            "backend": batch.backend}


__all__ = ["B200EnvBatch", "batch_create", "bench_actions", "bench_throughput",
           "resolve_backend", "STAT_NAMES", "ConfigError", "VehicleParams"]
