"""Edge cases of the step the reference defines (tasks.py:201-230,
dynamics.py:246-306, thrusters.py:97-119): non-finite inputs, out-of-range and
infinite throttles, integration failure mid-step (last finite state kept,
reason 2), tiny and ragged batches.  GPU results are compared with the oracle
(bit-exact for done / reason / counters, tolerance for floats) or, where fp32
and fp64 fail at different sub-steps, with a self-consistent fp32 construction.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2410_14117_b200 as uuv
from oracle import oracle as orc
from tests import parity as P

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _cfg(n=512, kind="station_keeping", precision="fp32", **task):
    spec = uuv.TaskSpec(kind=kind, **task)
    return uuv.engine_config_dict(uuv.default_params(), spec, n, 9, 0, None,
                                  precision=precision, device=0)


def _pair(cfg):
    g = uuv.B200EnvBatch(cfg, cfg["seed"], pinned=False)
    o = orc.OracleBatch(cfg, threads=0)
    g.reset_all(cfg["seed"])
    o.reset_all(cfg["seed"])
    return g, o


def _fp32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_nonfinite_and_out_of_range_actions(precision):
    cfg = _cfg(precision=precision)
    g, o = _pair(cfg)
    n, a = g.num_envs, g.action_dim
    act = orc.bench_actions(9, n, a)
    act[::7, 0] = np.nan                    # NaN passes the clamp (ref: t > 1 / t < -1 false)
    act[1::7, 1] = np.inf                   # clamped to +1
    act[2::7, 2] = -np.inf                  # clamped to -1
    act[3::7, :] *= 50.0                    # far outside [-1, 1]
    act = _fp32(act) if precision == "fp32" else act
    for _ in range(3):
        go, gr, gd, grs = g.step_ex(act)
        oo, orw, od, ors = o.step(act, with_reason=True)
        assert np.array_equal(gd, od) and np.array_equal(grs, ors)
        np.testing.assert_allclose(gr, orw, rtol=P.REL_TOL, atol=P.ABS_TOL)
    # every NaN env failed on its first sub-step (reason 2) and was reset
    assert np.all(ors[::7] == 2)
    rc_g, pc_g = g.counters()
    rc_o, pc_o = o.counters()
    assert np.array_equal(rc_g, rc_o) and np.array_equal(pc_g, pc_o)
    sg, so = g.states(), o.states()
    # failed envs were re-drawn: reset states equal fp32 of the oracle's fp64 draw
    want = _fp32(so[::7]) if precision == "fp32" else so[::7]
    assert np.array_equal(sg[::7], want)
    g.close()
    o.close()


def test_nonfinite_state_fails_and_keeps_last_finite_state():
    cfg = _cfg(n=300)
    g, o = _pair(cfg)
    s = o.states()
    s[::5, 9] = np.nan                      # NaN roll rate
    s[1::5, 6] = np.inf                     # infinite surge velocity
    g.set_states(s)
    o.set_states(_fp32(s))
    act = _fp32(orc.bench_actions(9, g.num_envs, g.action_dim))
    go, gr, gd, grs = g.step_ex(act)
    oo, orw, od, ors = o.step(act, with_reason=True)
    assert np.array_equal(grs, ors) and np.all(grs[::5] == 2) and np.all(grs[1::5] == 2)
    # the reward of a failed env is taken at its last finite (= initial) state
    np.testing.assert_allclose(gr, orw, rtol=P.REL_TOL, atol=P.ABS_TOL)
    g.close()
    o.close()


def test_failure_mid_step_keeps_last_finite_substep():
    """fp32 overflow in sub-step k > 1: the reward and the terminal observation
    must be those of the state after k-1 sub-steps.  fp64 would overflow at a
    different sub-step, so the expectation is built from fp32 runs of the same
    engine with n_substeps = k-1 and k at the same sub_dt."""
    from paper_2410_14117_b200.torchrl_env import VecEnv

    def run(n_sub, states):
        cfg = _cfg(n=64, control_dt=0.005 * n_sub, n_substeps=n_sub)
        vec = VecEnv(uuv.B200EnvBatch(cfg, 9, pinned=False))
        vec.reset(9)
        vec.batch.set_states(states)
        act = torch.zeros((64, vec.action_dim), device=vec.device)
        out = vec.step(act)
        res = (out.reward.double().cpu().numpy(), out.reason.cpu().numpy(),
               out.next_obs.double().cpu().numpy())
        vec.close()
        return res

    assert np.float32(0.05 / 10) == np.float32(0.005 * 3 / 3)
    base = uuv.B200EnvBatch(_cfg(n=64), 9, pinned=False)
    s = base.states()
    base.close()
    s[:, 6] = np.linspace(2e17, 6e18, 64)   # surge: quadratic damping overflows within a few sub-steps
    r10, why10, obs10 = run(10, s)
    assert np.all(why10 == 2)
    first_fail = np.full(64, 99)
    prefix = {}
    for k in range(1, 10):
        rk, whyk, obsk = run(k, s)
        prefix[k] = (rk, obsk)
        first_fail[(whyk == 2) & (first_fail == 99)] = k
    first_fail[first_fail == 99] = 10
    assert np.any(first_fail > 1)
    for e in range(64):
        k = first_fail[e]
        if k == 1:                          # failed at once: the initial state is kept
            continue
        rk, obsk = prefix[k - 1]
        assert r10[e] == rk[e], (e, k)
        assert np.array_equal(obs10[e], obsk[e]), (e, k)


@pytest.mark.parametrize("n", [1, 31, 129, 257])
def test_tiny_and_ragged_batches(n):
    cfg = _cfg(n=n, kind="circle", episode_len=7)
    g, o = _pair(cfg)
    act = _fp32(orc.bench_actions(9, n, g.action_dim))
    for _ in range(15):                     # two truncations
        _, gr, gd, grs = g.step_ex(act)
        _, orw, od, ors = o.step(act, with_reason=True)
        assert np.array_equal(gd, od) and np.array_equal(grs, ors)
        np.testing.assert_allclose(gr, orw, rtol=1e-4, atol=1e-5)
    assert np.array_equal(g.step_counts(), o.step_counts())
    g.close()
    o.close()


def test_slab_beyond_device_memory_is_a_config_error():
    import ctypes
    import json
    cfg = _cfg(n=(1 << 31) - 4096, precision="fp64")   # ~257 GB of fp64 state: cannot fit
    lib = uuv._core.load()
    h = ctypes.c_uint64(0)
    code = lib.uuvsim_create(json.dumps(cfg).encode(), ctypes.byref(h))
    assert code == 1
    assert "MiB of device memory" in uuv._core.last_error(lib)


@pytest.mark.slow
def test_maximum_slab_high_indices_exact():
    """2^27 envs (~10 GB of state, +13 GB of host state rows): the last envs of the slab reset
    exactly like the oracle's envs at the same global index, and a step touches
    every env (64-bit row offsets everywhere)."""
    n = 1 << 27
    cfg = _cfg(n=n, kind="circle")
    g = uuv.B200EnvBatch(cfg, 9, pinned=False)
    tail = dict(cfg)
    tail["batch"] = dict(cfg["batch"], num_envs=64, env_offset=n - 64)
    o = orc.OracleBatch(tail, threads=0)
    o.reset_all(9)
    s = g.states_tensor()
    torch.cuda.synchronize()
    assert np.array_equal(s[-64:].double().cpu().numpy(), _fp32(o.states()))
    act = g.bench_actions_tensor()
    for _ in range(2):
        g.step_tensors(act)
    torch.cuda.synchronize()
    assert g.stats()["env_steps"] == 2 * n
    assert int(g.step_counts()[-1]) == 2
    o.close()
    g.close()


def test_host_staging_is_allocated_on_first_host_use():
    """The device face needs no host-ABI staging: an engine driven only through
    uuvsim_dev_* never allocates it; the first host-face call does."""
    import ctypes
    import json
    n = 4096
    cfg = _cfg(n=n)
    lib = uuv._core.load()
    h = ctypes.c_uint64(0)
    assert lib.uuvsim_create(json.dumps(cfg).encode(), ctypes.byref(h)) == 0

    def staging():
        buf = ctypes.create_string_buffer(1 << 16)
        assert lib.uuvsim_info(h, buf, len(buf)) > 0
        return json.loads(buf.value.decode())["abi_staging_bytes"]

    try:
        spec = (ctypes.c_uint64 * 4)()
        assert lib.uuvsim_spec(h, spec) == 0
        od, ad = int(spec[1]), int(spec[2])
        assert staging() == 0
        a = torch.zeros((n, ad), device="cuda")
        o = torch.empty((n, od), device="cuda")
        r = torch.empty(n, device="cuda")
        d = torch.empty(n, dtype=torch.uint8, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        assert lib.uuvsim_dev_step(h, a.data_ptr(), a.numel(), o.data_ptr(), o.numel(),
                                   r.data_ptr(), n, d.data_ptr(), n, None, 0, st) == 0
        torch.cuda.synchronize()
        assert staging() == 0
        s = np.empty((n, 12))
        assert lib.uuvsim_states(h, s.ctypes.data, s.size) == 0
        assert staging() == n * 96                 # state rows only
        act = np.zeros((n, ad))
        obs, rew = np.empty((n, od)), np.empty(n)
        done = np.empty(n, dtype=np.uint8)
        assert lib.uuvsim_step(h, act.ctypes.data, act.size, obs.ctypes.data, obs.size,
                               rew.ctypes.data, n, done.ctypes.data, n) == 0
        assert staging() > n * 96
        assert np.isfinite(obs).all()
    finally:
        lib.uuvsim_destroy(h)


@pytest.mark.gpu
@pytest.mark.timeout(3600)
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "initcheck", "synccheck"])
def test_compute_sanitizer_clean(tool):
    """compute-sanitizer over every kernel family (tools/sanitize_run.py): the step
    kernels incl. the concurrent fp64 band kernel and its in-kernel tail, the TMA
    ring, host-ABI zero-copy / staged steps, fp64 engine, tcgen05 policy kernel."""
    import shutil
    import subprocess
    import sys
    from pathlib import Path
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not Path(cs).is_file():
        pytest.skip("compute-sanitizer not found")
    root = Path(__file__).resolve().parent.parent
    extra = ["--racecheck-report", "all"] if tool == "racecheck" else []
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "9", *extra, sys.executable,
                        str(root / "tools" / "sanitize_run.py")],
                       capture_output=True, text=True, timeout=3500, cwd=root)
    out = r.stdout + r.stderr
    if "closed on this pool" in out:   # the GPU pool's wrapper refuses compute-sanitizer
        pytest.skip("compute-sanitizer is disabled on this GPU pool: " + out.strip()[:160])
    log = root / "gpurun_out" / f"sanitizer_{tool}.log"
    log.parent.mkdir(exist_ok=True)
    log.write_text(out)
    assert r.returncode == 0, out[-3000:]
    assert "sanitize workload done" in out
    assert "ERROR SUMMARY: 0 errors" in out, out[-2000:]


@pytest.mark.gpu
def test_rejected_episode_resample_is_runtime_error():
    """A per-episode DR redraw whose M_RB + M_A is not positive definite: the
    reference engine panics there (engine.rs:553-558), which its C ABI maps to
    code 4 (capi.rs:58-70); uuvsim_step returns code 4 too.  The env keeps its
    previous parameters and the device face counts the rejection in the stats.
    (A heave added mass of -0.85 m keeps the base vehicle PD; with seed 2 the
    create-time draw is PD and the first per-episode redraw is not -- found with
    the oracle's sample_params.)"""
    veh = uuv.default_params().to_dict()
    am = [list(r) for r in veh["added_mass"]]
    am[2][2] = -0.85 * veh["mass"]
    veh["added_mass"] = am
    ranges = uuv.RandomizationRanges(mass=(0.9, 1.1), added_mass=(0.5, 2.0), per_episode=True)
    spec = uuv.TaskSpec(kind="station_keeping", episode_len=1)
    cfg = uuv.engine_config_dict(veh, spec, 1, 2, 0, ranges, device=0)
    env = uuv.B200EnvBatch(cfg)
    before = env.dr_factors()
    act = np.zeros((1, env.action_dim))
    with pytest.raises(uuv.NativeError) as ei:
        env.step(act)
    assert ei.value.code == 4 and "not positive definite" in ei.value.message
    assert np.array_equal(env.dr_factors(), before)          # previous parameters kept
    env.close()
    dev = uuv.B200EnvBatch(cfg)
    import torch
    a = torch.zeros((1, dev.action_dim), device="cuda")
    dev.stats(clear=True)
    dev.step_tensors(a)
    torch.cuda.synchronize()
    assert dev.stats()["resample_rejected"] == 1
    dev.close()
