"""Host-ABI step transports (``device.host_io``): DMA copies through a captured
graph vs zero-copy mapped page-locked buffers.  Both must give bit-identical
results, with pageable or page-locked caller buffers, and the Python API must
hand back fresh arrays every step (reference _native.py:159-172 returns copies).
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

import paper_2410_14117_b200 as uuv

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

CASES = {
    "station_heavy": dict(kind="station_keeping", dr=False, n=4096, L=37),
    "lemniscate_dr": dict(kind="lemniscate", dr=True, n=3000, L=29),
    "circle_big": dict(kind="circle", dr=False, n=140000, L=23),   # pair kernel, staged rows
    # zero-copy with the action rows staged through shared memory (>= 512 KiB of
    # actions): paired station kernel, and the DR tracking kernel with a ragged
    # last block and staged observation rows in front of the action rows
    "station_16k": dict(kind="station_keeping", dr=False, n=16384, L=31),
    "lemniscate_dr_10k": dict(kind="lemniscate", dr=True, n=10000, L=27),
}


def _cfg(case, host_io):
    c = CASES[case]
    spec = uuv.TaskSpec(kind=c["kind"], episode_len=c["L"])
    ranges = uuv.default_ranges(per_episode=True) if c["dr"] else None
    cfg = uuv.engine_config_dict(uuv.default_params(), spec, c["n"], 5, 0, ranges, device=0)
    cfg["device"]["host_io"] = host_io
    return cfg


def _run(cfg, steps, pinned):
    env = uuv.B200EnvBatch(cfg, 5, pinned=pinned)
    act = uuv.bench_actions(env)
    if pinned:
        t = torch.empty(act.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[:] = act
        act = t.numpy()
    out = []
    for _ in range(steps):
        o, r, d, rs = env.step_ex(act)
        out.append((o.copy(), r.copy(), d.copy(), rs.copy()))
    st = env.states()
    env.close()
    return out, st


@pytest.mark.parametrize("case", list(CASES))
def test_copy_and_mapped_are_bit_identical(case):
    steps = 2 * CASES[case]["L"] + 3          # crosses two episode boundaries
    ref, st_ref = _run(_cfg(case, "copy"), steps, pinned=False)
    for mode, pinned in (("copy", True), ("mapped", True), ("auto", True), ("mapped", False)):
        got, st = _run(_cfg(case, mode), steps, pinned)
        for a, b in zip(ref, got):
            for x, y in zip(a, b):
                assert np.array_equal(x, y), (mode, pinned)
        assert np.array_equal(st_ref, st)


def test_api_returns_fresh_arrays():
    env = uuv.B200EnvBatch(_cfg("station_heavy", "auto"), 5)
    act = uuv.bench_actions(env)
    o1, r1, d1 = env.step(act)
    keep = (o1.copy(), r1.copy(), d1.copy())
    o2, r2, d2 = env.step(act)
    assert not np.shares_memory(o1, o2) and not np.shares_memory(r1, r2)
    for x, y in zip(keep, (o1, r1, d1)):
        assert np.array_equal(x, y)            # the first step's arrays were not overwritten
    assert d2.dtype == np.bool_ and o2.dtype == np.float64 and o2.shape == (4096, 12)
    env.close()


def test_api_pool_never_overwrites_held_outputs():
    env = uuv.B200EnvBatch(_cfg("station_heavy", "auto"), 5)
    ref = uuv.B200EnvBatch(_cfg("station_heavy", "copy"), 5, pinned=False)
    act = uuv.bench_actions(env)
    held = []
    for i in range(12):
        out = env.step_ex(act)
        want = ref.step_ex(act)
        if i % 4 == 0:
            held.append((out, [w.copy() for w in want]))        # the whole tuple
        elif i % 4 == 1:
            held.append((out[0][5:9], want[0][5:9].copy()))     # a sub-view only
        elif i % 4 == 2:
            held.append((out[1], want[1].copy()))               # one array
    for got, want in held:
        if isinstance(got, tuple):
            for g, w in zip(got, want):
                assert np.array_equal(g, w)
        else:
            assert np.array_equal(got, want)
    assert len(env._pool) <= env._POOL_MAX
    env.close()
    ref.close()


def test_raw_abi_with_alternating_pinned_buffers():
    """The captured-graph cache is keyed by pointer + allocation id."""
    cfg = _cfg("station_heavy", "copy")
    env = uuv.B200EnvBatch(cfg, 5)
    ref = uuv.B200EnvBatch(cfg, 5, pinned=False)
    act = uuv.bench_actions(env)
    lib, h = env._lib, env._handle
    n, d = env.num_envs, env.obs_dim
    for i in range(12):
        bufs = [torch.empty((n, d), dtype=torch.float64, pin_memory=True),
                torch.empty(n, dtype=torch.float64, pin_memory=True),
                torch.empty(n, dtype=torch.uint8, pin_memory=True)]
        if i % 3 == 2:
            bufs = [b.numpy().copy() for b in bufs]     # pageable every third step
        arrs = [b if isinstance(b, np.ndarray) else b.numpy() for b in bufs]
        P = [a.ctypes.data_as(ctypes.c_void_p) for a in arrs]
        assert lib.uuvsim_step(h, act.ctypes.data_as(ctypes.c_void_p), act.size, P[0], n * d,
                               P[1], n, P[2], n) == 0
        o, r, dn = ref.step(act)
        assert np.array_equal(arrs[0], o) and np.array_equal(arrs[1], r)
        assert np.array_equal(arrs[2].astype(bool), dn)
        del bufs, arrs
    env.close()
    ref.close()


def test_bench_throughput_and_bench_actions_match_reference_protocol():
    env = uuv.batch_create(uuv.TaskSpec(), uuv.bluerov2_params(), None, 1024, 7, device=0)
    host = uuv.bench_actions(env)                   # reference batch.py:168-176 (f64 host)
    dev = env.bench_actions_tensor().double().cpu().numpy()
    assert np.array_equal(dev, host.astype(np.float32).astype(np.float64))
    r = uuv.bench_throughput(env, 20, threads=4)    # reference batch.py:179-197
    assert set(r) == {"env_steps_per_sec", "wall_time_s", "n_steps", "num_envs", "threads",
                      "backend"}
    assert r["n_steps"] == 20 and r["num_envs"] == 1024 and r["threads"] == 4
    assert r["backend"] == "b200" and r["env_steps_per_sec"] > 0
    env.close()


def test_mapped_transport_with_misaligned_pinned_buffers():
    """A page-locked obs buffer that is only 8-byte aligned takes the DMA path
    (zero-copy writes use 16-byte vector stores) and gives the same results."""
    cfg = _cfg("lemniscate_dr", "mapped")
    a = uuv.B200EnvBatch(cfg, 5, pinned=False)
    b = uuv.B200EnvBatch(cfg, 5, pinned=False)
    act = uuv.bench_actions(a)
    n, d = a.num_envs, a.obs_dim
    blk = torch.empty(n * d * 8 + 64, dtype=torch.uint8, pin_memory=True).numpy()
    obs = blk[8:8 + n * d * 8].view(np.float64).reshape(n, d)       # base + 8 bytes
    rew = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    done = torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy()
    P = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    for _ in range(CASES["lemniscate_dr"]["L"] + 3):
        assert a._lib.uuvsim_step(a._handle, P(act), act.size, P(obs), obs.size, P(rew), n,
                                  P(done), n) == 0
        o, r, dn = b.step(act)
        assert np.array_equal(obs, o) and np.array_equal(rew, r)
        assert np.array_equal(done.astype(bool), dn)
    a.close()
    b.close()


def test_fast_binding_equals_ctypes_path():
    """B200EnvBatch.step through the CPython fast-call binding (csrc/hostcall.c)
    and through ctypes (binding disabled) give bit-identical streams; inputs the
    binding declines (float32, Fortran order, lists) take the general path."""
    cfg = _cfg("lemniscate_dr", "auto")
    a, b = uuv.B200EnvBatch(cfg, 5), uuv.B200EnvBatch(cfg, 5)
    assert a._fast is not None, "hostcall extension not built"
    b._fast = None
    act = uuv.bench_actions(a)
    variants = [act, act.astype(np.float32), np.asfortranarray(act), (0.5 * act).tolist()]
    for k in range(24):
        x = variants[k % len(variants)]
        oa, ra, da, sa = a.step_ex(x)
        ob, rb, db, sb = b.step_ex(x)
        assert np.array_equal(oa, ob) and np.array_equal(ra, rb)
        assert np.array_equal(da, db) and np.array_equal(sa, sb)
    with pytest.raises(ValueError):
        a.step(act[:10])
    a.close()
    b.close()
