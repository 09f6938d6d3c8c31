"""Random sequences of API calls on two engines that must stay bit-identical:
host-ABI steps (zero-copy vs DMA transport, pooled outputs), device-face steps,
native graph replays, resets with new seeds, teacher-forced state / step-count
writes, snapshot + restore round trips and observations.  Catches stale cached
state (ABI graphs, pools, captured graphs) across every kind of call."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2410_14117_b200 as uuv

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _cfg(host_io):
    spec = uuv.TaskSpec(kind="helix", episode_len=17, lookahead=3)
    cfg = uuv.engine_config_dict([uuv.default_params(), uuv.bluerov2_params()], spec, 1500, 21,
                                 0, uuv.default_ranges(per_episode=True), device=0,
                                 vehicle_mix=[700, 1500])
    cfg["device"]["host_io"] = host_io
    return cfg


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_api_sequences_agree(seed):
    rng = np.random.default_rng(seed)
    a = uuv.B200EnvBatch(_cfg("mapped"), 21)
    b = uuv.B200EnvBatch(_cfg("copy"), 21, pinned=False)
    n, A = a.num_envs, a.action_dim
    act_h = rng.uniform(-1, 1, (n, A))
    act_d = torch.tensor(act_h, dtype=torch.float32, device="cuda")
    act_h32 = act_d.double().cpu().numpy()
    a.capture_graph(act_d, 2)
    b.capture_graph(act_d, 2)
    snap = None
    for _ in range(60):
        op = rng.integers(0, 8)
        if op <= 1:
            x, y = a.step_ex(act_h32), b.step_ex(act_h32)
            for u, v in zip(x, y):
                assert np.array_equal(u, v)
        elif op == 2:
            x, y = a.step_tensors(act_d), b.step_tensors(act_d)
            torch.cuda.synchronize()
            for u, v in zip(x, y):
                assert torch.equal(u, v)
        elif op == 3:
            a.replay_graph()
            b.replay_graph()
            torch.cuda.synchronize()
        elif op == 4:
            s = int(rng.integers(0, 1000))
            assert np.array_equal(a.reset_all(s), b.reset_all(s))
        elif op == 5:
            st = a.states()
            idx = rng.choice(n, 50, replace=False)
            st[idx, 6:12] = rng.normal(0, 0.5, (50, 6))
            a.set_states(st)
            b.set_states(st)
            sc = rng.integers(0, 17, n)
            a.set_step_counts(sc)
            b.set_step_counts(sc)
        elif op == 6:
            if snap is None:
                snap = (a.snapshot(), b.snapshot())
            else:
                a.restore(snap[0])
                b.restore(snap[1])
                snap = None
        else:
            x, y = a.observe_tensors(), b.observe_tensors()
            torch.cuda.synchronize()
            assert torch.equal(x, y)
        assert np.array_equal(a.states(), b.states())
        assert np.array_equal(a.step_counts(), b.step_counts())
    ca, cb = a.counters(), b.counters()
    assert np.array_equal(ca[0], cb[0]) and np.array_equal(ca[1], cb[1])
    a.close()
    b.close()


@pytest.mark.parametrize("seed", [3, 4])
def test_random_api_sequences_track_the_oracle(seed):
    """The same kind of sequence mirrored on the C oracle (no snapshots: the oracle
    cannot set RNG counters): done masks, reasons, step counters and RNG counters
    stay bit-exact; states stay within the rollout drift bound."""
    from oracle import oracle as orc
    from tests import parity as P
    rng = np.random.default_rng(seed)
    cfg = _cfg("auto")
    a = uuv.B200EnvBatch(cfg, 21)
    o = orc.OracleBatch(cfg, threads=0)
    o.reset_all(21)
    n, A = a.num_envs, a.action_dim
    act_d = torch.tensor(0.3 * rng.uniform(-1, 1, (n, A)), dtype=torch.float32, device="cuda")
    act_h32 = act_d.double().cpu().numpy()
    for _ in range(40):
        op = rng.integers(0, 5)
        if op <= 1:
            _, gr, gd, gq = a.step_ex(act_h32)
            _, orw, od, oq = o.step(act_h32, with_reason=True)
            assert np.array_equal(gd, od) and np.array_equal(gq, oq)
        elif op == 2:
            _, _, gd, gq = a.step_tensors(act_d)
            torch.cuda.synchronize()
            _, _, od, oq = o.step(act_h32, with_reason=True)
            assert np.array_equal(gd.cpu().numpy().astype(bool), od)
        elif op == 3:
            s = int(rng.integers(0, 1000))
            a.reset_all(s)
            o.reset_all(s)
        else:   # teacher-force: both continue from the oracle's state
            st = o.states()
            a.set_states(st)
            o.set_states(np.asarray(st, np.float32).astype(np.float64))
        assert np.array_equal(a.step_counts(), o.step_counts())
    ca, co = a.counters(), o.counters()
    assert np.array_equal(ca[0], co[0]) and np.array_equal(ca[1], co[1])
    band = np.abs(o.states()[:, 4]) > P.PITCH_BAND
    err = P.abs_err(a.states(), o.states(), P.STATE_ANGLES)[~band]
    assert err.max() < 2e-4
    a.close()
    o.close()
