"""RL-library adapter: terminated/truncated split and
terminal observations on the device face.

The terminal observation is checked against the oracle: the engine with
``episode_len = L`` truncates every surviving env at step L, and its terminal
row must equal the oracle's observation after L steps of an otherwise
identical batch whose episodes are longer (same resets, same actions).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2410_14117_b200 as uuv
from paper_2410_14117_b200 import torchrl_env as T
from oracle import oracle as orc
from tests import parity as P


def test_torchrl_adapter_is_import_gated():
    try:
        import torchrl  # noqa: F401
    except ImportError:
        with pytest.raises(ImportError, match="torchrl"):
            T.make_torchrl_env(None)


def test_reason_codes_match_reference_tasks():
    # tasks.py:41-42, 205: 0 truncation, 1 divergence, 2 integration failure
    assert (T.REASON_TRUNCATED, T.REASON_DIVERGED, T.REASON_FAILED) == (0, 1, 2)


def _cfg(kind, L, n, dr, precision="fp32"):
    spec = uuv.TaskSpec(kind=kind, episode_len=L)
    ranges = uuv.default_ranges(per_episode=True) if dr else None
    return uuv.engine_config_dict(uuv.default_params(), spec, n, 3, 0, ranges,
                                  precision=precision, device=0)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,dr", [("station_keeping", False), ("lemniscate", True)])
def test_terminal_obs_and_split(kind, dr):
    L, n = 40, 4096
    cfg = _cfg(kind, L, n, dr)
    vec = T.VecEnv(uuv.B200EnvBatch(cfg, 3))
    vec.reset(3)
    act = vec.batch.bench_actions_tensor() * 0.25   # power of 2: exact in fp32
    term_seen = torch.zeros(n, dtype=torch.bool, device=vec.device)
    for t in range(L):
        out = vec.step(act)
        assert torch.equal(out.done, out.terminated | out.truncated)
        assert not torch.any(out.terminated & out.truncated)
        keep = ~out.done
        assert torch.equal(out.next_obs[keep], out.obs[keep])
        if t < L - 1:
            assert not out.truncated.any()
        term_seen |= out.terminated
    assert out.truncated[~term_seen].all()        # every survivor truncates at step L
    gpu_terminal = out.next_obs.double().cpu().numpy()
    gpu_post = out.obs.double().cpu().numpy()
    alive = (~term_seen).cpu().numpy()
    vec.close()

    # oracle: same batch with longer episodes, observed after L steps
    cfg_long = _cfg(kind, L + 10, n, dr)
    ob = orc.OracleBatch(cfg_long, threads=0)
    ob.reset_all(3)
    a = orc.bench_actions(3, n, ob.action_dim).astype(np.float32).astype(np.float64) * 0.25
    done_any = np.zeros(n, dtype=bool)
    band = np.zeros(n, dtype=bool)       # envs that ever reach the pitch band (tests/parity.py)
    for _ in range(L):
        _o, _r, d = ob.step(a)
        done_any |= d
        band |= np.abs(ob.states()[:, 4]) > P.PITCH_BAND
    want = ob.observe()
    ob.close()
    sel = alive & ~done_any & ~band
    assert sel.mean() > 0.9
    # a 40-step rollout, not one step: the documented 100-step drift bound applies
    err = np.abs(gpu_terminal[sel] - want[sel])
    assert np.max(err) < 2e-4, np.max(err)
    # and the post-reset rows are genuine resets (differ from the terminal rows)
    assert np.all(np.any(gpu_post[sel] != gpu_terminal[sel], axis=1))


@pytest.mark.gpu
def test_final_obs_not_written_by_host_abi_step():
    cfg = _cfg("station_keeping", 5, 256, False)
    vec = T.VecEnv(uuv.B200EnvBatch(cfg, 3))
    vec.final_obs.fill_(7.0)
    b = vec.batch
    b.reset_all(3)
    act = uuv.bench_actions(b)
    for _ in range(5):
        b.step(act)
    torch.cuda.synchronize()
    assert torch.all(vec.final_obs == 7.0)
    vec.close()


def _fake_torchrl(monkeypatch):
    """Minimal stand-ins for tensordict / torchrl (not installed in this image) so the
    import-gated EnvBase subclass can be exercised."""
    import sys
    import types

    class TensorDict(dict):
        def __init__(self, d, batch_size=None, device=None):
            super().__init__(d)
            self.batch_size, self.device = batch_size, device

        def get(self, k, default=None):
            return dict.get(self, k, default)

    class EnvBase:
        def __init__(self, device=None, batch_size=None):
            self.device, self.batch_size = device, batch_size

    class Spec:
        def __init__(self, *a, **kw):
            self.args, self.kw = a, kw

    td = types.ModuleType("tensordict")
    td.TensorDict = TensorDict
    trl = types.ModuleType("torchrl")
    envs = types.ModuleType("torchrl.envs")
    envs.EnvBase = EnvBase
    data = types.ModuleType("torchrl.data")
    for name in ("Composite", "Unbounded", "Bounded", "Categorical"):
        setattr(data, name, type(name, (Spec,), {}))
    trl.envs, trl.data = envs, data
    for k, v in (("tensordict", td), ("torchrl", trl), ("torchrl.envs", envs),
                 ("torchrl.data", data)):
        monkeypatch.setitem(sys.modules, k, v)
    return TensorDict


@pytest.mark.gpu
def test_torchrl_env_protocol_with_stand_in_modules(monkeypatch):
    TensorDict = _fake_torchrl(monkeypatch)
    L, n = 6, 512
    vec = T.VecEnv(uuv.B200EnvBatch(_cfg("circle", L, n, False), 3))
    env = T.make_torchrl_env(vec, seed=3)
    assert tuple(env.batch_size) == (n,)
    td0 = env._reset(None)
    assert td0["observation"].shape == (n, vec.obs_dim) and not td0["done"].any()
    act = torch.zeros((n, vec.action_dim), device=vec.device)
    for t in range(L):
        td = env._step(TensorDict({"action": act}))
        assert td["reward"].shape == (n, 1) and td["done"].shape == (n, 1)
        assert torch.equal(td["done"], td["terminated"] | td["truncated"])
    assert td["truncated"].all()                       # every env hits episode_len
    # the terminal observation is reported; the collector's partial reset gets the
    # already reset observation from the engine
    post = env._reset(TensorDict({"_reset": td["done"].clone()}))["observation"]
    assert not torch.equal(post, td["observation"])
    assert torch.equal(post, vec.batch.observe_tensors())
    vec.close()
