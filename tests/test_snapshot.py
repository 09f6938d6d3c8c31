"""Exact slab checkpoint / resume (uuvsim_snapshot / uuvsim_restore).

The reference keeps its RNG counters private (engine.rs:338-339), so a run
cannot be resumed there; here a snapshot carries states, step counters, running
returns, RNG counters, DR records and the root seed, and a restored engine
continues bit-for-bit.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2410_14117_b200 as uuv
from paper_2410_14117_b200._core import NativeError

pytestmark = pytest.mark.gpu


def _cfg(seed, precision="fp32", episode_len=23, kind="lemniscate", n=3000):
    spec = uuv.TaskSpec(kind=kind, episode_len=episode_len)
    return uuv.engine_config_dict(uuv.default_params(), spec, n, seed, 0,
                                  uuv.default_ranges(per_episode=True), precision=precision,
                                  device=0)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_restore_continues_bit_for_bit(precision):
    a = uuv.B200EnvBatch(_cfg(4, precision), 4, pinned=False)
    act = uuv.bench_actions(a)
    for _ in range(30):                      # crosses resets + per-episode DR redraws
        a.step(act)
    blob = a.snapshot()
    want = [tuple(x.copy() for x in a.step_ex(act)) for _ in range(40)]
    want_states, want_ctr = a.states(), a.counters()
    b = uuv.B200EnvBatch(_cfg(99, precision), 99, pinned=False)   # other seed, other history
    b.step(uuv.bench_actions(b))
    b.restore(blob)
    assert b.root_seed == 4
    for w in want:
        got = b.step_ex(act)
        for x, y in zip(w, got):
            assert np.array_equal(x, y)
    assert np.array_equal(b.states(), want_states)
    for x, y in zip(b.counters(), want_ctr):
        assert np.array_equal(x, y)
    a.close()
    b.close()


def test_restore_rejects_other_configurations():
    a = uuv.B200EnvBatch(_cfg(4), 4, pinned=False)
    blob = a.snapshot()
    for other in (_cfg(4, episode_len=24), _cfg(4, n=3001), _cfg(4, precision="fp64"),
                  _cfg(4, kind="circle")):
        b = uuv.B200EnvBatch(other, 4, pinned=False)
        with pytest.raises(NativeError) as ei:
            b.restore(blob)
        assert ei.value.code == 1
        b.close()
    with pytest.raises(NativeError):
        a.restore(blob[:-1])
    with pytest.raises(NativeError):
        a.restore(b"XXXXXXXX" + blob[8:])
    a.restore(blob)                          # still fine after the failures
    a.close()
