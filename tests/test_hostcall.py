"""The CPython fast path of the host-ABI step (csrc/hostcall.c), without a GPU:
bound to a ctypes callback standing in for uuvsim_step_ex, it must pass the
handle, the action buffer and the output pointers through unchanged, return the
callee's code, and decline (-100) anything that is not a C-contiguous float64
[n_env, act_dim] array so B200EnvBatch.step falls back to the general path."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from paper_2410_14117_b200 import batch as B
from paper_2410_14117_b200 import build


@pytest.fixture()
def hostcall():
    if build.build_hostcall() is None:
        pytest.skip("Python headers not available")
    from paper_2410_14117_b200 import _hostcall
    yield _hostcall
    for addr, fn in B._FAST.items():   # restore the real binding for later tests
        if fn is not None:
            _hostcall.bind(addr)


def test_fast_step_passes_arguments_through(hostcall):
    u64, vp = ctypes.c_uint64, ctypes.c_void_p
    seen = []
    proto = ctypes.CFUNCTYPE(ctypes.c_int32, u64, vp, u64, vp, u64, vp, u64, vp, u64, vp, u64)

    def fake(*args):
        seen.append(args)
        return 3 if args[0] == 99 else 0

    cb = proto(fake)
    hostcall.bind(ctypes.cast(cb, vp).value)
    act = np.arange(12, dtype=np.float64).reshape(4, 3)
    ptrs = (1000, 48, 2000, 4, 3000, 4, 4000, 4)
    assert hostcall.step_ex(7, act, 4, 3, ptrs) == 0
    h, ap, alen, o, olen, r, rlen, d, dlen, rs, rslen = seen[-1]
    assert (h, ap, alen) == (7, act.ctypes.data, 12)
    assert (o, olen, r, rlen, d, dlen, rs, rslen) == ptrs
    assert hostcall.step_ex(99, act, 4, 3, ptrs) == 3          # the callee's code
    n = len(seen)
    for bad in (act.astype(np.float32), act.T, act.reshape(12), act[:2], act.tolist(),
                np.asfortranarray(np.ones((4, 3)))[:, :]):
        if isinstance(bad, np.ndarray) and bad.flags.c_contiguous and bad.shape == (4, 3) \
                and bad.dtype == np.float64:
            continue
        assert hostcall.step_ex(7, bad, 4, 3, ptrs) == -100    # general path instead
    assert len(seen) == n                                       # callee never reached
    with pytest.raises(TypeError):
        hostcall.step_ex(7, act, 4, 3, (1, 2))
