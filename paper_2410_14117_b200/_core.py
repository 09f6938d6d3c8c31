"""ctypes binding of libuuvsim_core.so (include/uuvsim.h).

The library is built in-tree by ``paper_2410_14117_b200.build`` and loaded
from ``paper_2410_14117_b200/_lib``.  There is no CPU fallback: if the
library is missing or its ABI version differs, ``load()`` raises.  Binding
mirrors the reference's ``_native._bind`` (reference
pkg/src/uuvsim/_native.py:49-78) for the ten ABI-v1 symbols, plus the B200
extensions.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

ABI_VERSION = 1
LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libuuvsim_core.so"

_ERR_NAMES = {0: "ok", 1: "invalid config", 2: "invalid handle", 3: "bad buffer size",
              4: "runtime error"}


class NativeError(RuntimeError):
    """Error code + message from the core (reference _native.py:32-35)."""

    def __init__(self, code: int, message: str):
        self.code = code
        self.message = message
        super().__init__(f"{_ERR_NAMES.get(code, 'error')} ({code}): {message}")


def _bind(lib: ctypes.CDLL) -> ctypes.CDLL:
    u64, i64, i32, u32 = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
    vp, cp = ctypes.c_void_p, ctypes.c_char_p
    sig = {
        "uuvsim_abi_version": (u32, []),
        "uuvsim_create": (i32, [cp, ctypes.POINTER(u64)]),
        "uuvsim_spec": (i32, [u64, ctypes.POINTER(u64)]),
        "uuvsim_reset": (i32, [u64, u64, vp, u64]),
        "uuvsim_step": (i32, [u64, vp, u64, vp, u64, vp, u64, vp, u64]),
        "uuvsim_states": (i32, [u64, vp, u64]),
        "uuvsim_step_counts": (i32, [u64, vp, u64]),
        "uuvsim_set_threads": (i32, [u64, u64]),
        "uuvsim_destroy": (i32, [u64]),
        "uuvsim_last_error": (i64, [cp, u64]),
        "uuvsim_step_ex": (i32, [u64, vp, u64, vp, u64, vp, u64, vp, u64, vp, u64]),
        "uuvsim_set_states": (i32, [u64, vp, u64]),
        "uuvsim_set_step_counts": (i32, [u64, vp, u64]),
        "uuvsim_counters": (i32, [u64, vp, vp, u64]),
        "uuvsim_dr_factors": (i32, [u64, vp, u64]),
        "uuvsim_wrench": (i32, [u64, vp, u64, vp, u64]),
        "uuvsim_stats": (i32, [u64, vp, u64, i32]),
        "uuvsim_info": (i64, [u64, cp, u64]),
        "uuvsim_dev_step": (i32, [u64, vp, u64, vp, u64, vp, u64, vp, u64, vp, u64, u64]),
        "uuvsim_dev_reset": (i32, [u64, u64, vp, u64, u64]),
        "uuvsim_dev_observe": (i32, [u64, vp, u64, u64]),
        "uuvsim_dev_bench_actions": (i32, [u64, vp, u64, u64]),
        "uuvsim_dev_stats": (i32, [u64, vp, u64, i32, u64]),
        "uuvsim_dev_states": (i32, [u64, vp, u64, u64]),
        "uuvsim_dev_set_final_obs": (i32, [u64, vp, u64]),
        "uuvsim_dev_set_pdl": (i32, [u64, i32]),
        "uuvsim_dev_set_done_f32": (i32, [u64, vp, u64]),
        "uuvsim_dev_pd_actions": (i32, [u64, vp, vp, vp, u64, u64]),
        "uuvsim_snapshot_size": (i32, [u64, ctypes.POINTER(u64)]),
        "uuvsim_snapshot": (i32, [u64, vp, u64]),
        "uuvsim_restore": (i32, [u64, vp, u64]),
        "uuvsim_dev_graph_capture": (i32, [u64, vp, vp, vp, vp, vp, u32]),
        "uuvsim_dev_graph_launch": (i32, [u64, u64]),
        "uuvsim_synchronize": (i32, [u64]),
        "uuvsim_rl_policy_blocks": (u32, [u64]),
        "uuvsim_rl_policy_act": (i32, [vp, u64]),
        "uuvsim_rl_post": (i32, [vp, u64]),
        "uuvsim_rl_image_bytes": (u64, [u32]),
        "uuvsim_rl_prepare": (i32, [vp, vp, u64, u64]),
        "uuvsim_rl_gae": (i32, [vp, vp, vp, vp, u32, u64, ctypes.c_float, ctypes.c_float,
                                vp, vp, u64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)   # AttributeError on a missing export, like the reference
        fn.restype = res
        fn.argtypes = args
    return lib


SYMBOLS = ("uuvsim_abi_version", "uuvsim_create", "uuvsim_spec", "uuvsim_reset", "uuvsim_step",
           "uuvsim_states", "uuvsim_step_counts", "uuvsim_set_threads", "uuvsim_destroy",
           "uuvsim_last_error")

_lib = None


def lib_path() -> Path:
    return Path(os.environ.get("UUVSIM_B200_LIB", str(LIB_PATH)))


def load() -> ctypes.CDLL:
    """Load and bind the in-tree core; raise loudly when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not path.is_file():
        raise RuntimeError(
            f"B200 core library not found at {path}; build it with "
            "`python -m paper_2410_14117_b200.build` (there is no CPU fallback)")
    lib = _bind(ctypes.CDLL(str(path)))
    v = lib.uuvsim_abi_version()
    if v != ABI_VERSION:
        raise RuntimeError(f"{path}: ABI version {v}, expected {ABI_VERSION}")
    _lib = lib
    return lib


def last_error(lib) -> str:
    buf = ctypes.create_string_buffer(4096)
    n = lib.uuvsim_last_error(buf, 4096)
    return buf.raw[: max(0, min(n, 4096))].decode("utf-8", "replace")


def check(lib, code: int) -> None:
    if code != 0:
        raise NativeError(code, last_error(lib))
