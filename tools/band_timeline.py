"""Per-block %globaltimer timeline of one flushed graph replay (step kernel and
concurrent band kernel), from a UUV_BAND_CLOCK build:

    python -m paper_2410_14117_b200.build -D UUV_BAND_CLOCK --out _variants/clk/libuuvsim_core.so
    UUVSIM_B200_LIB=$PWD/_variants/clk/libuuvsim_core.so python tools/band_timeline.py c2 8 side,none,off

Prints, per replay, [min, median, max] over blocks of each event relative to the
step kernel's first block start (ns): when the blocks start, when the band
kernel's scan is done, when the last block of each kernel ends.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
NAMES = ("step_start", "step_end", "band_start", "band_scan", "band_end", "step_loaded", "step_subs",
         "band_loaded", "band_replayed", "band_gen", "loop_cycles", "loop_n")


def child(name, reps, stream):
    import ctypes

    import numpy as np
    import torch
    sys.path.insert(0, str(ROOT))
    import bench
    import paper_2410_14117_b200 as uuv
    from paper_2410_14117_b200 import _core
    lib = _core.load()
    tl = np.zeros((len(NAMES), 8192), dtype=np.uint64)
    ptr = tl.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong))
    flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
    cfg, _ = bench.build_config(name, 0, "fp32", band64=stream != "off")
    if stream != "off":
        cfg["device"]["band_stream"] = stream
    if os.environ.get("BAND_MARGIN"):   # e.g. 10: every env a band candidate
        cfg["device"]["band_margin"] = float(os.environ["BAND_MARGIN"])
    env = uuv.B200EnvBatch(cfg)
    act = env.bench_actions_tensor()
    env.capture_graph(act, n_steps=1)
    for _ in range(300):
        env.replay_graph()
    torch.cuda.synchronize()
    acc = {k: [] for k in NAMES[1:]}
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev = []
    for r in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        lib.uuvsim_debug_timeline(ptr)
        a.record()
        env.replay_graph()
        b.record()
        torch.cuda.synchronize()
        ev.append(a.elapsed_time(b) * 1e6)
        assert lib.uuvsim_debug_timeline(ptr) > 0
        t0 = tl[0][tl[0] > 0].astype(np.int64).min()
        for i in (NAMES.index("loop_cycles"), NAMES.index("loop_n")):
            tl[i][tl[i] > 0] += np.uint64(t0)
        row = []
        for i, nm in enumerate(NAMES):
            v = tl[i][tl[i] > 0].astype(np.int64) - t0
            if len(v):
                row.append(f"{nm} [{v.min():6d},{np.median(v):7.0f},{v.max():6d}] n={len(v)}")
                if nm != "step_start":
                    acc[nm].append(v.min() if nm == "band_start" else np.median(v) if nm in ("step_loaded", "step_subs") else v.max())
        print(f"rep {r}: event {ev[-1]:7.0f}  " + "  ".join(row), flush=True)
    print(f"median ns: event={np.median(ev):.0f}  " +
          "  ".join(f"{k}={np.median(v):.0f}" for k, v in acc.items() if v))
    env.close()


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]), sys.argv[4])
        return
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    for stream in (sys.argv[3] if len(sys.argv) > 3 else "side,none").split(","):
        res = subprocess.run([sys.executable, __file__, "--child", name, str(reps), stream],
                             capture_output=True, text=True, env=os.environ.copy())
        print(f"== {name} band_stream={stream} rc={res.returncode}", flush=True)
        if res.returncode:
            print(res.stderr[-2000:])
        print(res.stdout, flush=True)


if __name__ == "__main__":
    main()
