"""Latency probe of the fp64 band replay: C2/C5 bench engines, graph replays,
device time per step with and without band64 (for ncu: -k regex:k_band64)."""
from __future__ import annotations

import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2410_14117_b200 as uuv  # noqa: E402


FLUSH = os.environ.get("BAND_PROBE_FLUSH", "0") == "1"
EAGER = os.environ.get("BAND_PROBE_EAGER", "0") == "1"   # stream launches instead of the graph
VARIANTS = os.environ.get("BAND_PROBE_VARIANTS", "side,same,side-10,none-10,off").split(",")


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    n_sub = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
    table = {"side": (True, "side", None), "same": (True, "same", None),
             "side-10": (True, "side", -10.0), "none-10": (True, "none", -10.0),
             "bandfirst": (True, "side", None, "band_first"),
             "mainfirst": (True, "side", None, "main_first"),
             "per4096": (True, "side", None, None, 4096), "per2048": (True, "side", None, None, 2048),
             "per8192": (True, "side", None, None, 8192),
             "off": (False, "side", None)}
    for spec in (table[v] for v in VARIANTS):
        band, stream, margin = spec[:3]
        order = spec[3] if len(spec) > 3 else None
        per = spec[4] if len(spec) > 4 else None
        cfg, _ = bench.build_config(name, 0, "fp32", band64=band)
        cfg["device"]["band_stream"] = stream
        if order:
            cfg["device"]["band_order"] = order
        if per:
            cfg["device"]["band_per"] = per
        if margin is not None:
            cfg["device"]["band_margin"] = margin
            cfg["device"]["band_tail"] = False
        cfg["task"]["n_substeps"] = n_sub
        cfg["task"]["control_dt"] = 0.005 * n_sub
        env = uuv.B200EnvBatch(cfg)
        act = env.bench_actions_tensor()
        env.capture_graph(act, n_steps=1)
        run = (lambda: env.step_tensors(act)) if EAGER else env.replay_graph
        for _ in range(300):          # into the tumbling regime
            run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        env.stats(clear=True)
        if FLUSH:
            tot = 0.0
            for _ in range(steps):
                flush.zero_()
                a.record()
                run()
                b.record()
                torch.cuda.synchronize()
                tot += a.elapsed_time(b)
            a_ms = tot
        else:
            a.record()
            for _ in range(steps):
                run()
            b.record()
            torch.cuda.synchronize()
            a_ms = a.elapsed_time(b)
        st = env.stats()
        print(name, "eager" if EAGER else "graph", "n_sub", n_sub, "band64", band, stream, order or "", per or "", "margin", margin, "us/step %.2f" % (a_ms * 1e3 / steps),
              "band steps/step %.1f" % (st["band64_steps"] / steps), flush=True)
        env.close()


if __name__ == "__main__":
    main()
