"""C3 ablation: per-step device time (L2 flushed) with features toggled.

    python tools/c3_ablation.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2410_14117_b200 as uuv  # noqa: E402


def timed(cfg, steps=300, read_flush=False):
    env = uuv.B200EnvBatch(cfg, 0, pinned=False)
    act = env.bench_actions_tensor()
    env.capture_graph(act, 1)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for _ in range(10):
        env.replay_graph()
    evs = []
    sink = torch.empty((), dtype=torch.float32, device="cuda")
    for _ in range(steps):
        if read_flush:   # evict with reads: the L2 ends clean instead of dirty
            torch.sum(flush, dim=0, out=sink)
        else:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        env.replay_graph()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    env.close()
    ts = sorted(x.elapsed_time(y) * 1e3 for x, y in evs)
    return round(ts[len(ts) // 2], 2)


def main():
    heavy = uuv.default_params()
    spec = uuv.TaskSpec(kind="lemniscate")
    cfg = uuv.engine_config_dict(heavy, spec, 65536, 0, 0, uuv.default_ranges(per_episode=True),
                                 device=0)
    c2 = uuv.engine_config_dict(uuv.bluerov2_params(), uuv.TaskSpec(), 4096, 0, 0, None, device=0)
    for rf in (False, True, False, True):
        print(json.dumps({"c3": True, "read_flush": rf, "median_us": timed(cfg, read_flush=rf)}),
              flush=True)
        print(json.dumps({"c2": True, "read_flush": rf, "median_us": timed(c2, read_flush=rf)}),
              flush=True)
    if len(sys.argv) > 1 and sys.argv[1] == "flush-only":
        return
    cases = [("lemniscate", True, True, 5), ("lemniscate", False, True, 5),
             ("lemniscate", True, False, 5), ("station_keeping", True, True, 5),
             ("lemniscate", True, True, 1)]
    for kind, dr, stats, la in cases + cases[::-1]:
        spec = uuv.TaskSpec(kind=kind, lookahead=la)
        ranges = uuv.default_ranges(per_episode=True) if dr else None
        cfg = uuv.engine_config_dict(heavy, spec, 65536, 0, 0, ranges, device=0, stats=stats)
        print(json.dumps({"kind": kind, "dr": dr, "stats": stats, "lookahead": la,
                          "median_us": timed(cfg)}), flush=True)


if __name__ == "__main__":
    main()
