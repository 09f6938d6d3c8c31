"""Per-step time of the same C3 engine re-created several times (allocation /
placement sensitivity), plus the arena address of each instance.

    python tools/alloc_variance.py [n]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2410_14117_b200 as uuv  # noqa: E402
from tools.c3_ablation import timed  # noqa: E402


def timed_info(cfg, steps=300):
    env = uuv.B200EnvBatch(cfg, 0, pinned=False)
    base = int(env.info["arena_address"])
    act = env.bench_actions_tensor()
    env.capture_graph(act, 1)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for _ in range(10):
        env.replay_graph()
    evs = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        env.replay_graph()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    ts = sorted(x.elapsed_time(y) * 1e3 for x, y in evs)
    out = (round(ts[len(ts) // 2], 2), base, act.data_ptr())
    env.close()
    return out


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    spec = uuv.TaskSpec(kind="lemniscate")
    cfg = uuv.engine_config_dict(uuv.default_params(), spec, 65536, 0, 0,
                                 uuv.default_ranges(per_episode=True), device=0)
    keep = []
    for i in range(n):
        t, base, ap = timed_info(cfg)
        print(json.dumps({"run": i, "median_us": t, "arena_mod_2M": base % (2 << 20),
                          "arena_hex": hex(base), "act_hex": hex(ap)}), flush=True)
        keep.append(torch.empty(int(3 << 20) * (i + 1), dtype=torch.uint8, device="cuda"))  # shift allocations


if __name__ == "__main__":
    main()
