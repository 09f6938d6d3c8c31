"""Per-step device time vs n_substeps at a latency-bound size (how much of the
step is the sub-step chain).  L2 flushed between steps, as bench.py.

    python tools/substep_latency.py [num_envs]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2410_14117_b200 as uuv  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for k in (1, 2, 5, 10, 20):
        spec = uuv.TaskSpec(n_substeps=k, control_dt=0.005 * k)
        env = uuv.batch_create(spec, uuv.bluerov2_params(), None, n, 0, device=0)
        act = env.bench_actions_tensor()
        env.capture_graph(act, 1)
        for _ in range(20):
            env.replay_graph()
        res = {}
        for mode in ("flushed", "resident"):
            evs = []
            for _ in range(300):
                if mode == "flushed":
                    flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                env.replay_graph()
                b.record()
                evs.append((a, b))
            torch.cuda.synchronize()
            ts = sorted(x.elapsed_time(y) * 1e3 for x, y in evs)
            res[mode] = round(ts[len(ts) // 2], 2)
        print(json.dumps({"envs": n, "n_substeps": k, "median_us": res}), flush=True)
        env.close()


if __name__ == "__main__":
    main()
