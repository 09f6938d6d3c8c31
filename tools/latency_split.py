"""Split C2 step time into fixed (memory/launch/cold) and per-sub-step parts by
varying n_substeps (control_dt scaled to keep dt)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2410_14117_b200 as uuv
from bench import build_config
from tools.latency_probe import timed

flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
for nsub in (1, 2, 5, 10, 20):
    cfg, _ = build_config(name, 0, "fp32")
    cfg["task"]["n_substeps"] = nsub
    cfg["task"]["control_dt"] = 0.005 * nsub
    env = uuv.B200EnvBatch(cfg)
    act = env.bench_actions_tensor()
    env.capture_graph(act, n_steps=1)
    for _ in range(10):
        env.replay_graph()
    torch.cuda.synchronize()
    w = timed(env, None)
    f = timed(env, flush)
    env.capture_graph(act, n_steps=20)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(50):
        env.replay_graph()
    e1.record(st)
    torch.cuda.synchronize()
    print(f"{name} n_sub={nsub:3d}: warm {w[1]:.2f} us, flushed {f[1]:.2f} us, in-graph {e0.elapsed_time(e1) * 1e3 / 1000:.2f} us/step")
    env.close()
