"""C2 latency probe: kernel-only vs per-launch step time, graph of 1 vs K steps."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2410_14117_b200 as uuv
from bench import build_config

for cfgname in sys.argv[1:] or ["c2"]:
    cfg, _ = build_config(cfgname, 0, "fp32")
    env = uuv.B200EnvBatch(cfg)
    act = env.bench_actions_tensor()
    st = torch.cuda.current_stream()
    for k in (1, 10, 100):
        env.capture_graph(act, n_steps=k)
        for _ in range(5):
            env.replay_graph()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(1, 2000 // k)
        e0.record(st)
        for _ in range(reps):
            env.replay_graph()
        e1.record(st)
        torch.cuda.synchronize()
        print(f"{cfgname} graph_steps={k:4d}: {e0.elapsed_time(e1) / (reps * k) * 1e3:.3f} us/step")
    # eager (no graph): launch overhead
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(1000):
        env.step_tensors(act)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"{cfgname} eager: {e0.elapsed_time(e1):.3f} us/step")
