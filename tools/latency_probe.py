"""C2-style latency probe: per-step time (graph of 1 step) warm vs L2-flushed,
with episode statistics on/off; also graph-of-K amortisation."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2410_14117_b200 as uuv
from bench import build_config


def timed(env, flush, reps=400):
    st = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for i in range(reps):
        if flush is not None:
            flush.zero_()
        ev[i][0].record(st)
        env.replay_graph()
        ev[i][1].record(st)
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return sum(ts) / len(ts), ts[len(ts) // 2]


def main():
  flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
  for cfgname in sys.argv[1:] or ["c2"]:
    for stats in (True, False):
        cfg, _ = build_config(cfgname, 0, "fp32")
        cfg["device"]["stats"] = stats
        env = uuv.B200EnvBatch(cfg)
        act = env.bench_actions_tensor()
        env.capture_graph(act, n_steps=1)
        for _ in range(10):
            env.replay_graph()
        torch.cuda.synchronize()
        w = timed(env, None)
        f = timed(env, flush)
        print(f"{cfgname} stats={stats}: warm mean {w[0]:.2f} med {w[1]:.2f} us | "
              f"flushed mean {f[0]:.2f} med {f[1]:.2f} us  regs={env.info['step_kernel_registers']}")
        env.close()


if __name__ == "__main__":
    main()
