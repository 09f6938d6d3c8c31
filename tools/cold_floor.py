"""Cold-start floor under the bench's L2-flush protocol: trivial kernels timed like a step."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()


def timed(fn, do_flush, reps=300):
    g = torch.cuda.CUDAGraph()
    fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for i in range(reps):
        if do_flush:
            flush.zero_()
        ev[i][0].record(st)
        g.replay()
        ev[i][1].record(st)
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return ts[len(ts) // 2]


small = torch.zeros(4096 * 12, device="cuda")
mid = torch.zeros(4096 * 64, device="cuda")
for name, fn in (("empty-ish (1 elem add)", lambda: small[:1].add_(1)),
                 ("48 KB add (state-size)", lambda: small.add_(1)),
                 ("1 MB add", lambda: mid.add_(1))):
    print(f"{name:28s} warm {timed(fn, False):6.2f} us   flushed {timed(fn, True):6.2f} us")


def timed_eager(fn, do_flush, reps=300):
    fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for i in range(reps):
        if do_flush:
            flush.zero_()
        ev[i][0].record(st)
        fn()
        ev[i][1].record(st)
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return ts[len(ts) // 2]


print("eager 48 KB add: warm %.2f flushed %.2f" % (timed_eager(lambda: small.add_(1), False),
                                                   timed_eager(lambda: small.add_(1), True)))
import paper_2410_14117_b200 as uuv
from bench import build_config
cfg, _ = build_config("c2", 0, "fp32")
env = uuv.B200EnvBatch(cfg)
act = env.bench_actions_tensor()
env.capture_graph(act, 1)
print("uuv c2 eager step: warm %.2f flushed %.2f" % (timed_eager(lambda: env.step_tensors(act), False),
                                                     timed_eager(lambda: env.step_tensors(act), True)))
print("uuv c2 native graph: warm %.2f flushed %.2f" % (timed_eager(env.replay_graph, False),
                                                       timed_eager(env.replay_graph, True)))
print("uuv c2 torch graph: warm %.2f flushed %.2f" % (timed(lambda: env.step_tensors(act), False),
                                                      timed(lambda: env.step_tensors(act), True)))
