"""Which feature carries the fixed per-step cost? (n_substeps=1, in-graph timing)"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2410_14117_b200 as uuv


def run(label, n, kind, vehicle, dr, per_episode, episode_len=600, nsub=1, la=5):
    spec = uuv.TaskSpec(kind=kind, episode_len=episode_len, n_substeps=nsub, control_dt=0.005 * nsub,
                        lookahead=la)
    veh = uuv.default_params() if vehicle == "heavy" else uuv.bluerov2_params()
    ranges = uuv.default_ranges(per_episode=per_episode) if dr else None
    env = uuv.batch_create(spec, veh, ranges, n, 0, device=0)
    act = env.bench_actions_tensor()
    env.capture_graph(act, 20)
    for _ in range(3):
        env.replay_graph()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(50):
        env.replay_graph()
    e1.record(st)
    torch.cuda.synchronize()
    s = env.stats()
    dones = s["done_truncation"] + s["done_divergence"] + s["done_failure"]
    print(f"{label:38s} {e0.elapsed_time(e1) * 1e3 / 1000:7.2f} us/step  dones/step={dones / 1070:.1f}  regs={env.info['step_kernel_registers']}")
    env.close()


n = 65536
if len(sys.argv) > 1 and sys.argv[1] == "la":
    for la in (1, 2, 3, 5, 8):
        run(f"lemniscate heavy no DR la={la}", n, "lemniscate", "heavy", False, False, 600, 1, la)
    run("station heavy no DR", n, "station_keeping", "heavy", False, False)
    sys.exit(0)
run("lemniscate heavy DR per-episode", n, "lemniscate", "heavy", True, True)
run("lemniscate heavy DR at create", n, "lemniscate", "heavy", True, False)
run("lemniscate heavy no DR", n, "lemniscate", "heavy", False, False)
run("station heavy no DR", n, "station_keeping", "heavy", False, False)
run("station heavy DR per-episode", n, "station_keeping", "heavy", True, True)
run("lemniscate heavy no DR, ep_len 10^6", n, "lemniscate", "heavy", False, False, 10**6)
run("lemniscate heavy no DR nsub10", n, "lemniscate", "heavy", False, False, 600, 10)
run("lemniscate heavy DR-ep nsub10", n, "lemniscate", "heavy", True, True, 600, 10)
