#!/usr/bin/env python
"""Benchmark of the batched env step (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c5]
    python bench.py --impl reference ...       # the reference arm (CPU oracle port)

Workload (default ``c2`` = BASELINE.json configs[1]): BlueROV2 station-keeping,
4,096 envs per GPU, seed 0, fixed U[-1,1] bench actions (reference
batch.py:168-197), synthetic, one CUDA-graph-replayed fused step per timed
step.  Timing: W warm-up steps, then K steps, each bracketed by CUDA events on
the launching stream with an L2 flush (256 MiB write) between steps; barrier +
synchronize on both sides; max over ranks.  ``value`` = env-steps/s of the
whole job with inputs resident in HBM; ``e2e`` = the same metric through the
reference-facing C ABI (``uuvsim_step`` with pinned host f64 buffers, H2D of
actions and D2H of obs/reward/done inside the timed region).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONTROL_DT = 0.05
# Algorithmic flops per env-step of the reference path (counted on
# the reference's flat kernels for the 8-thruster Heavy; each thruster fewer
# removes its thrust curve (2) and allocation column (12) = 14 flop).
FLOPS_8THR = {"station_keeping": 4073, "circle": 4157, "helix": 4169, "lemniscate": 4181}
L2_FLUSH_BYTES = 256 << 20

CONFIGS = {
    "c2": dict(workload="C2 BlueROV2 station-keeping, 4096 envs/GPU", kind="station_keeping",
               vehicles=["bluerov2"], num_envs=4096, dr=None),
    "c3": dict(workload="C3 BlueROV2-Heavy lemniscate tracking + per-episode DR, 65536 envs/GPU",
               kind="lemniscate", vehicles=["bluerov2_heavy"], num_envs=65536, dr="episode"),
    # lemniscate is the headline, circle and helix are also reported
    "c3_circle": dict(workload="C3 BlueROV2-Heavy circle tracking + per-episode DR, 65536 envs/GPU",
                      kind="circle", vehicles=["bluerov2_heavy"], num_envs=65536, dr="episode"),
    "c3_helix": dict(workload="C3 BlueROV2-Heavy helix tracking + per-episode DR, 65536 envs/GPU",
                     kind="helix", vehicles=["bluerov2_heavy"], num_envs=65536, dr="episode"),
    "c4": dict(workload="C4 BlueROV2 circle tracking, 16384 envs/GPU", kind="circle",
               vehicles=["bluerov2"], num_envs=16384, dr=None),
    "c5": dict(workload="C5 mixed BlueROV2/Heavy station-keeping, 1048576 envs/GPU",
               kind="station_keeping", vehicles=["bluerov2_heavy", "bluerov2"],
               num_envs=1 << 20, dr=None),
}


def flops_per_env_step(kind: str, n_thr_list) -> float:
    n = float(np.mean(n_thr_list))
    return FLOPS_8THR[kind] - 14.0 * (8.0 - n)


def bytes_per_env_step(kind: str, n_act: int, obs_dim: int, dr: bool) -> int:
    """Minimum HBM bytes per env-step of the fp32 device path."""
    b = 48 * 2            # state read + write (12 fp32)
    b += 4 * n_act        # actions
    b += 4 * obs_dim      # observation
    b += 4 + 1 + 1        # reward, done, reason
    b += 4 * 2            # step counter read + write
    b += 4 * 2            # running episode return read + write
    if dr:
        b += 40           # randomised parameter record (10 fp32)
    if kind != "station_keeping":
        pass              # trajectory table is a few KB, L1/L2 resident
    return b


def build_config(name: str, rank: int, precision: str, pair: str = "auto",
                 stage_obs: str = "auto", band64: bool = True, strong: bool = False):
    """Engine config of workload ``name`` for this rank: weak scaling (default) =
    num_envs per rank at global offset rank * num_envs; strong = num_envs for
    the whole job split into rank slabs.  Mixed vehicles: a 50/50 global mix."""
    import paper_2410_14117_b200 as uuv
    c = CONFIGS[name]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if strong:
        total = c["num_envs"]
        off = total * rank // world
        n = total * (rank + 1) // world - off
    else:
        n = c["num_envs"]
        total, off = n * world, rank * n
    spec = uuv.TaskSpec(kind=c["kind"])
    ranges = uuv.default_ranges(per_episode=True) if c["dr"] == "episode" else None
    vdocs = [uuv.VehicleParams(uuv.vehicles.get_vehicle(v)) for v in c["vehicles"]]
    if len(vdocs) > 1:
        cfg = uuv.engine_config_dict(vdocs, spec, n, 0, 0, ranges, precision=precision,
                                     device=rank_device(), env_offset=off,
                                     vehicle_mix=[total // 2, total - total // 2])
    else:
        cfg = uuv.engine_config_dict(vdocs[0], spec, n, 0, 0, ranges, precision=precision,
                                     device=rank_device(), env_offset=off)
    cfg["device"]["pair"] = pair
    cfg["device"]["stage_obs"] = stage_obs
    cfg["device"]["band64"] = band64
    return cfg, [v.n_thrusters() for v in vdocs]


def c4_loop(env, horizon: int = 64, reps: int = 5) -> dict:
    """C4 rollout loop: normalise -> 2x64 tanh actor-critic -> Gaussian sample ->
    clamp -> fused env step -> rollout buffers, one CUDA graph per horizon
    (paper_2410_14117_b200.rollout).  Device time of `reps` graph replays."""
    import torch

    from paper_2410_14117_b200 import rollout as R
    cfg = R.TrainConfig(num_envs=env.num_envs, horizon=horizon)
    pol = R.ActorCritic(env.obs_dim, env.action_dim, seed=0).cuda()
    norm = R.RunningNorm(env.obs_dim, "cuda")
    ro = R.Rollout(env, pol, norm, cfg, use_graph=True)
    ro.reset(0)
    ro.collect()                       # warm-up + capture + first replay
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        ro.collect()
    b.record()
    torch.cuda.synchronize()
    s = a.elapsed_time(b) / 1e3
    return {"env_steps_per_sec": env.num_envs * horizon * reps / s,
            "us_per_env_step_batch": s / (horizon * reps) * 1e6, "horizon": horizon,
            "what": "policy (2x64 tanh actor-critic) + sampling + fused step + buffers, "
                    "one CUDA graph per horizon"}


def rank_device() -> int:
    """LOCAL_RANK's GPU (wrapped when there are fewer GPUs than ranks: the
    N>1 code path can run on one device for testing)."""
    r = int(os.environ.get("LOCAL_RANK", "0"))
    try:
        import torch
        n = torch.cuda.device_count()
        return r % n if n else r
    except Exception:
        return r


def workload_config(name: str, world: int, precision: str = "fp32") -> dict:
    """The ``config`` object of the JSON line (identical in both arms)."""
    c = CONFIGS[name]
    return {"workload": c["workload"], "num_envs_per_gpu": c["num_envs"],
            "num_envs_total": c["num_envs"] * world, "task": c["kind"],
            "vehicles": c["vehicles"], "randomization": c["dr"] or "none", "n_substeps": 10,
            "control_dt": CONTROL_DT, "parallelism": f"env-slab x{world}",
            "precision": precision}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def build_hash() -> str:
    """sha256[:16] of the loaded engine library (ties ncu-derived numbers to a build)."""
    import hashlib
    p = ROOT / "paper_2410_14117_b200" / "_lib" / "libuuvsim_core.so"
    try:
        return hashlib.sha256(p.read_bytes()).hexdigest()[:16]
    except OSError:
        return "missing"


NCU_METRICS = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
               "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,"
               "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,"
               "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,"
               "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,"
               "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,"
               "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum")


def ncu_probe(name: str) -> int:
    """Child process of ncu_measure: create workload ``name`` and step it eagerly."""
    import torch
    import paper_2410_14117_b200 as uuv
    torch.cuda.set_device(rank_device())
    cfg, _ = build_config(name, 0, "fp32")
    env = uuv.B200EnvBatch(cfg)
    act = env.bench_actions_tensor()
    for _ in range(310):          # into the tumbling regime (band kernel busy), then profiled
        env.step_tensors(act)
    torch.cuda.synchronize()
    return 0


def ncu_measure(name: str, timeout: float = 300.0):
    """One ncu pass over the CURRENT build: per-launch DRAM bytes and executed FP32
    (and FP64) flops of the step kernel and the band kernel for workload ``name``
    (ncu flushes caches before each launch: cold traffic).  None when ncu is
    unavailable.  The numbers are read, not timed: ncu's durations are serialised."""
    import csv
    import io
    import shutil
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not Path(ncu).is_file():
        return None
    cmd = [ncu, "--metrics", NCU_METRICS, "--csv", "-k", "regex:k_step|k_band",
           "--launch-skip", "600", "--launch-count", "4", sys.executable, str(ROOT / "bench.py"),
           "--ncu-probe", name]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    except Exception as e:   # noqa: BLE001
        return {"error": str(e)[:200]}
    rows = [ln for ln in r.stdout.splitlines() if ln.startswith('"')]
    if not rows:
        return {"error": (r.stdout + r.stderr)[-300:]}
    per = {}
    for rec in csv.DictReader(io.StringIO("\n".join(rows))):
        k = rec.get("Kernel Name", "")
        kind = "band" if "k_band" in k else "step"
        d = per.setdefault((rec.get("ID"), kind), {"kernel": k.split("(")[0]})
        try:
            d[rec["Metric Name"]] = float(rec["Metric Value"].replace(",", ""))
        except (KeyError, ValueError):
            pass
    out = {}
    for (_, kind), d in per.items():
        out.setdefault(kind, []).append(d)
    res = {}
    for kind, launches in out.items():
        m = {k: float(np.mean([x.get(k, 0.0) for x in launches])) for k in launches[0]
             if k != "kernel"}
        m["kernel"] = launches[0]["kernel"]
        m["launches"] = len(launches)
        res[kind] = m
    return res


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = Path(os.environ.get("TMPDIR", "/tmp")) / f"uuv_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=self.f, stderr=subprocess.DEVNULL)
            # the timed region starts only once the sampler is producing lines
            t0 = time.time()
            while time.time() - t0 < 5.0 and self.path.stat().st_size == 0:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.05)   # one more sample after the timed region
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None or not self.path.is_file():
            return None
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        try:
            self.path.unlink()
        except OSError:
            pass
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.is_file():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6551.7)), float(d.get("sm_max_mhz", 1965.0)), "measured"
    return 6650.0, 1965.0, "fallback"


# --------------------------------------------------------------------------- CPU arm
def cpu_oracle_run(cfg: dict, n_steps_cap: int, seconds: float, threads: int):
    """Time the oracle port (uuv_oracle.c) on host cores over a bounded sample."""
    from oracle import oracle as orc
    b = orc.OracleBatch(cfg, threads=threads)
    act = orc.bench_actions(cfg["seed"], b.num_envs, b.action_dim)
    b.step(act)   # warm
    t0 = time.perf_counter()
    steps = 0
    while steps < n_steps_cap and (time.perf_counter() - t0) < seconds:
        b.step(act)
        steps += 1
    wall = time.perf_counter() - t0
    b.close()
    return b.num_envs * steps / wall, steps, wall


def cpu_sample_config(cfg: dict, max_envs: int) -> dict:
    c = json.loads(json.dumps(cfg))
    c["batch"]["num_envs"] = min(int(c["batch"]["num_envs"]), max_envs)
    return c


def reference_python_c1(seconds_cap: float = 60.0):
    """The reference's OWN CPU path, timed as itself: uuvsim.bench_throughput on a
    PyEnvBatch at C1 (station keeping, Heavy defaults, 64 envs x 1,000 steps, seed
    0; reference batch.py:179-197), imported from baseline/_ref (the offline
    install shipped with the repo).  None when it is not installed."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "uuvsim" / "__init__.py").is_file():
        return None
    code = ("import sys, json; sys.path.insert(0, %r); import uuvsim;"
            "b = uuvsim.batch_create(uuvsim.TaskSpec(), uuvsim.default_params(), None, 64, 0,"
            " backend='python'); print(json.dumps(uuvsim.bench_throughput(b, 1000)))" % str(ref))
    try:
        env = dict(os.environ)
        env.pop("UUVSIM_CORE_LIB", None)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                           timeout=seconds_cap * 4, env=env)
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:   # noqa: BLE001
        return {"error": str(e)[:200]}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    cfg, n_thr = build_config(args.config, 0, "fp32")
    sample = cpu_sample_config(cfg, 16384)
    n = sample["batch"]["num_envs"]
    # warmup steps untimed, then K steps each a bounded slice of the workload
    from oracle import oracle as orc
    b = orc.OracleBatch(sample, threads=threads)
    act = orc.bench_actions(0, n, b.action_dim)
    for _ in range(args.warmup):
        b.step(act)
    # at least ~1 s of timed work (the per-step slice is ~1.6 ms at C2): a
    # K-step window alone would be dominated by timer noise
    t0 = time.perf_counter()
    k = 0
    budget = 120.0
    while (k < args.steps or time.perf_counter() - t0 < 1.0) and time.perf_counter() - t0 < budget:
        b.step(act)
        k += 1
    wall = time.perf_counter() - t0
    value = n * k / wall
    world = int(os.environ.get("WORLD_SIZE", "1"))
    line = {
        "impl": "reference", "metric": "env_steps_per_sec", "value": value,
        "unit": "env-steps/s", "n_gpus": args.gpus, "steps": k, "warmup": args.warmup,
        "ms_per_step": wall / k * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.config, world, "fp32"),
        "rtf": {"aggregate": value * CONTROL_DT},
        "cpu_baseline": {"value": value, "unit": "env-steps/s", "cores": threads,
                         "kind": "port", "cpu_model": cpu_model(),
                         "sample": f"{n} envs x {k} steps of {args.config} on the C oracle "
                                   f"(uuv_oracle.c: the reference's flat kernels restated in "
                                   f"fp64 C, bit-exact against its PyEnvBatch; OpenMP {threads} "
                                   f"threads); the Rust reference engine cannot be built here "
                                   f"(no cargo/rustc)"},
        "e2e": {"value": value, "unit": "env-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU arm
def timed_steps(env, flush, stream, k: int):
    """k graph-replayed steps, L2 flushed (256 MiB write) before each, CUDA events
    around each step on the launching stream; returns the summed seconds."""
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(k)]
    torch.cuda.synchronize()
    for i in range(k):
        flush.zero_()
        ev[i][0].record(stream)
        env.replay_graph()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / 1e3


def make_engine(name, rank, args, precision="fp32", strong=False):
    import paper_2410_14117_b200 as uuv
    cfg, n_thr = build_config(name, rank, precision, args.pair, args.stage_obs,
                              args.band64 == "on", strong=strong)
    env = uuv.B200EnvBatch(cfg)
    act = env.bench_actions_tensor()
    env.capture_graph(act, n_steps=1)
    return env, act, n_thr


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--pair", default="auto", choices=["auto", "on", "off"],
                    help="two envs per thread (default: auto by env count)")
    ap.add_argument("--stage-obs", default="auto", choices=["auto", "on", "off"],
                    help="observation rows through shared memory (default: tracking only)")
    ap.add_argument("--band64", default="on", choices=["on", "off"],
                    help="fp64 steps for envs whose pitch may leave |theta| <= 1.4 (default on)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend for N > 1 (gloo: test the path on one GPU)")
    ap.add_argument("--no-sweep", action="store_true", help="skip the secondary config sweep")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-ncu", action="store_true", help="skip the ncu traffic / flop pass")
    ap.add_argument("--ncu-probe", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.ncu_probe:
        return ncu_probe(args.ncu_probe)
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    import paper_2410_14117_b200 as uuv

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dev = rank_device()
    torch.cuda.set_device(dev)
    gloo = args.dist_backend == "gloo"
    if world > 1:
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))

    def barrier():
        if world > 1:
            dist.barrier()

    def reduce(x: float, op) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if gloo else "cuda")
        dist.all_reduce(t, op=op)
        return float(t.item())

    def max_over_ranks(x: float) -> float:
        return reduce(x, dist.ReduceOp.MAX) if world > 1 else x

    c = CONFIGS[args.config]
    env, act, n_thr = make_engine(args.config, rank, args, args.precision)
    n = env.num_envs
    stream = torch.cuda.current_stream()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        env.replay_graph()
    env.stats(clear=True)
    torch.cuda.synchronize()
    barrier()

    # ---- timed region: K steps, L2 flushed between steps, events per step
    with ClockSampler(dev) as clk:
        local_s = timed_steps(env, flush, stream, args.steps)
        # episode statistics: one all-reduce per timed window (not per step)
        st = env.stats_tensor(clear=False)
        ar_ms = None
        if world > 1:
            st_r = st.cpu() if gloo else st
            t0 = time.perf_counter()
            dist.all_reduce(st_r)
            if not gloo:
                torch.cuda.synchronize()
            ar_ms = (time.perf_counter() - t0) * 1e3
            st = st_r
        torch.cuda.synchronize()
    barrier()
    elapsed = max_over_ranks(local_s)
    value = n * world * args.steps / elapsed
    ms_per_step = elapsed / args.steps * 1e3
    clocks = clk.summary()
    stats = dict(zip(uuv.STAT_NAMES, st.double().cpu().tolist()))

    # ---- steady state (L2-resident, back-to-back 1-step graph replays) and a
    # 10-step graph (per-env real-time factor of an open-loop rollout)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        env.replay_graph()
    e1.record(stream)
    torch.cuda.synchronize()
    b2b_ms = e0.elapsed_time(e1) / args.steps
    env.capture_graph(act, n_steps=10)
    for _ in range(5):
        env.replay_graph()
    torch.cuda.synchronize()
    k10 = max(10, args.steps // 10)
    e0.record(stream)
    for _ in range(k10):
        env.replay_graph()
    e1.record(stream)
    torch.cuda.synchronize()
    g10_ms = e0.elapsed_time(e1) / (10 * k10)
    env.capture_graph(act, n_steps=1)

    # ---- e2e through the reference-facing C ABI with pinned host f64 buffers
    act_h = torch.empty((n, env.action_dim), dtype=torch.float64, pin_memory=True)
    act_h.copy_(act.double().cpu())
    act_np = act_h.numpy()
    env.use_pinned_host_buffers()
    for _ in range(args.warmup):
        env.step(act_np)
    barrier()
    k_e2e = max(10, min(args.steps, 300))
    t0 = time.perf_counter()
    for _ in range(k_e2e):
        obs, rew, done = env.step(act_np)
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e_value = n * world * k_e2e / e2e_s
    h2d = n * env.action_dim * 8
    d2h = n * env.obs_dim * 8 + n * 8 + n * 1

    # ---- roofline of the step (FP32 pipe bound)
    hbm_peak, sm_max_mhz, peak_src = measured_peaks()
    sm_count = int(env.info["sm_count"])
    fp32_peak = sm_count * 128 * 2 * sm_max_mhz * 1e6 / 1e12   # TFLOP/s
    fl = flops_per_env_step(c["kind"], n_thr)
    kern_s = local_s / args.steps
    achieved = fl * n / kern_s / 1e12
    bpe = bytes_per_env_step(c["kind"], env.action_dim, env.obs_dim, bool(c["dr"]))
    hbm_achieved = bpe * n / kern_s / 1e9
    launches_per_step = 2 if env.info.get("band64") else 1
    bhash = build_hash()

    line = {
        "metric": "env_steps_per_sec", "value": value, "unit": "env-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.precision.replace("fp", "f"), "data": "synthetic",
        "config": {**workload_config(args.config, world, args.precision),
                   "l2": "flushed between timed steps (256 MiB write)",
                   "step": "fused fp32 step kernel + concurrent fp64 band kernel per step, "
                           "one CUDA-graph replay"},
        "rtf": {"aggregate": value * CONTROL_DT,
                "per_env": CONTROL_DT / (ms_per_step / 1e3),
                "per_env_l2_resident": CONTROL_DT / (b2b_ms / 1e3),
                "per_env_graph10": CONTROL_DT / (g10_ms / 1e3),
                "graph10_ms_per_step": g10_ms,
                "note": "per_env = control_dt / step time (L2 flushed); graph10 = one CUDA "
                        "graph of 10 consecutive steps replayed back to back (open-loop "
                        "rollout, no flush)"},
        "steady_state": {"ms_per_step": b2b_ms, "value": n * world / (b2b_ms / 1e3),
                         "note": "back-to-back 1-step graph replays, L2 not flushed"},
        "e2e": {"value": e2e_value, "unit": "env-steps/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": k_e2e,
                "path": "B200EnvBatch.step -> uuvsim_step_ex (C ABI v1), page-locked host f64 "
                        f"buffers, device.host_io={env.info.get('host_io', '?')}"},
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": fp32_peak,
                     "unit": "TFLOP/s", "frac": achieved / fp32_peak, "traffic": None,
                     "flops_per_env_step": fl,
                     "peak_source": f"derived: {sm_count} SMs x 128 FP32 lanes x 2 x "
                                    f"{sm_max_mhz:.0f} MHz (sm_max_mhz, {peak_src})",
                     "hbm": {"achieved": hbm_achieved, "peak": hbm_peak, "unit": "GB/s",
                             "frac": hbm_achieved / hbm_peak, "bytes_per_env_step": bpe,
                             "peak_source": peak_src}},
        "gpu_launches": args.steps * launches_per_step,
        "clocks": clocks,
        "episode_stats": stats,
        "stats_allreduce_ms": max_over_ranks(ar_ms) if world > 1 else None,
        "engine": {**{k: env.info[k] for k in ("precision", "block", "grid",
                                               "step_kernel_registers", "device_name",
                                               "sm_count", "band64")},
                   "build_hash": bhash},
    }
    env_info_n = n
    del env
    torch.cuda.empty_cache()

    def step_time(name, precision="fp32", strong=False, k=50):
        e2, a2, nt2 = make_engine(name, rank, args, precision, strong=strong)
        for _ in range(5):
            e2.replay_graph()
        ks = timed_steps(e2, flush, stream, k) / k
        out = (e2.num_envs, ks, nt2, e2.action_dim, e2.obs_dim,
               e2.info["step_kernel_registers"], e2.stats()["band64_steps"])
        del e2, a2
        torch.cuda.empty_cache()
        return out

    # ---- N > 1: the north-star scaling workload (C5, 2^20 envs) in the same line
    if world > 1:
        sc = {}
        for mode, strong in (("weak", False), ("strong", True)):
            barrier()
            nn, ks, *_ = step_time("c5", strong=strong, k=30)
            tmax = max_over_ranks(ks)
            total = reduce(float(nn), dist.ReduceOp.SUM)
            sc[mode] = {"envs_per_rank": nn, "envs_total": int(total), "ms_per_step": tmax * 1e3,
                        "value": total / tmax,
                        "env_offset": CONFIGS["c5"]["num_envs"] * rank if not strong else
                        CONFIGS["c5"]["num_envs"] * rank // world}
        line["scaling_c5"] = {"workload": CONFIGS["c5"]["workload"], "weak": sc["weak"],
                              "strong": sc["strong"],
                              "note": "max over ranks of the per-rank device time; weak = "
                                      "2^20 envs per GPU, strong = 2^20 envs for the job"}

    # ---- secondary sizes in the same JSON line (roofline at scale, fp64 mode)
    if not args.no_sweep and world == 1:
        sweep = []
        for name, prec in (("c4", "fp32"), ("c3", "fp32"), ("c3_circle", "fp32"),
                           ("c3_helix", "fp32"), ("c5", "fp32"), ("c2", "fp64"), ("c5", "fp64")):
            if name == args.config and prec == args.precision:
                continue
            nn, ks, nt2, na2, no2, regs, b64 = step_time(name, prec)
            c2 = CONFIGS[name]
            fl2 = flops_per_env_step(c2["kind"], nt2)
            b2 = bytes_per_env_step(c2["kind"], na2, no2, bool(c2["dr"]))
            ent = {"config": name, "precision": prec, "workload": c2["workload"],
                   "num_envs": nn, "ms_per_step": ks * 1e3, "env_steps_per_sec": nn / ks,
                   "fp32_frac": fl2 * nn / ks / 1e12 / fp32_peak,
                   "hbm_frac": (b2 * (2 if prec == "fp64" else 1)) * nn / ks / 1e9 / hbm_peak,
                   "registers": regs,
                   "fp64_band_env_steps_per_step": b64 / 55.0}
            sweep.append(ent)
            if name == "c4" and prec == "fp32":   # env-only and loop
                e2, a2, _ = make_engine("c4", rank, args)
                ent["loop"] = c4_loop(e2)
                del e2, a2
                torch.cuda.empty_cache()
            if name == "c5" and prec == "fp32":   # the kernel where it is throughput-bound
                ach = fl2 * nn / ks / 1e12
                line["roofline_at_scale"] = {
                    "config": name, "bound": "fp32", "achieved": ach, "peak": fp32_peak,
                    "unit": "TFLOP/s", "frac": ach / fp32_peak, "traffic": None,
                    "flops_per_env_step": fl2, "step_ms": ks * 1e3,
                    "hbm": {"achieved": b2 * nn / ks / 1e9, "peak": hbm_peak,
                            "unit": "GB/s", "frac": b2 * nn / ks / 1e9 / hbm_peak,
                            "bytes_per_env_step": b2}}
        line["sweep"] = sweep

    # ---- ncu pass over THIS build: per-launch DRAM traffic and executed flops
    if not args.no_ncu and world == 1 and rank == 0:
        for key, name in (("roofline", args.config), ("roofline_at_scale", "c5")):
            if key not in line:
                continue
            m = ncu_measure(name)
            roof = line[key]
            if not m or "step" not in m:
                roof["traffic"] = None
                roof["ncu"] = m
                continue
            stp = m["step"]
            nenv = env_info_n if name == args.config else CONFIGS[name]["num_envs"]
            traffic = stp.get("dram__bytes_read.sum", 0.0) + stp.get("dram__bytes_write.sum", 0.0)
            ex32 = (2 * stp.get("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", 0.0)
                    + stp.get("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", 0.0)
                    + stp.get("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", 0.0))
            band = m.get("band", {})
            ex64 = (2 * band.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0)
                    + band.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0.0)
                    + band.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0.0))
            step_s = (roof.get("step_ms", ms_per_step)) / 1e3
            roof["traffic"] = traffic
            roof["traffic_source"] = (f"ncu dram__bytes_read+write per launch of {stp['kernel']} "
                                      f"(this run, build {bhash}, cache flushed by ncu)")
            roof["algorithmic_bytes_per_launch"] = roof["hbm"]["bytes_per_env_step"] * nenv
            roof["executed_flops_per_env_step"] = ex32 / nenv
            roof["executed_achieved"] = ex32 / step_s / 1e12
            roof["executed_frac"] = ex32 / step_s / 1e12 / roof["peak"]
            roof["band_fp64_flops_per_launch"] = ex64
            roof["ncu_build_hash"] = bhash

    # ---- CPU baseline: the oracle port on this box's host cores (rank 0, N=1)
    if not args.no_cpu and world == 1 and rank == 0:
        threads = os.cpu_count() or 1
        cfg, _ = build_config(args.config, 0, "fp32")
        sample = cpu_sample_config(cfg, 16384)
        v, k, wall = cpu_oracle_run(sample, 100000, 10.0, threads)
        v1, k1, wall1 = cpu_oracle_run(cpu_sample_config(cfg, 1024), 100000, 5.0, 1)
        line["cpu_baseline"] = {
            "value": v, "unit": "env-steps/s", "cores": threads, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{sample['batch']['num_envs']} envs x {k} steps ({wall:.1f} s) of "
                      f"{args.config} on the C oracle (fp64, OpenMP {threads} threads)",
            "one_thread": {"value": v1, "cores": 1,
                           "sample": f"1024 envs x {k1} steps ({wall1:.1f} s), 1 thread"},
            "reference_python_c1": reference_python_c1()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
