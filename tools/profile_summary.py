"""Turn ncu captures into the committed evidence under profiles/.

    python tools/profile_summary.py --tag r1 gpurun_out/prof_c2.ncu-rep:c2:4096 \
        gpurun_out/prof_c5.ncu-rep:c5:1048576 ... [--launches gpurun_out/launches_c2.csv]

Writes profiles/<tag>_ncu_summary.md (key metrics, executed-instruction mix
per env-step, algorithmic vs executed FP32 work, dram traffic per env-step).
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

KEYS = [
    ("gpu__time_duration.sum", "kernel duration (cold caches, serialised)"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps / cycle / SMSP"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "thread FFMA"),
    ("sm__sass_thread_inst_executed_op_fmul_pred_on.sum", "thread FMUL"),
    ("sm__sass_thread_inst_executed_op_fadd_pred_on.sum", "thread FADD"),
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    return dict(zip(rows[0], rows[-1])), dict(zip(rows[0], rows[1]))


def to_bytes(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v) * mult


def mix(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv",
                                           "--print-source", "sass"))))
    hdr = rows[1]
    ia, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
    by = collections.Counter()
    for r in rows[2:]:
        try:
            n = int(r[ia])
        except (ValueError, IndexError):
            continue
        op = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip())
        by[op.split()[0].split(".")[0] if op else "?"] += n
    return by


def launch_share(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    dur = collections.defaultdict(list)
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) > iv and r[im] == "gpu__time_duration.sum":
            name = r[ik].split("(")[0].split("<")[0].replace("void ", "").strip()
            dur[name].append(float(r[iv]))
    return dur


def main():
    from bench import CONFIGS, bytes_per_env_step, flops_per_env_step
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+",
                    help="rep.ncu-rep:config:num_envs[:band] (band: the fp64 band kernel)")
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--launches", action="append", default=[])
    a = ap.parse_args()
    out = [f"# ncu summary ({a.tag})", "",
           "Captured with `ncu --set full --clock-control none --import-source on` on one B200"
           " (tools/ncu_run_r2.sh; step kernel `-k regex:k_step`, fp64 band kernel"
           " `-k regex:k_band`, both after 300 steps in the tumbling regime).  ncu flushes"
           " caches and serialises launches, so durations are cold-cache and the band kernel"
           " is shown alone (in a step it runs concurrently with the step kernel);"
           " bench.py's CUDA-event timings are the reported numbers.", ""]
    traffic = {}
    for spec in a.reports:
        parts = spec.split(":")
        rep, cfg, n = parts[:3]
        n = int(n)
        v, u = raw(rep)
        c = CONFIGS[cfg]
        if len(parts) > 3 and parts[3] == "band":
            by = mix(rep)
            out += [f"## {cfg} band kernel: {c['workload']}", "",
                    f"report: `{Path(rep).name}`  kernel: `{v.get('Kernel Name', '?')[:90]}`", "",
                    "| metric | value |", "|---|---|"]
            for k, label in KEYS:
                if k in v:
                    out.append(f"| {label} (`{k}`) | {v[k]} {u.get(k, '')} |")
            ex64 = 2 * by.get("DFMA", 0) + by.get("DMUL", 0) + by.get("DADD", 0)
            tot = sum(by.values())
            out += ["", f"* executed warp-instructions: {tot:.0f} (fp64 DFMA x2 + DMUL + DADD "
                    f"warp-ops: {ex64:.0f}); the kernel scans {n} flag bytes and steps this "
                    f"step's band candidates in fp64", "", "| opcode | warp-instructions |",
                    "|---|---|"]
            for k2, cnt in by.most_common(12):
                out.append(f"| {k2} | {cnt:.0f} |")
            out.append("")
            continue
        name = [k for k in v if k == "Kernel Name"]
        out += [f"## {cfg}: {c['workload']}", "", f"report: `{Path(rep).name}`  kernel: "
                f"`{v.get('Kernel Name', '?')[:90]}`", "", "| metric | value |", "|---|---|"]
        for k, label in KEYS:
            if k in v:
                out.append(f"| {label} (`{k}`) | {v[k]} {u.get(k, '')} |")
        rd = to_bytes(v["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
        wr = to_bytes(v["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
        traffic[cfg] = rd + wr
        n_thr = [8 if vv == "bluerov2_heavy" else 6 for vv in c["vehicles"]]
        n_act = max(n_thr)
        obs_dim = 12 if c["kind"] == "station_keeping" else 36
        alg_b = bytes_per_env_step(c["kind"], n_act, obs_dim, bool(c["dr"]))
        fl = flops_per_env_step(c["kind"], n_thr)
        by = mix(rep)
        per = n / 32                     # warp-instructions -> thread-instructions per env
        ex = (2 * by.get("FFMA", 0) + by.get("FMUL", 0) + by.get("FADD", 0)) / per
        out += ["", f"* DRAM traffic per env-step: {(rd + wr) / n:.1f} B (algorithmic minimum "
                f"{alg_b} B; below it when L2 still holds dirty lines at kernel end)",
                f"* FP32 work per env-step: algorithmic {fl:.0f} flop (reference dense count),"
                f" executed {ex:.0f} flop (SASS FFMA x2 + FMUL + FADD; the structure-"
                f"specialised kernel skips the reference's exact-zero terms)", ""]
        warps = n / 32 / (2 if "pair" in v.get("Kernel Name", "") else 1)
        tot = sum(by.values())
        out += [f"Executed warp-instructions per env-step: **{tot / (n / 32):.0f}**", "",
                "| opcode | per env-step |", "|---|---|"]
        for k2, cnt in by.most_common(16):
            out.append(f"| {k2} | {cnt / (n / 32):.1f} |")
        out.append("")
    for lp in a.launches:
        dur = launch_share(lp)
        tot = sum(sum(x) for x in dur.values())
        harness = sum(sum(x) for k2, x in dur.items() if k2.startswith("at::"))
        step = sum(sum(x) for k2, x in dur.items() if k2.startswith("uuv::k_step"))
        out += [f"## launch list `{Path(lp).name}` (gpu__time_duration, cold, serialised)", "",
                "`at::*` kernels are bench.py's 256 MiB L2-flush writes between timed steps"
                " (harness, not the step); without them the step kernel is "
                f"{step / max(tot - harness, 1e-9):.1%} of the device time.", "",
                "| kernel | launches | mean us | share |", "|---|---|---|---|"]
        for k2, xs in sorted(dur.items(), key=lambda kv: -sum(kv[1])):
            out.append(f"| {k2[:60]} | {len(xs)} | {sum(xs) / len(xs) / 1e3:.2f} | "
                       f"{sum(xs) / tot:.1%} |")
        out.append("")
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    (prof / f"{a.tag}_ncu_summary.md").write_text("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
