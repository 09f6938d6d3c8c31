"""Summarise an ncu report: per-opcode executed instructions per env-step and key metrics.

    python tools/ncu_mix.py gpurun_out/prof.ncu-rep [num_envs]
"""
import collections
import csv
import io
import re
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[-1])), dict(zip(rows[0], rows[1]))


def mix(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
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


if __name__ == "__main__":
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
    v, u = raw(rep)
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
            "smsp__warps_eligible.avg.per_cycle_active", "smsp__inst_executed.sum",
            "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
            "sm__sass_thread_inst_executed_op_fmul_pred_on.sum",
            "sm__sass_thread_inst_executed_op_fadd_pred_on.sum"]
    for k in keys:
        if k in v:
            print(f"{k:70s} {v[k]:>16s} {u.get(k, '')}")
    by = mix(rep)
    warps = n / 32
    tot = sum(by.values())
    print(f"warp-instructions per env-step: {tot / warps:.1f}")
    for k, c in by.most_common(25):
        print(f"  {k:10s} {c / warps:8.1f}")
