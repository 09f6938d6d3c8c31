"""bench.py keeps the driver's JSON-line contract (both arms)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _run(*args, timeout=600):
    env = dict(os.environ)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                       text=True, timeout=timeout, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "3", "--warmup", "1")
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["metric"] == "env_steps_per_sec" and d["value"] > 0 and d["higher_is_better"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_gpu_arm_line():
    d = _run("--steps", "20", "--warmup", "3", "--no-sweep", "--no-ncu")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "roofline", "cpu_baseline", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["steps"] == 20 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["metric"] == "env_steps_per_sec"
    assert "workload" in d["config"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"]
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"]
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in d["clocks"]
    # the fused step kernel, plus the concurrent fp64 band kernel (band64 on)
    assert d["gpu_launches"] == 20 * (2 if d["engine"]["band64"] else 1)
    for k in ("per_env", "per_env_graph10"):
        assert d["rtf"][k] > 0
    assert d["cpu_baseline"]["one_thread"]["cores"] == 1 and d["cpu_baseline"]["cpu_model"]


def test_reference_arm_under_torchrun_prints_once():
    """Driver launch for N > 1: rank 0 alone runs and prints; the others exit 0."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", "29531", str(ROOT / "bench.py"), "--impl", "reference",
                        "--gpus", "2", "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2


@pytest.mark.gpu
def test_gpu_arm_under_torchrun_two_ranks():
    """The N > 1 path of the GPU arm (driver launch via torch.distributed.run):
    two ranks on one device with the gloo backend -- weak-scaling headline,
    max-over-ranks timing, the stats all-reduce and the C5 weak / strong
    scaling block execute; rank 0 alone prints the line."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", "29533", str(ROOT / "bench.py"), "--gpus", "2",
                        "--steps", "10", "--warmup", "3", "--dist-backend", "gloo",
                        "--no-cpu", "--no-ncu"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["num_envs_total"] == 2 * d["config"]["num_envs_per_gpu"]
    assert d["stats_allreduce_ms"] is not None
    assert d["episode_stats"]["env_steps"] > 0
    sc = d["scaling_c5"]
    assert sc["weak"]["envs_total"] == 2 * (1 << 20) and sc["strong"]["envs_total"] == 1 << 20
    assert sc["weak"]["value"] > 0 and sc["strong"]["value"] > 0
