"""A plain-C host (examples/host_step.c) drives the library through include/uuvsim.h
exactly as a non-Python caller of the reference's capi.rs would: it compiles here
(gcc, no GPU needed) and, on a GPU, steps a batch and checks the error contract."""

from __future__ import annotations

import json
import shutil
import subprocess
from pathlib import Path

import pytest

import paper_2410_14117_b200 as uuv

ROOT = Path(__file__).resolve().parent.parent


def _compile(tmp_path) -> Path:
    gcc = shutil.which("gcc") or "/usr/bin/gcc"
    exe = tmp_path / "host_step"
    lib = ROOT / "paper_2410_14117_b200" / "_lib"
    r = subprocess.run([gcc, "-O2", "-Wall", "-Wextra", "-Werror", "-I", str(ROOT / "include"),
                        str(ROOT / "examples" / "host_step.c"), "-L", str(lib), "-luuvsim_core",
                        f"-Wl,-rpath,{lib}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_host_compiles_against_the_header(tmp_path):
    _compile(tmp_path)


@pytest.mark.gpu
def test_c_host_steps_the_engine(tmp_path):
    exe = _compile(tmp_path)
    cfg = uuv.engine_config_dict(uuv.bluerov2_params(), uuv.TaskSpec(episode_len=50), 4096, 0)
    path = tmp_path / "c2.json"
    path.write_text(json.dumps(cfg))
    r = subprocess.run([str(exe), str(path), "120"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    f = r.stdout.split()
    vals = dict(zip(f[0::2], f[1::2]))
    assert int(vals["envs"]) == 4096 and int(vals["steps"]) == 120
    assert int(vals["dones"]) >= 2 * 4096                   # two truncations at least
    assert vals["bad_len_code"] == "3" and vals["stale_code"] == "2"
