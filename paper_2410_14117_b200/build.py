"""Build libuuvsim_core.so in-tree (sm_100a only).

    python -m paper_2410_14117_b200.build [--force]

nvcc compiles the kernels for ``-gencode arch=compute_100a,code=sm_100a`` with
``-lineinfo`` (fp32 TU normal, fp64 TU with ``-fmad=false``); g++ compiles the
host engine and the C ABI; nvcc links one shared library with the CUDA runtime
linked statically.  Output: paper_2410_14117_b200/_lib/libuuvsim_core.so.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
OBJDIR = LIBDIR / "obj"
LIB = LIBDIR / "libuuvsim_core.so"
REPO = PKG.parent
INCLUDE = REPO / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _cuda_home() -> Path:
    for c in (os.environ.get("CUDA_HOME"), "/usr/local/cuda"):
        if c and Path(c, "bin", "nvcc").is_file():
            return Path(c)
    nvcc = shutil.which("nvcc")
    if nvcc:
        return Path(nvcc).resolve().parent.parent
    raise RuntimeError("nvcc not found (set CUDA_HOME)")


def _nlohmann_include() -> Path:
    cands = [os.environ.get("NLOHMANN_INCLUDE", "")]
    cands += glob.glob(str(Path(sys.prefix) / "lib" / "python3*" / "site-packages" / "include" /
                           "cudnn_frontend" / "thirdparty"))
    cands += glob.glob("/opt/prime-rl/.venv/lib/python3*/site-packages/include/cudnn_frontend/thirdparty")
    for c in cands:
        if c and Path(c, "nlohmann", "json.hpp").is_file():
            return Path(c)
    raise RuntimeError("nlohmann/json.hpp not found (set NLOHMANN_INCLUDE)")


def _host_cxx() -> str:
    for c in ("/usr/bin/g++", shutil.which("g++") or ""):
        if c and Path(c).is_file():
            return c
    raise RuntimeError("g++ not found")


def _stale(out: Path, deps) -> bool:
    if not out.is_file():
        return True
    t = out.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: Path | None = None,
          defines=()) -> Path:
    """Compile + link.  ``out``/``defines`` build an experimental variant (own obj dir)."""
    cuda = _cuda_home()
    lib = Path(out) if out else LIB
    objdir = (lib.parent / "obj") if out else OBJDIR
    nvcc = str(cuda / "bin" / "nvcc")
    cxx = _host_cxx()
    objdir.mkdir(parents=True, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    headers = sorted(glob.glob(str(CSRC / "*.h")) + glob.glob(str(CSRC / "*.cuh")) +
                     [str(INCLUDE / "uuvsim.h")])
    common_nv = [nvcc, "-std=c++17", "-O3", "-lineinfo", *ARCH, "-ccbin", cxx,
                 "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills", "-I", str(CSRC), *dflags]
    jobs = [
        (objdir / "k_f32.o", [*common_nv, "-c", str(CSRC / "k_f32.cu")], [CSRC / "k_f32.cu"]),
        (objdir / "k_f64.o", [*common_nv, "-fmad=false", "-c", str(CSRC / "k_f64.cu")],
         [CSRC / "k_f64.cu"]),
        (objdir / "k_band.o", [*common_nv, "-fmad=false", "-c", str(CSRC / "k_band.cu")],
         [CSRC / "k_band.cu"]),
        (objdir / "rl_kernels.o", [*common_nv, "-c", str(CSRC / "rl_kernels.cu")],
         [CSRC / "rl_kernels.cu", INCLUDE / "uuvsim_rl.h"]),
    ]
    host = [cxx, "-std=c++17", "-O2", "-fPIC", "-Wall", "-Wno-unused-function",
            "-I", str(cuda / "include"), "-I", str(_nlohmann_include()), "-I", str(CSRC), "-c"]
    for name in ("engine.cpp", "capi.cpp"):
        jobs.append((objdir / (name[:-4] + ".o"), [*host, *dflags, str(CSRC / name)], [CSRC / name]))
    todo = [(o, cmd + ["-o", str(o)]) for o, cmd, src in jobs
            if force or _stale(o, [*src, *headers])]

    def run(item):
        o, cmd = item
        if verbose:
            print(" ".join(cmd))
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed for {o.name}:\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with ThreadPoolExecutor(max_workers=4) as ex:
        for msg in ex.map(run, todo):
            if msg and verbose:
                print(msg)
    if out is None:
        build_hostcall(force)
    objs = [str(o) for o, _, _ in jobs]
    if force or todo or _stale(lib, objs):
        cmd = [nvcc, "-shared", *ARCH, "-ccbin", cxx, "-o", str(lib), *objs,
               "-Xlinker", "--exclude-libs,ALL"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


def build_hostcall(force: bool = False) -> Path | None:
    """CPython fast path of the host-ABI step (csrc/hostcall.c -> _hostcall<EXT>),
    binding glue only; skipped (None) when the Python headers are absent."""
    import sysconfig
    inc = sysconfig.get_paths().get("include", "")
    if not inc or not Path(inc, "Python.h").is_file():
        return None
    out = PKG / ("_hostcall" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))
    src = CSRC / "hostcall.c"
    if not force and not _stale(out, [src]):
        return out
    cc = shutil.which("gcc") or shutil.which("cc")
    if not cc:
        return None
    cmd = [cc, "-O2", "-shared", "-fPIC", "-Wall", "-I", inc, str(src), "-o", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"hostcall build failed:\n{r.stdout}\n{r.stderr}")
    return out


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--out", default=None, help="variant library path (own obj dir)")
    ap.add_argument("-D", action="append", default=[], help="preprocessor define")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.v, out=a.out, defines=a.D))
