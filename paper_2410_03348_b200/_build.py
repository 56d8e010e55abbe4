"""Build the sm_100a C-ABI library ``libsgb200.so`` in-tree with nvcc.

Every translation unit is compiled for ``-gencode arch=compute_100a,code=sm_100a`` with
``-lineinfo`` (so ncu's source page maps to the kernels) and linked into one shared
library with the static CUDA runtime.  The fused DTKP apply kernel is compiled once per
proof count K (``dtkp_apply_k.cu`` with ``-DSG_DTKP_K=K``) so the variants build in
parallel.  Usage: ``python -m paper_2410_03348_b200._build [--force]``.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
BUILD = PKG / "build"
LIB = PKG / "libsgb200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the sm_100a library cannot be built")


def _units():
    """(object name, source, extra flags) for every translation unit."""
    units = [
        ("damp.o", CSRC / "damp.cu", []),
        ("chain_g4.o", CSRC / "chain.cu", ["-DSG_CHAIN_GROUPS=4"]),
        ("chain_g8.o", CSRC / "chain.cu", ["-DSG_CHAIN_GROUPS=8"]),
        ("chain_g16.o", CSRC / "chain.cu", ["-DSG_CHAIN_GROUPS=16"]),
        ("chain_api.o", CSRC / "chain_api.cu", []),
        ("dtkp.o", CSRC / "dtkp.cu", []),
        ("maxprod.o", CSRC / "maxprod.cu", []),
        ("maxchain.o", CSRC / "maxchain.cu", []),
    ]
    for k in range(1, 9):
        units.append((f"dtkp_apply_k{k}.o", CSRC / "dtkp_apply_k.cu", [f"-DSG_DTKP_K={k}"]))
    return units


def _deps(src: Path = None):
    """A unit depends on its own source and every header (a .cu never includes another)."""
    heads = sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))
    return heads + [src] if src is not None else sorted(CSRC.glob("*.cu")) + heads


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    nvcc = _nvcc()
    BUILD.mkdir(exist_ok=True)
    deps = _deps()
    jobs = []
    for obj, src, extra in _units():
        out = BUILD / obj
        if force or _stale(out, _deps(src)):
            cmd = [nvcc, *ARCH, *NVCC_FLAGS, *os.environ.get("SG_NVCC_EXTRA", "").split(), f"-I{INCLUDE}", *extra,
                   "-c", str(src), "-o", str(out)]
            jobs.append((obj, cmd))

    def run(job):
        obj, cmd = job
        if verbose:
            print(" ".join(cmd), flush=True)
        proc = subprocess.run(cmd, capture_output=True, text=True)
        if proc.returncode != 0:
            raise RuntimeError(f"nvcc failed for {obj}:\n{proc.stdout}\n{proc.stderr}")
        return obj

    if jobs:
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as pool:
            list(pool.map(run, jobs))
    objs = [BUILD / obj for obj, _, _ in _units()]
    if force or jobs or _stale(LIB, objs):
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-cudart", "static"]
        proc = subprocess.run(cmd, capture_output=True, text=True)
        if proc.returncode != 0:
            raise RuntimeError(f"link failed:\n{proc.stdout}\n{proc.stderr}")
        os.replace(tmp, LIB)
    build_planner(force)
    return LIB


PLANNER_SRC = CSRC / "planner.cpp"


def planner_path() -> Path:
    import sysconfig

    return PKG / f"_planner{sysconfig.get_config_var('EXT_SUFFIX')}"


def build_planner(force: bool = False) -> Path:
    """The native host planner (CPython extension, g++ -O2): apply_if's map/shuffle loop."""
    import sysconfig

    out = planner_path()
    if not force and not _stale(out, [PLANNER_SRC]):
        return out
    cxx = os.environ.get("CXX") or shutil.which("g++") or "g++"
    tmp = out.with_name(out.name + ".tmp")
    cmd = [cxx, "-O2", "-std=c++17", "-shared", "-fPIC", "-fno-strict-aliasing", "-Wall",
           f"-I{sysconfig.get_paths()['include']}", str(PLANNER_SRC), "-o", str(tmp)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"planner build failed:\n{proc.stdout}\n{proc.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    path = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(path)
