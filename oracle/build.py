"""ORACLE — TEST INFRASTRUCTURE ONLY: build recipe for the CPU checkers.

* ``oracle/_build/liboracle.so``  — gcc build of the plain-C restatement
  ``oracle/dedup_topk.c`` (always; travels to the GPU box).
* ``oracle/_ref/``                — the reference's own native proof kernel, compiled from
  its source where it lies (``/root/reference/pkg/src/symgrad/_dtkpcore.pyx``): cython
  generates C into ``oracle/_ref/`` and gcc builds ``_dtkpcore*.so`` there.  Only when
  ``/root/reference`` exists (this container); the GPU box uses the prebuilt files.

Usage: ``python -m oracle.build``.  Nothing here is imported by the product package.
"""

from __future__ import annotations

import shutil
import subprocess
import sys
import sysconfig
from pathlib import Path

HERE = Path(__file__).resolve().parent
BUILD = HERE / "_build"
REF_OUT = HERE / "_ref"
REF_PYX = Path("/root/reference/pkg/src/symgrad/_dtkpcore.pyx")
LIB = BUILD / "liboracle.so"


def build_c(force: bool = False) -> Path:
    src = HERE / "dedup_topk.c"
    BUILD.mkdir(exist_ok=True)
    if force or not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        cmd = ["gcc", "-O2", "-shared", "-fPIC", "-std=c11", str(src), "-o", str(LIB)]
        subprocess.run(cmd, check=True)
    return LIB


def build_ref(force: bool = False) -> Path | None:
    """Cythonize + gcc the reference's _dtkpcore.pyx into oracle/_ref (sources stay put)."""
    if not REF_PYX.exists():
        return None
    REF_OUT.mkdir(exist_ok=True)
    ext = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
    so = REF_OUT / f"_dtkpcore{ext}"
    if so.exists() and not force:
        return so
    try:
        import numpy as np
    except ImportError:  # pragma: no cover
        return None
    cython = shutil.which("cython") or shutil.which("cython3")
    c_file = REF_OUT / "_dtkpcore.c"
    if cython:
        cmd = [cython, "-3", str(REF_PYX), "-o", str(c_file)]
    else:
        cmd = [sys.executable, "-m", "cython", "-3", str(REF_PYX), "-o", str(c_file)]
    subprocess.run(cmd, check=True, capture_output=True)
    inc = [sysconfig.get_paths()["include"], np.get_include()]
    cmd = ["gcc", "-O2", "-shared", "-fPIC", "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION",
           *[f"-I{i}" for i in inc], str(c_file), "-o", str(so)]
    subprocess.run(cmd, check=True, capture_output=True)
    return so


def build(force: bool = False):
    lib = build_c(force)
    ref = None
    try:
        ref = build_ref(force)
    except (subprocess.CalledProcessError, OSError) as exc:  # the reference is optional
        print(f"oracle/_ref not built: {exc}", file=sys.stderr)
    return lib, ref


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
