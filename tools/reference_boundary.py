"""Boundary proof from the reference side: the reference's OWN tests, run on a copy of the
installed reference (baseline/_ref) whose FFI point ``kernels.py`` carries the binding
stub of INTEGRATION.md §2 — extracted from that document, so the documented stub is
exactly what runs — with ``dedup_topk`` served by ``sg_dedup_topk`` on the B200.

What is patched in the COPY (baseline/_ref itself stays unmodified):
  * kernels.py: the INTEGRATION.md §2 stub (``_sg`` loader, ``_dedup_topk_b200``,
    ``backend_name``) and the one-line dispatch at the top of ``dedup_topk``;
  * ``_dtkpcore``: a shim module whose ``dedup_topk`` is the B200 backend, so the
    reference's compiled-vs-numpy equivalence tests (test_kernels.py:86-111) compare the
    sm_100a kernel against the reference's numpy implementation.

Then pytest runs the reference's test_kernels.py (except the dispatch-name test, which
hard-codes "compiled"; its B200 counterpart is checked here), test_provenance.py,
test_distribution.py and test_programs.py: every DTKP conj / disj / group_disj /
tags_from_proofs of those suites goes through the sm_100a kernel.

    python tools/reference_boundary.py [--out profiles/r02_reference_boundary.txt]
"""

from __future__ import annotations

import argparse
import os
import re
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
LIB = ROOT / "paper_2410_03348_b200" / "libsgb200.so"

SHIM = '''"""B200 shim of the compiled proof core (boundary test only): dedup_topk -> sg_dedup_topk."""
from symgrad.kernels import _dedup_topk_b200 as dedup_topk  # noqa: F401
'''


def integration_stub() -> tuple[str, str]:
    """(loader + backend function, dispatch code) from INTEGRATION.md §2's python block."""
    text = (ROOT / "INTEGRATION.md").read_text()
    sec = text[text.index("## 2."):]
    block = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    head, _, tail = block.partition("def backend_name()")
    return head, "def backend_name()" + tail


def patch_copy(dst: Path):
    shutil.copytree(REF / "symgrad", dst / "symgrad")
    k = dst / "symgrad" / "kernels.py"
    src = k.read_text()
    head, tail = integration_stub()
    # the stub's loader and backend go right after the reference's own backend selection
    anchor = "def backend_name() -> str:"
    i = src.index(anchor)
    src = src[:i] + head + "\n\n" + src[i:]
    # the stub's backend_name replaces the reference's; its dispatch line opens dedup_topk
    src = re.sub(r"def backend_name\(\) -> str:\n    return \"numpy\" if _compiled is None else \"compiled\"\n",
                 "def backend_name() -> str:\n    return \"sm_100a\" if _sg is not None else "
                 "(\"numpy\" if _compiled is None else \"compiled\")\n", src)
    body = "    member = np.ascontiguousarray(member, dtype=np.uint8)\n"
    j = src.index(body, src.index("def dedup_topk(member, present, p, k):"))
    src = src[:j] + "    if _sg is not None:\n        return _dedup_topk_b200(member, present, p, k)\n" + src[j:]
    k.write_text(src)
    assert "_dedup_topk_b200" in tail  # the documented dispatch is what was inserted
    for so in (dst / "symgrad").glob("_dtkpcore*.so"):
        so.unlink()
    (dst / "symgrad" / "_dtkpcore.py").write_text(SHIM)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    if not (REF / "symgrad").exists() or not (REF / "tests").exists():
        raise SystemExit("baseline/_ref (with tests/) missing: run __graft_entry__.build() where /root/reference exists")
    with tempfile.TemporaryDirectory(prefix="symgrad_b200_") as tmp:
        tmp = Path(tmp)
        patch_copy(tmp)
        shutil.copytree(REF / "tests", tmp / "tests")
        env = dict(os.environ, SYMGRAD_B200="1", SGB200_LIB=str(LIB), PYTHONPATH=str(tmp))
        env.pop("SYMGRAD_PURE", None)
        check = subprocess.run([sys.executable, "-c", "import symgrad.kernels as k, symgrad._dtkpcore as c; "
                                "print(k.backend_name(), c.dedup_topk.__name__)"],
                               capture_output=True, text=True, env=env, cwd=tmp)
        lines = [f"backend: {check.stdout.strip()} {check.stderr.strip()[-300:]}"]
        tests = ["tests/test_kernels.py", "tests/test_provenance.py", "tests/test_distribution.py",
                 "tests/test_programs.py"]
        run = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", *tests, "-k",
                              "not test_dispatch_matches_environment"], capture_output=True, text=True, env=env,
                             cwd=tmp)
        lines.append(run.stdout[-4000:])
        lines.append(run.stderr[-2000:])
        ok = run.returncode == 0 and check.stdout.startswith("sm_100a _dedup_topk_b200")
        lines.append(f"RESULT: {'PASS' if ok else 'FAIL'} (pytest rc={run.returncode})")
    report = "\n".join(lines)
    print(report)
    if args.out:
        Path(args.out).write_text(report + "\n")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
