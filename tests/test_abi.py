"""CPU: the C-ABI library loads, exports every entry point of include/sgb200.h, and the
ctypes mirrors of its structs have the C layout (no kernel is launched here)."""

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "sgb200.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t)\s+(sg_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_hot_path():
    names = declared_functions()
    for required in ["sg_damp_apply_fwd", "sg_damp_apply_bwd", "sg_dtkp_apply", "sg_dtkp_probs_fwd",
                     "sg_dtkp_probs_bwd", "sg_dedup_topk", "sg_rows_gather", "sg_damp_rows_add", "sg_segsum_run"]:
        assert required in names


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2410_03348_b200 import _native

    lib = _native.load()
    for name in declared_functions():
        assert hasattr(lib, name), f"libsgb200.so does not export {name}"
        assert name in _native.EXPORTS, f"{name} has no ctypes prototype"
    assert lib.sg_version() >= 2
    nm = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True, text=True)
    exported = set(re.findall(r"\bT (sg_\w+)", nm.stdout))
    assert set(declared_functions()) <= exported


def test_library_is_sm100a():
    from paper_2410_03348_b200 import _native

    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_struct_layout_matches_c(tmp_path):
    from paper_2410_03348_b200 import _native as N
    import ctypes

    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "sgb200.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(sg_segsum),"
        " sizeof(sg_damp_plan), sizeof(sg_dtkp_operand), sizeof(sg_dtkp_apply_desc), offsetof(sg_damp_plan, fwd),"
        " offsetof(sg_dtkp_apply_desc, p), offsetof(sg_dtkp_apply_desc, seg), offsetof(sg_dtkp_apply_desc, merge),"
        " sizeof(sg_maxprod_plan), offsetof(sg_maxprod_plan, seg_off), offsetof(sg_maxprod_plan, in_recs),"
        " offsetof(sg_dtkp_apply_desc, inner_ops), offsetof(sg_dtkp_apply_desc, rows_ranked));"
        "return 0;}\n"
    )
    exe = tmp_path / "layout"
    subprocess.run(["gcc", f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    expect = [
        ctypes.sizeof(N.SgSegsum), ctypes.sizeof(N.SgDampPlan), ctypes.sizeof(N.SgDtkpOperand),
        ctypes.sizeof(N.SgDtkpApplyDesc), N.SgDampPlan.fwd.offset, N.SgDtkpApplyDesc.p.offset,
        N.SgDtkpApplyDesc.seg.offset, N.SgDtkpApplyDesc.merge.offset, ctypes.sizeof(N.SgMaxprodPlan),
        N.SgMaxprodPlan.seg_off.offset, N.SgMaxprodPlan.in_recs.offset, N.SgDtkpApplyDesc.inner_ops.offset,
        N.SgDtkpApplyDesc.rows_ranked.offset,
    ]
    assert vals == expect
