"""The opt-in staged short-filter Toeplitz kernels (SG_CONV_STAGED=1: k_convs_fwd/bwd)
against the reference fixtures, in a subprocess (the switch is read once per process)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r'''
import sys
sys.path.insert(0, "{root}"); sys.path.insert(0, "{root}/tests")
import numpy as np
from paper_2410_03348_b200 import _native as N, ops
from runners import assert_close_rel, load_golden, run_gpu
from paper_2410_03348_b200.plan import build_plan
kp = build_plan(lambda a, b: a + b, None, [tuple(range(10))] * 2).kernel_plan()
assert ops.conv_staged(kp), "staged kernels not selected"
for name in ("damp_sweep_a2_s10", "damp_sum2", "damp_sum4", "damp_bcast_reuse", "damp_sweep_a2_s37"):
    gold = load_golden(name)
    got = run_gpu(name)
    assert got["symbols"] == gold["symbols"], name
    assert_close_rel(got["probs"], gold["probs"], 1e-5, 1e-7, what=name)
    for i in range(int(gold["n_inputs"])):
        assert_close_rel(got["grads"][i], gold[f"grad{{i}}"], 1e-5, 1e-6, what=name)
print("staged ok")
'''


def test_staged_conv_kernels_match_reference(cuda):
    env = dict(os.environ, SG_CONV_STAGED="1", SG_FUSE_CHAINS="0")
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], capture_output=True, text=True, env=env,
                         timeout=600)
    assert out.returncode == 0 and "staged ok" in out.stdout, out.stderr[-3000:]
