"""Generate tests/golden/*.npz by running the REFERENCE implementation (symgrad) itself.

Run in the build container (needs baseline/_ref or /root/reference):
    python tools/make_golden.py
Each workload in tests/golden_cases.py is executed by the reference's own API; the
fixture stores inputs, output symbols (repr), probabilities, the loss weights and the
gradient of sum(w * probs) w.r.t. every input (reference tape), and for DTKP the output
proof matrices in the reference layout (member u8 [b,n,k,I], present u8 [b,n,k]).
Inputs are fp32-representable values fed as float64, so the fp32 GPU path and the fp64
reference see identical numbers.  The fixtures pin both the oracle restatement
(tests/test_oracle.py) and the CUDA path (tests/test_gpu_golden.py).
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT))
for cand in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if (cand / "symgrad").exists():
        sys.path.insert(0, str(cand))
        break

import symgrad as S  # noqa: E402
from symgrad import programs as SP  # noqa: E402
from symgrad import tensor as T  # noqa: E402
from symgrad.kernels import dedup_topk as ref_dedup_topk  # noqa: E402

import golden_cases as G  # noqa: E402

OUT = ROOT / "tests" / "golden"


def run_case(name):
    prov_name, k, prog, syms_fn, _, _ = G.CASES[name]
    prov = S.provenance_from_name(prov_name, k or 1)
    inputs = G.case_inputs(name)
    symbol_lists = syms_fn(SP)
    ctx = S.ProgramContext(prov)
    leaves = [ctx.tape.leaf(x) for x in inputs]
    dists = [S.make_distribution(ctx, lf, s) for lf, s in zip(leaves, symbol_lists)]
    out = prog(S, SP, ctx, dists)
    probs = S.get_probs(out)
    w = G.loss_weights(name, probs.shape)
    loss = T.reduce_sum(T.reduce_sum(T.mul(probs, T.Tensor(w)), 1), 0)
    grads = ctx.tape.backward(loss)
    res = {"symbols": json.dumps([repr(s) for s in out.symbols]), "probs": probs.data.copy(), "w": w,
           "n_inputs": len(inputs)}
    for i, (x, lf) in enumerate(zip(inputs, leaves)):
        res[f"in{i}"] = x
        res[f"grad{i}"] = grads[lf].data.copy()
    if prov_name == "dtkp":
        res["member"] = out.tags.aligned_member().copy()
        res["present"] = out.tags.present.copy()
    return res


def loss_nll_cases():
    """The reference's learn.loss_nll (learn.py:92-119) and its tape gradient on fp32-
    representable probabilities: rows short of and past 1 (clamped disjunctions), None
    targets (floor penalty), and shapes that take each kernel schedule of the fused loss
    (one-pass, chunked row sums at small batch / many symbols)."""
    from symgrad.learn import loss_nll

    rng = np.random.default_rng(31)
    specs = [(8, 12, 1.0, 2), (3, 8, None, 0), (64, 300, 1.0, 1), (1000, 20, 3.0, 17), (40, 2500, 0.5, 3),
             (5, 7, 0.0, 1)]
    out = {"n_cases": len(specs)}
    for c, (b, n, scale, n_none) in enumerate(specs):
        if scale is None:
            probs = np.full((b, n), 1.0 / n)
        elif scale == 0.0:
            probs = rng.uniform(0.0, 1.0, size=(b, n)) * (rng.uniform(size=(b, n)) < 0.3)
        else:
            probs = rng.uniform(0.0, 1.0, size=(b, n))
            probs = probs / probs.sum(axis=1, keepdims=True) * scale * rng.uniform(0.5, 1.5, size=(b, 1))
        probs = probs.astype(np.float32).astype(np.float64)
        targets = rng.integers(0, n, size=b).tolist()
        for i in rng.choice(b, size=n_none, replace=False):
            targets[int(i)] = None
        tape = T.GradientTape()
        leaf = tape.leaf(probs)
        loss = loss_nll(leaf, targets)
        grad = tape.backward(loss)[leaf].data
        out[f"c{c}_probs"] = probs
        out[f"c{c}_targets"] = np.asarray([-1 if t is None else t for t in targets], dtype=np.int64)
        out[f"c{c}_loss"] = np.float64(loss.item())
        out[f"c{c}_grad"] = grad
    return out


def save(name, **arrays):
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / f"{name}.npz", **{k: np.asarray(v) for k, v in arrays.items()})
    print("wrote", name)


def main():
    only = [a for a in sys.argv[1:] if not a.startswith("-")]
    for name in G.CASES:
        if G.CASES[name][0] == "max":  # no max provenance in the reference: tools/make_golden_max.py
            continue
        if only and name not in only:
            continue
        t0 = time.perf_counter()
        save(name, **run_case(name))
        print(f"  {name}: {time.perf_counter() - t0:.1f} s", flush=True)
    if only:
        if "loss_nll" in only:
            save("loss_nll", **loss_nll_cases())
        return
    # dedup_topk: compiled-reference outputs on fuzz cases with exact ties (test_kernels.py:98-111)
    cases = {}
    rng = np.random.default_rng(30)
    for c in range(80):
        M, R, I, k = int(rng.integers(1, 6)), int(rng.integers(1, 12)), int(rng.integers(1, 130)), int(rng.integers(1, 9))
        member = (rng.uniform(size=(M, R, I)) < 0.4).astype(np.uint8)
        present = (rng.uniform(size=(M, R)) < 0.8).astype(np.uint8)
        member &= present[:, :, None]
        p = np.round(rng.uniform(0.05, 0.95, size=(M, I)), 1)
        om, op = ref_dedup_topk(member, present, p, k)
        cases.update({f"c{c}_member": member, f"c{c}_present": present, f"c{c}_p": p, f"c{c}_k": k,
                      f"c{c}_om": om, f"c{c}_op": op})
    save("dedup_topk_fuzz", n_cases=80, **cases)
    save("loss_nll", **loss_nll_cases())
    print("reference backend:", S.backend_name())


if __name__ == "__main__":
    main()
