"""Generate tests/golden/max_*.npz for the max-product ("max/DAMP") variant.

The reference has no max provenance, so these fixtures are computed with
the REFERENCE's own Tensor primitives on its own GradientTape (symgrad/tensor.py):
select_rows (gather), mul (conj fold, distribution.py:267-269), reduce_max over each
output's records in first-derivation order (tensor.py:319-325, gradient to the first
maximal entry), concat, clamp(0, 1) (tensor.py:275-287).  Output symbols and record
lists come from the reference's own apply_if run on a DAMP context (the same
map/shuffle), so the symbol order is the reference's.

    python tools/make_golden_max.py
"""

from __future__ import annotations

import json
import sys
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

import golden_cases as G  # noqa: E402

OUT = ROOT / "tests" / "golden"


class RDist:
    """A distribution whose tag is a reference Tensor (B, n) on the reference tape."""

    def __init__(self, ctx, symbols, tag):
        self.ctx, self.symbols, self.tag = ctx, tuple(symbols), tag

    def __len__(self):
        return len(self.symbols)

    @property
    def batch(self):
        return self.tag.shape[0]

    def filter(self, pred):
        keep = [i for i, s in enumerate(self.symbols) if pred(s)]
        return RDist(self.ctx, [self.symbols[i] for i in keep], T.select_rows(self.tag, keep, axis=1))


class RCtx:
    def __init__(self):
        self.tape = T.GradientTape()
        self.damp = S.ProgramContext(S.provenance_from_name("damp"))  # symbol order only


def _records(f, cond, dists):
    """Output symbols (reference order, checked) and each output's records (combos in
    enumeration order) from the reference's own map/shuffle."""
    import itertools

    shadow = [S.make_distribution(d.ctx.damp, np.ones((1, len(d))), list(d.symbols)) for d in dists]
    ref = S.apply_if(f, cond, *shadow)
    out_syms = list(ref.symbols)
    pos = {s: i for i, s in enumerate(out_syms)}
    recs = [[] for _ in out_syms]
    for combo in itertools.product(*[range(len(d)) for d in dists]):
        args = [d.symbols[i] for d, i in zip(dists, combo)]
        if cond is not None and not cond(*args):
            continue
        y = f(*args)
        if y is S.UNDEFINED or y is RAPI.UNDEFINED:
            continue
        recs[pos[y]].append(combo)
    return out_syms, recs


def _max_col(t, cols):
    return T.reshape(T.reduce_max(T.select_rows(t, cols, axis=1), axis=1), (t.shape[0], 1))


def _bcast(t, B):
    return t if t.shape[0] == B else T.mul(t, T.Tensor(np.ones((B, t.shape[1]))))


class RAPI:
    from paper_2410_03348_b200.plan import UNDEFINED

    @staticmethod
    def apply_if(f, cond, *dists):
        ctx = dists[0].ctx
        B = max(d.batch for d in dists)
        if any(len(d) == 0 for d in dists):
            return RDist(ctx, (), T.Tensor(np.zeros((B, 0))))
        fr = lambda *a: S.UNDEFINED if f(*a) is RAPI.UNDEFINED else f(*a)  # noqa: E731
        syms, recs = _records(fr, cond, dists)
        if not syms:
            return RDist(ctx, (), T.Tensor(np.zeros((B, 0))))
        flat = [c for r in recs for c in r]
        prod = None
        for i, d in enumerate(dists):
            g = _bcast(T.select_rows(d.tag, [c[i] for c in flat], axis=1), B)
            prod = g if prod is None else T.mul(prod, g)
        parts, at = [], 0
        for r in recs:
            parts.append(_max_col(prod, list(range(at, at + len(r)))))
            at += len(r)
        return RDist(ctx, syms, T.clamp(T.concat(parts, axis=1), 0.0, 1.0))

    @staticmethod
    def apply(f, *dists):
        return RAPI.apply_if(f, None, *dists)

    @staticmethod
    def union(d1, d2):
        if len(d1) == 0:
            return d2
        if len(d2) == 0:
            return d1
        B = max(d1.batch, d2.batch)
        both = T.concat([_bcast(d1.tag, B), _bcast(d2.tag, B)], axis=1)
        symbols = list(d1.symbols)
        index = {s: i for i, s in enumerate(d1.symbols)}
        groups = [[i] for i in range(len(d1))]
        for j, s in enumerate(d2.symbols):
            p = index.get(s)
            if p is None:
                symbols.append(s)
                groups.append([len(d1) + j])
            else:
                groups[p].append(len(d1) + j)
        return RDist(d1.ctx, symbols, T.clamp(T.concat([_max_col(both, g) for g in groups], axis=1), 0.0, 1.0))


class RP:
    from paper_2410_03348_b200.programs import Coord

    @staticmethod
    def sum_n(ctx, d):
        from paper_2410_03348_b200.programs import _add

        res = d[0]
        for x in d[1:]:
            res = RAPI.apply(_add, res, x)
        return res

    @staticmethod
    def path_closure(ctx, edges):
        from paper_2410_03348_b200.programs import _ends_match, _join_ends

        derived = edges
        while True:
            new = RAPI.apply_if(_join_ends, _ends_match, derived, edges)
            merged = RAPI.union(derived, new)
            if set(merged.symbols) == set(derived.symbols):
                return merged
            derived = merged


def run_case(name):
    prov, k, prog, syms_fn, _, _ = G.CASES[name]
    assert prov == "max"
    inputs = G.case_inputs(name)
    ctx = RCtx()
    leaves = [ctx.tape.leaf(x) for x in inputs]
    dists = [RDist(ctx, s, lf) for lf, s in zip(leaves, syms_fn(RP))]
    out = prog(RAPI, RP, ctx, dists)
    w = G.loss_weights(name, out.tag.shape)
    loss = T.reduce_sum(T.reduce_sum(T.mul(out.tag, T.Tensor(w)), 1), 0)
    grads = ctx.tape.backward(loss)
    res = {"symbols": json.dumps([repr(s) for s in out.symbols]), "probs": out.tag.data.copy(), "w": w,
           "n_inputs": len(inputs)}
    for i, (x, lf) in enumerate(zip(inputs, leaves)):
        res[f"in{i}"] = x
        res[f"grad{i}"] = grads[lf].data.copy()
    return res


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    for name, case in G.CASES.items():
        if case[0] == "max":
            np.savez_compressed(OUT / f"{name}.npz", **{k: np.asarray(v) for k, v in run_case(name).items()})
            print("wrote", name)


if __name__ == "__main__":
    main()
