"""Reference CPU arm: time the REFERENCE implementation (``symgrad``, installed from
/root/reference into baseline/_ref by ``__graft_entry__.build()``) on a bench workload,
on this host's cores.  Prints one JSON object.

Every workload runs through the reference's own public API and stock code path
(``make_distribution`` / ``apply`` / programs / ``get_probs`` / ``learn.loss_nll`` /
``tape.backward``; compiled ``_dtkpcore`` backend).  The reference is single-threaded
numpy, so "all the host threads it can use" means what a user would do on a many-core
host: the batch — every sample is independent on this path — is split into equal
shards, one per worker process (fork), each running the unmodified reference on its
shard; a step is timed from dispatch until the last shard finished.  Timing follows the
reference's bench pattern (bench.py:41-53): warm-up steps, then timed steps.

    python tools/ref_bench.py --workload sum15 --batch 16384 --steps 3 --warmup 1

There is no silent substitution: a missing baseline/_ref is an error.  ``--port`` runs
the oracle restatement instead (kind "port") only when asked to.
"""

from __future__ import annotations

import argparse
import importlib.util
import json
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

_W = {}  # per-process workload state (inherited through fork)


def digit_rows(rng, n, B, cols=10):
    r = rng.uniform(0.05, 1.0, size=(n, B, cols))
    r = r / r.sum(axis=2, keepdims=True)
    return r.astype(np.float32).astype(np.float64)


def sum_chain_combos(n):
    return sum(10 * (9 * i + 1) for i in range(1, n))


HWF7_SIZES = [(10,), (10, 4), (40, 10), (283, 4), (1132, 10), (7678, 4), (30712, 10), (208767,)]


def _kinship():
    spec = importlib.util.spec_from_file_location("sg_kinship", ROOT / "paper_2410_03348_b200" / "kinship.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


# ----------------------------------------------------------------------------- workloads
def setup(workload, B, seed=0, arity=2, size=10):
    """-> (run(lo, hi) -> (fwd_s, bwd_s), units per full batch, unit, description).
    Inputs for the WHOLE batch are built once; a shard runs rows [lo, hi)."""
    if not (REF / "symgrad").exists():
        raise SystemExit(f"reference not installed at {REF} (run __graft_entry__.build() where /root/reference "
                         "exists); refusing to substitute another implementation")
    sys.path.insert(0, str(REF))
    import symgrad as S
    from symgrad import programs as SP
    from symgrad import tensor as T
    from symgrad.learn import Adam, Mlp, loss_nll

    rng = np.random.default_rng(seed)

    def nll_step(ctx, out, targets, lo, hi, t0):
        probs = S.get_probs(out)
        loss = loss_nll(probs, [out.find(t) for t in targets[lo:hi]])
        t1 = time.perf_counter()
        ctx.tape.backward(loss)
        return t1 - t0, time.perf_counter() - t1

    if workload in ("sum15", "sum2"):
        n = 15 if workload == "sum15" else 2
        xs = digit_rows(rng, n, B)
        targets = rng.integers(0, 9 * n + 1, size=B).tolist()

        def run(lo, hi):
            ctx = S.ProgramContext(S.Damp())
            leaves = [ctx.tape.leaf(xs[i, lo:hi]) for i in range(n)]
            t0 = time.perf_counter()
            dists = [S.make_distribution(ctx, lf, list(range(10))) for lf in leaves]
            out = SP.sum_n(ctx, dists)
            return nll_step(ctx, out, targets, lo, hi, t0)

        return run, B * sum_chain_combos(n), "symbol-combos/s", f"Sum-{n} chain DAMP fwd+loss+bwd"

    if workload in ("sum2train", "sum15train"):
        n = 2 if workload == "sum2train" else 15
        labels = rng.integers(0, 10, size=(n, B))
        centers = rng.normal(0.0, 1.0, size=(10, 784))
        feats = centers[labels] * (5.0 / np.sqrt(784)) + rng.normal(0.0, 1.0, size=(n, B, 784))
        targets = labels.sum(axis=0).tolist()

        def run(lo, hi):
            if ("mlp", lo) not in _W:  # one model + optimizer per shard, kept across steps
                _W[("mlp", lo)] = (Mlp(784, 128, 10, seed=0), Adam(1e-3))
            model, opt = _W[("mlp", lo)]
            ctx = S.ProgramContext(S.Damp())
            t0 = time.perf_counter()
            dists = [S.make_distribution(ctx, model.forward(ctx.tape, feats[i, lo:hi]), list(range(10)))
                     for i in range(n)]
            out = SP.sum_n(ctx, dists)
            probs = S.get_probs(out)
            loss = loss_nll(probs, [out.find(t) for t in targets[lo:hi]])
            t1 = time.perf_counter()
            grads = model.grad_arrays(ctx.tape.backward(loss))
            model.params = opt.step(model.params, grads)
            return t1 - t0, time.perf_counter() - t1

        return run, B, "train samples/s", f"Sum-{n} train step (reference Mlp 784-128-10 + DAMP + loss_nll + Adam)"

    if workload == "hwf7":
        xs = rng.uniform(0.05, 1.0, size=(7, B, 14))
        xs = (xs / xs.sum(axis=2, keepdims=True)).astype(np.float32).astype(np.float64)
        targets = None

        def run(lo, hi):
            ctx = S.ProgramContext(S.DtkpAm(3))
            leaves = [ctx.tape.leaf(xs[i, lo:hi]) for i in range(7)]
            t0 = time.perf_counter()
            dists = [S.make_distribution(ctx, lf, list(SP.TOKEN_ALPHABET)) for lf in leaves]
            out = SP.hwf(ctx, dists, 7)
            probs = S.get_probs(out)
            loss = loss_nll(probs, [i % len(out.symbols) for i in range(lo, hi)])
            t1 = time.perf_counter()
            ctx.tape.backward(loss)
            return t1 - t0, time.perf_counter() - t1

        combos = sum(int(np.prod(s)) for s in HWF7_SIZES)
        return run, B, "samples/s", f"HWF-7 DTKP k=3 fwd+loss+bwd ({combos} symbol combos per sample)"

    if workload == "clutrr":
        K = _kinship()
        facts = K.story_facts(5)
        compose = K.compose_with(S.UNDEFINED)
        x = rng.uniform(0.05, 0.95, size=(B, len(facts))).astype(np.float32).astype(np.float64)

        def run(lo, hi):
            ctx = S.ProgramContext(S.DtkpAm(5))
            leaf = ctx.tape.leaf(x[lo:hi])
            t0 = time.perf_counter()
            derived = d = S.make_distribution(ctx, leaf, facts)
            while True:
                merged = S.union(derived, S.apply_if(compose, K.chain_link, derived, d))
                if set(merged.symbols) == set(derived.symbols):
                    break
                derived = merged
            probs = S.get_probs(merged)
            loss = loss_nll(probs, [i % len(merged.symbols) for i in range(lo, hi)])
            t1 = time.perf_counter()
            ctx.tape.backward(loss)
            return t1 - t0, time.perf_counter() - t1

        return run, B, "samples/s", "CLUTRR-style closure, 5 entities x 20 relations, DTKP k=5, fwd+loss+bwd"

    if workload == "sweep":
        xs = digit_rows(rng, arity, B, size)
        n_out = arity * (size - 1) + 1
        w = rng.uniform(-1.0, 1.0, size=(B, n_out))
        f = (lambda a, b: a + b) if arity == 2 else (lambda a, b, c: a + b + c)

        def run(lo, hi):
            ctx = S.ProgramContext(S.Damp())
            leaves = [ctx.tape.leaf(xs[i, lo:hi]) for i in range(arity)]
            t0 = time.perf_counter()
            dists = [S.make_distribution(ctx, lf, list(range(size))) for lf in leaves]
            out = S.apply(f, *dists)
            loss = T.reduce_sum(T.reduce_sum(T.mul(S.get_probs(out), T.Tensor(w[lo:hi])), 1), 0)
            t1 = time.perf_counter()
            ctx.tape.backward(loss)
            return t1 - t0, time.perf_counter() - t1

        return run, B * size**arity, "symbol-combos/s", f"sweep apply f=sum arity {arity} |S|={size} fwd+bwd"
    raise SystemExit(f"unknown workload {workload!r}")


def setup_port(workload, B, seed=0, **_):
    """The oracle restatement (kind "port") for Sum-N only; run only with --port."""
    sys.path.insert(0, str(ROOT))
    from oracle import programs as OP
    from paper_2410_03348_b200.plan import UNDEFINED

    n = 15 if workload == "sum15" else 2
    xs = digit_rows(np.random.default_rng(seed), n, B)

    def run(lo, hi):
        ctx = OP.OContext("damp", None, undefined=UNDEFINED)
        t0 = time.perf_counter()
        dists = [OP.make_distribution(ctx, xs[i, lo:hi], list(range(10))) for i in range(n)]
        out = OP.sum_n(dists)
        probs = OP.get_probs(out)
        t1 = time.perf_counter()
        OP.grad_inputs(out, np.ones_like(probs))
        return t1 - t0, time.perf_counter() - t1

    return run, B * sum_chain_combos(n), "symbol-combos/s", f"Sum-{n} chain DAMP fwd+bwd (oracle port)"


def _shard(args):
    lo, hi = args
    return _W["run"](lo, hi)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="sum15")
    ap.add_argument("--batch", type=int, default=16384)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--procs", type=int, default=0, help="worker processes (0: one per available core, <= batch)")
    ap.add_argument("--arity", type=int, default=2)
    ap.add_argument("--size", type=int, default=10)
    ap.add_argument("--port", action="store_true", help="time the oracle restatement instead (explicit only)")
    args = ap.parse_args()

    cores = len(os.sched_getaffinity(0))
    procs = args.procs or cores
    procs = max(1, min(procs, args.batch))
    build = setup_port if args.port else setup
    run, units, unit, desc = build(args.workload, args.batch, arity=args.arity, size=args.size)
    _W["run"] = run
    base, extra = divmod(args.batch, procs)
    shards, lo = [], 0
    for r in range(procs):
        hi = lo + base + (1 if r < extra else 0)
        shards.append((lo, hi))
        lo = hi
    times = []
    if procs == 1:
        for i in range(args.warmup + args.steps):
            t = time.perf_counter()
            f, b = run(0, args.batch)
            if i >= args.warmup:
                times.append((time.perf_counter() - t, f, b))
    else:
        ctx = mp.get_context("fork")
        with ctx.Pool(procs) as pool:
            for i in range(args.warmup + args.steps):
                t = time.perf_counter()
                res = pool.map(_shard, shards, chunksize=1)
                wall = time.perf_counter() - t
                if i >= args.warmup:
                    times.append((wall, max(r[0] for r in res), max(r[1] for r in res)))
    walls = [t[0] for t in times]
    mean = float(np.mean(walls))
    backend = "oracle-port"
    if not args.port:
        import symgrad as S

        backend = S.backend_name()
    print(json.dumps({
        "value": units / mean, "unit": unit, "seconds_per_step": mean, "min_seconds_per_step": min(walls),
        "fwd_s": float(np.mean([t[1] for t in times])), "bwd_s": float(np.mean([t[2] for t in times])),
        "steps": args.steps, "warmup": args.warmup, "cores": procs, "cpu_count": os.cpu_count(),
        "affinity_cores": cores, "kind": "port" if args.port else "reference", "backend": backend,
        "batch": args.batch, "samples_per_s": args.batch / mean,
        "sample": f"{desc}, B={args.batch} split over {procs} processes "
                  f"({args.batch // procs}-{-(-args.batch // procs)} samples each), mean of {args.steps} steps "
                  f"after {args.warmup} warm-up",
        "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
    }))


if __name__ == "__main__":
    main()
