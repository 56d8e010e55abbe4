"""CPU baseline leg: time the REFERENCE implementation (symgrad, from baseline/_ref) on a
bounded sample of a bench workload, on this host's cores.  Prints one JSON object.

Run as a subprocess by bench.py so OPENBLAS_NUM_THREADS is set before numpy loads:
    OPENBLAS_NUM_THREADS=<cores> python tools/ref_bench.py --workload sum15 --batch 1024
Falls back to the oracle port (oracle/, kind "port") when baseline/_ref is absent.
Timing follows the reference's own bench pattern (bench.py:41-53): one warm-up, then the
minimum of ``--repeats`` runs; forward = program + get_probs, backward = tape.backward.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def sum_chain_inputs(n, B, seed=0):
    rng = np.random.default_rng(seed)
    r = rng.uniform(0.05, 1.0, size=(n, B, 10))
    r = r / r.sum(axis=2, keepdims=True)
    return r.astype(np.float32).astype(np.float64)


def combos_sum_chain(n):
    return sum(10 * (9 * i + 1) for i in range(1, n))


def run_reference(workload, B, repeats):
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    import symgrad as S
    from symgrad import programs as SP
    from symgrad import tensor as T
    from symgrad.learn import loss_nll

    if workload == "sum15":
        n = 15
        xs = sum_chain_inputs(n, B)
        targets = np.random.default_rng(1).integers(0, 9 * n + 1, size=B)

        def once():
            ctx = S.ProgramContext(S.Damp())
            leaves = [ctx.tape.leaf(xs[i]) for i in range(n)]
            dists = [S.make_distribution(ctx, lf, list(range(10))) for lf in leaves]
            t0 = time.perf_counter()
            out = SP.sum_n(ctx, dists)
            probs = S.get_probs(out)
            loss = loss_nll(probs, [out.index_of(int(t)) for t in targets])
            t1 = time.perf_counter()
            ctx.tape.backward(loss)
            t2 = time.perf_counter()
            return t1 - t0, t2 - t1

        units = B * combos_sum_chain(n)
        return once, units, S.backend_name(), f"Sum-15 chain DAMP fwd+bwd, B={B} (reference symgrad)"
    raise ValueError(workload)


def run_port(workload, B, repeats):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle import programs as OP
    from paper_2410_03348_b200.plan import UNDEFINED

    n = 15
    xs = sum_chain_inputs(n, B)

    def once():
        ctx = OP.OContext("damp", None, undefined=UNDEFINED)
        dists = [OP.make_distribution(ctx, xs[i], list(range(10))) for i in range(n)]
        t0 = time.perf_counter()
        out = OP.sum_n(dists)
        probs = OP.get_probs(out)
        t1 = time.perf_counter()
        OP.grad_inputs(out, np.ones_like(probs))
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1

    return once, B * combos_sum_chain(n), "oracle-port", f"Sum-15 chain DAMP fwd+bwd, B={B} (oracle port)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="sum15")
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--port", action="store_true")
    args = ap.parse_args()
    kind = "reference"
    if args.port or not (ROOT / "baseline" / "_ref" / "symgrad").exists():
        once, units, backend, sample = run_port(args.workload, args.batch, args.repeats)
        kind = "port"
    else:
        once, units, backend, sample = run_reference(args.workload, args.batch, args.repeats)
    once()  # warm-up
    best = None
    fwd_best = bwd_best = None
    for _ in range(args.repeats):
        f, b = once()
        if best is None or f + b < best:
            best, fwd_best, bwd_best = f + b, f, b
    cores = len(os.sched_getaffinity(0))
    print(json.dumps({
        "value": units / best, "unit": "symbol-combos/s", "seconds_per_step": best, "fwd_s": fwd_best,
        "bwd_s": bwd_best, "cores": cores, "cpu_count": os.cpu_count(), "kind": kind, "backend": backend,
        "sample": sample, "batch": args.batch, "samples_per_s": args.batch / best,
        "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
    }))


if __name__ == "__main__":
    main()
