"""Measure every BASELINE.json config on one B200 (the headline line is bench.py's).

Each workload step (symbolic forward + loss + backward, and for the train configs the
LeNet perception forward/backward + Adam) is warmed up eagerly, captured in a CUDA graph
and replayed; time = CUDA events around ``--iters`` replays.  Prints one JSON object per
measurement (see DESIGN.md §Measurement for the unit definitions).

    python tools/bench_configs.py [--only sum2,hwf7,clutrr,sweep,sum15train,maxsweep]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2410_03348_b200 as sg  # noqa: E402
from paper_2410_03348_b200 import programs as P  # noqa: E402
from paper_2410_03348_b200.learn import LeNet, loss_nll  # noqa: E402

DEV = torch.device("cuda", 0)
HBM = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]


def timed(step, iters=20, graph=True):
    """ms per step: eager warm-up, CUDA-graph capture, replay timing (eager if capture fails)."""
    side = torch.cuda.Stream(DEV)
    side.wait_stream(torch.cuda.current_stream(DEV))
    with torch.cuda.stream(side):
        for _ in range(3):
            step()
    torch.cuda.current_stream(DEV).wait_stream(side)
    torch.cuda.synchronize(DEV)
    mode = "eager"
    g = None
    if graph:
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                step()
            g.replay()
            torch.cuda.synchronize(DEV)
            mode = "cuda_graph"
        except Exception as exc:  # noqa: BLE001 - report and fall back to eager timing
            import traceback

            traceback.print_exc(limit=15)
            g = None
            mode = f"eager (capture failed: {type(exc).__name__}: {str(exc)[:160]})"
            torch.cuda.synchronize(DEV)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        if g is not None:
            g.replay()
        else:
            step()
    e1.record()
    torch.cuda.synchronize(DEV)
    return e0.elapsed_time(e1) / iters, mode


def rows(rng, B, n):
    r = rng.uniform(0.05, 1.0, size=(B, n))
    return (r / r.sum(axis=1, keepdims=True)).astype(np.float32)


def emit(d):
    print(json.dumps(d), flush=True)


# ------------------------------------------------------------------ configs 1 / 2: training
def train_sum(n_digits, B, iters, label):
    """LeNet perception in bf16 autocast + channels_last (cuDNN autotuned); the softmax
    outputs and the whole symbolic path are fp32."""
    torch.manual_seed(0)
    torch.backends.cudnn.benchmark = True
    model = LeNet(10).to(DEV).to(memory_format=torch.channels_last)
    opt = torch.optim.Adam(model.parameters(), lr=1e-3, capturable=True)
    rng = np.random.default_rng(0)
    imgs = torch.tensor(rng.normal(size=(n_digits * B, 1, 28, 28)).astype(np.float32), device=DEV)
    imgs = imgs.to(memory_format=torch.channels_last)
    targets = torch.tensor(rng.integers(0, 9 * n_digits + 1, size=B), device=DEV)

    def step():
        opt.zero_grad(set_to_none=False)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            probs = model(imgs).float().view(n_digits, B, 10)
        ctx = sg.ProgramContext(sg.Damp(), device=DEV)
        out = P.sum_n(ctx, [sg.make_distribution(ctx, probs[i], range(10)) for i in range(n_digits)])
        loss = loss_nll(sg.get_probs(out), targets)
        loss.backward()
        opt.step()
        return loss

    ms, mode = timed(step, iters)
    emit({"config": label, "metric": "train samples/s", "value": B / (ms * 1e-3), "ms_per_step": ms, "batch": B,
          "mode": mode, "perception": "LeNet-5 (synthetic 28x28), bf16 autocast + channels_last",
          "optimizer": "Adam", "symbolic_dtype": "f32"})


# ------------------------------------------------------------------ config 3: HWF-7 DTKP k=3
def hwf7(B, iters):
    rng = np.random.default_rng(1)
    xs = [torch.tensor(rows(rng, B, 14), device=DEV, requires_grad=True) for _ in range(7)]
    t0 = time.perf_counter()
    ctx = sg.ProgramContext(sg.DtkpAm(3), device=DEV)
    out = P.hwf(ctx, [sg.make_distribution(ctx, x, P.TOKEN_ALPHABET) for x in xs], 7)
    torch.cuda.synchronize(DEV)
    first = time.perf_counter() - t0
    n_out = len(out)
    del out, ctx  # drop the first call's autograd graph (its AccumulateGrad nodes live on the default stream)
    targets = torch.tensor(rng.integers(0, n_out, size=B), device=DEV)
    combos = 0
    from paper_2410_03348_b200.plan import plan_cache_info

    def step():
        c = sg.ProgramContext(sg.DtkpAm(3), device=DEV)
        o = P.hwf(c, [sg.make_distribution(c, x, P.TOKEN_ALPHABET) for x in xs], 7)
        loss = loss_nll(sg.get_probs(o), targets)
        return torch.autograd.grad(loss, xs)

    ms, mode = timed(step, iters)
    sizes = [(10,), (10, 4), (40, 10), (283, 4), (1132, 10), (7678, 4), (30712, 10), (208767,)]
    combos = sum(int(np.prod(s)) for s in sizes)
    emit({"config": "HWF-7 DTKP k=3 (BASELINE configs[2])", "metric": "samples/s (symbolic fwd+bwd)",
          "value": B / (ms * 1e-3), "ms_per_step": ms, "batch": B, "mode": mode, "output_symbols": n_out,
          "symbol_combos_per_s": B * combos / (ms * 1e-3), "first_call_s_incl_host_plans": first,
          "plan_cache": plan_cache_info()})


# ------------------------------------------------------------------ config 4: CLUTRR-style
def clutrr(B, iters, n_entities=5, k=5):
    sys.path.insert(0, str(ROOT / "tests"))
    from golden_cases import clutrr_facts

    rng = np.random.default_rng(2)
    facts = clutrr_facts(n_entities)
    x = torch.tensor(rng.uniform(0.05, 0.95, size=(B, len(facts))).astype(np.float32), device=DEV,
                     requires_grad=True)
    t0 = time.perf_counter()
    ctx = sg.ProgramContext(sg.DtkpAm(k), device=DEV)
    out = P.clutrr_closure(ctx, sg.make_distribution(ctx, x, facts))
    torch.cuda.synchronize(DEV)
    first = time.perf_counter() - t0
    targets = torch.tensor(rng.integers(0, len(out), size=B), device=DEV)
    n_derived = len(out)
    del out, ctx

    def step():
        c = sg.ProgramContext(sg.DtkpAm(k), device=DEV)
        o = P.clutrr_closure(c, sg.make_distribution(c, x, facts))
        loss = loss_nll(sg.get_probs(o), targets)
        return torch.autograd.grad(loss, [x])

    ms, mode = timed(step, iters)
    emit({"config": f"CLUTRR-style kinship closure, {n_entities} entities x 20 relations, DTKP k={k} "
                    "(BASELINE configs[3])", "metric": "samples/s (symbolic fwd+bwd)", "value": B / (ms * 1e-3),
          "ms_per_step": ms, "batch": B, "mode": mode, "derived_facts": n_derived, "input_facts": len(facts),
          "first_call_s_incl_host_plans": first})


# ------------------------------------------------------------------ config 5: sweep
def sweep(iters):
    for arity, size in [(2, 10), (2, 100), (2, 1000), (3, 10), (3, 30), (3, 100)]:
        for B in (1024, 16384, 65536):
            if arity == 3 and size == 100 and B > 16384:
                continue
            rng = np.random.default_rng(size + B)
            xs = [torch.tensor(rows(rng, B, size), device=DEV, requires_grad=True) for _ in range(arity)]
            syms = list(range(size))
            f = (lambda a, b: a + b) if arity == 2 else (lambda a, b, c: a + b + c)
            n_out = arity * (size - 1) + 1
            w = torch.tensor(rng.uniform(-1, 1, size=(B, n_out)).astype(np.float32), device=DEV)

            def fwd():
                c = sg.ProgramContext(sg.Damp(), device=DEV)
                return sg.get_probs(sg.apply(f, *[sg.make_distribution(c, x, syms) for x in xs]))

            def step():  # d(sum probs * w)/dx: the upstream gradient w goes straight in
                return torch.autograd.grad(fwd(), xs, grad_outputs=w)

            ms_f, mode = timed(lambda: fwd(), iters)
            ms, _ = timed(step, iters)
            C = size ** arity
            fb = 4 * B * (arity * size + n_out) + 4 * C
            bb = 4 * B * (n_out + 2 * arity * size) + 4 * C
            kp = sg.plan.build_plan(f, None, [tuple(syms)] * arity).kernel_plan()
            emit({"config": f"sweep arity {arity} |S|={size} f=sum B={B} (BASELINE configs[4])",
                  "path": "toeplitz" if kp.conv else "generic segmented", "batch": B,
                  "fwd_ms": ms_f, "fwd_bwd_ms": ms, "combos_per_s_fwd": B * C / (ms_f * 1e-3),
                  "combos_per_s_fwd_bwd": B * C / (ms * 1e-3),
                  "fwd_algorithmic_gbs": fb / (ms_f * 1e-3) / 1e9, "fwd_hbm_frac": fb / (ms_f * 1e-3) / 1e9 / HBM,
                  "fwd_bwd_algorithmic_gbs": (fb + bb) / (ms * 1e-3) / 1e9,
                  "fwd_bwd_hbm_frac": (fb + bb) / (ms * 1e-3) / 1e9 / HBM, "mode": mode})
            del xs, w
            torch.cuda.empty_cache()


# ------------------------------------------------------------------ max-product variant
def maxsweep(iters):
    """The max/DAMP variant (sg_maxprod_*) on sweep shapes and the Sum-15 chain."""
    cases = [(2, 10, 16384), (2, 10, 65536), (2, 100, 16384), (3, 10, 16384)]
    for arity, size, B in cases:
        rng = np.random.default_rng(7 * size + B)
        xs = [torch.tensor(rows(rng, B, size), device=DEV, requires_grad=True) for _ in range(arity)]
        syms = list(range(size))
        f = (lambda a, b: a + b) if arity == 2 else (lambda a, b, c: a + b + c)
        n_out = arity * (size - 1) + 1
        w = torch.tensor(rng.uniform(-1, 1, size=(B, n_out)).astype(np.float32), device=DEV)

        def fwd():
            c = sg.ProgramContext(sg.DampMax(), device=DEV)
            return sg.get_probs(sg.apply(f, *[sg.make_distribution(c, x, syms) for x in xs]))

        def step():
            return torch.autograd.grad(fwd(), xs, grad_outputs=w)

        ms_f, mode = timed(lambda: fwd(), iters)
        ms, _ = timed(step, iters)
        C = size ** arity
        fb = 4 * B * (arity * size + 2 * n_out)           # inputs + probs + argmax
        bb = 4 * B * (2 * n_out + 2 * arity * size)       # g + argmax + inputs + grads
        emit({"config": f"max variant: sweep arity {arity} |S|={size} f=sum B={B}", "batch": B,
              "fwd_ms": ms_f, "fwd_bwd_ms": ms, "combos_per_s_fwd": B * C / (ms_f * 1e-3),
              "combos_per_s_fwd_bwd": B * C / (ms * 1e-3),
              "fwd_hbm_frac": fb / (ms_f * 1e-3) / 1e9 / HBM, "fwd_bwd_hbm_frac": (fb + bb) / (ms * 1e-3) / 1e9 / HBM,
              "mode": mode})
        del xs, w
        torch.cuda.empty_cache()
    B = 16384
    rng = np.random.default_rng(15)
    xs = [torch.tensor(rows(rng, B, 10), device=DEV, requires_grad=True) for _ in range(15)]
    targets = torch.tensor(rng.integers(0, 136, size=B), device=DEV)

    def step15():
        c = sg.ProgramContext(sg.DampMax(), device=DEV)
        o = P.sum_n(c, [sg.make_distribution(c, x, list(range(10))) for x in xs])
        return torch.autograd.grad(loss_nll(sg.get_probs(o), targets), xs)

    ms, mode = timed(step15, iters)
    emit({"config": "max variant: Sum-15 chain B=16384 (14 max-product applies) + loss, fwd+bwd",
          "ms_per_step": ms, "combos_per_s": B * 9590 / (ms * 1e-3), "mode": mode})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="sum2,sum15train,hwf7,clutrr,sweep,maxsweep")
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    torch.cuda.set_device(DEV)
    only = set(args.only.split(","))
    if "sum2" in only:
        train_sum(2, 64, args.iters, "MNIST Sum-2 train, B=64, LeNet + DAMP (BASELINE configs[0])")
    if "sum15train" in only:
        train_sum(15, 16384, max(3, args.iters // 4), "MNIST Sum-15 train, B=16384, LeNet + DAMP (BASELINE configs[1])")
    if "hwf7" in only:
        hwf7(64, args.iters)
    if "clutrr" in only:
        clutrr(4096, args.iters)
    if "sweep" in only:
        sweep(args.iters)
    if "maxsweep" in only:
        maxsweep(args.iters)


if __name__ == "__main__":
    main()
