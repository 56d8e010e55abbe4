"""Per-config measurements for bench.py's ``configs`` key (BASELINE.json configs[0], [2],
[3], [4]; configs[1] is bench.py's headline) — also runnable on its own:

    python tools/bench_configs.py [--only sum2,hwf7,clutrr,sweep,maxsweep] [--no-cpu]

For every config, on one B200:
  device     the step (symbolic forward + loss + backward; for Sum-2 also the LeNet
             perception forward/backward and Adam) captured in a CUDA graph, replayed
             ``iters`` times with L2 flushed (512 MB write) before each replay; CUDA events
             on the launching stream around each replay.
  e2e        the same step through the public API, eager, with the step's inputs copied
             H2D from pinned host memory and the loss read back D2H every step.
  roofline   the step's algorithmic HBM bytes (ops.ALG_BYTES ledger: SURVEY §8(d)
             formulas evaluated per launch — inputs read once, outputs written once) /
             the device step time, vs MEASURED_PEAKS.json hbm_gbs; per-kernel shares.
  cpu        the reference symgrad (baseline/_ref) on the same config, batch split over
             the host's cores (tools/ref_bench.py), same run.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2410_03348_b200 as sg  # noqa: E402
from paper_2410_03348_b200 import ops  # noqa: E402
from paper_2410_03348_b200 import programs as P  # noqa: E402
from paper_2410_03348_b200.learn import LeNet, loss_nll  # noqa: E402

HWF7_SIZES = [(10,), (10, 4), (40, 10), (283, 4), (1132, 10), (7678, 4), (30712, 10), (208767,)]


def hbm_peak():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]), "measured"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback"


class Flusher:
    def __init__(self, dev):
        self.buf = torch.empty(512 * 1024 * 1024 // 4, device=dev, dtype=torch.float32)

    def __call__(self):
        self.buf.zero_()


def graph_time(step, dev, iters, flush):
    """ms per step of ``step`` captured in a CUDA graph, L2 flushed before every replay
    (outside the events).  Falls back to eager replays if capture fails (reported)."""
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side):
        for _ in range(3):
            step()
    torch.cuda.current_stream(dev).wait_stream(side)
    torch.cuda.synchronize(dev)
    mode, g = "cuda_graph", None
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, capture_error_mode="thread_local"):
            step()
        g.replay()
        torch.cuda.synchronize(dev)
    except Exception as exc:  # noqa: BLE001 - reported in the line
        g = None
        mode = f"eager (capture failed: {type(exc).__name__}: {str(exc)[:120]})"
        torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for a, b in ev:
        flush()
        a.record()
        if g is not None:
            g.replay()
        else:
            step()
        b.record()
    torch.cuda.synchronize(dev)
    return sum(a.elapsed_time(b) for a, b in ev) / iters, mode


def ledger(step):
    """Algorithmic bytes / work units of one eager step, per kernel."""
    ops.ALG_BYTES = []
    try:
        step()
        torch.cuda.synchronize()
        rec = ops.ALG_BYTES
    finally:
        ops.ALG_BYTES = None
    by = {}
    for k, nbytes, units in rec:
        e = by.setdefault(k, {"launches": 0, "bytes": 0, "units": 0})
        e["launches"] += 1
        e["bytes"] += nbytes
        e["units"] += units
    return sum(e["bytes"] for e in by.values()), by


def e2e_time(step_host, dev, iters):
    """ms per step of the eager public-API step fed from pinned host memory, the loss read
    back every step (host wall clock around ``iters`` steps after 2 warm-ups)."""
    for _ in range(2):
        step_host()
    torch.cuda.synchronize(dev)
    t = time.perf_counter()
    for _ in range(iters):
        step_host()
    torch.cuda.synchronize(dev)
    return (time.perf_counter() - t) * 1e3 / iters


def graphed_e2e(step_fn, dev_inputs, host_inputs, dev, iters):
    """ms per step through the public GraphedStep API with host buffers: each step copies
    its inputs H2D from pinned memory into the capture (one arena copy), replays the graph
    and reads the loss (output 0) back to the host."""
    from paper_2410_03348_b200.graph import GraphedStep

    g = GraphedStep(step_fn, dev_inputs)
    views = g.pinned_inputs(0)
    for v, h in zip(views, host_inputs):
        v.copy_(h)

    res = {}

    def once():
        out = g(*views)
        r = out[0] if isinstance(out, (tuple, list)) else out
        if r.numel() == 1:
            return float(r.detach())
        if "host" not in res:  # the step's (B, n) result goes back to the host
            res["host"] = torch.empty(r.shape, dtype=r.dtype).pin_memory()
        res["host"].copy_(r.detach(), non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        return None

    for _ in range(2):
        once()
    torch.cuda.synchronize(dev)
    t = time.perf_counter()
    for _ in range(iters):
        once()
    torch.cuda.synchronize(dev)
    ms = (time.perf_counter() - t) * 1e3 / iters
    del g
    return ms


def e2e_entry(graphed_ms, eager_ms, units, h2d, d2h, what):
    return {"ms_per_step": graphed_ms, "value": units / (graphed_ms * 1e-3), "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h,
            "api": f"GraphedStep (public API): {what}; inputs H2D from pinned host memory + graph replay + loss "
                   "read back every step",
            "eager": {"ms_per_step": eager_ms, "value": units / (eager_ms * 1e-3),
                      "api": "the same step through the eager API calls, inputs H2D + loss.item() every step"}}


def cpu_reference(workload, batch, steps=1, warmup=0, procs=0, **kw):
    env = dict(os.environ)
    env["OPENBLAS_NUM_THREADS"] = "1"
    cmd = [sys.executable, str(ROOT / "tools" / "ref_bench.py"), "--workload", workload, "--batch", str(batch),
           "--steps", str(steps), "--warmup", str(warmup), "--procs", str(procs)]
    for k, v in kw.items():
        cmd += [f"--{k}", str(v)]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600)
        if out.returncode != 0:
            return {"value": None, "error": out.stderr[-400:]}
        r = json.loads(out.stdout.strip().splitlines()[-1])
        return {k: r[k] for k in ("value", "unit", "seconds_per_step", "cores", "kind", "backend", "sample")}
    except Exception as exc:  # noqa: BLE001 - reported, not fatal
        return {"value": None, "error": str(exc)[:300]}


def roofline(alg_bytes, by_kernel, ms, hbm, peak_src):
    gbs = alg_bytes / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "alg_bytes_per_step": alg_bytes, "achieved_gbs": gbs, "peak": hbm, "unit": "GB/s",
            "frac": gbs / hbm, "peak_source": peak_src, "by_kernel": by_kernel,
            "method": "sum of per-launch algorithmic bytes (ops.ALG_BYTES, SURVEY 8(d) formulas) / graph-replayed "
                      "step time with L2 flushed"}


def issue_ceiling(prefix):
    """The DTKP kernels' issue-ceiling fractions from the committed ncu --set full captures
    (profiles/issue.json, tools/ncu_issue.py): the apply is instruction-issue bound
    (SURVEY 8(d)), so its roofline is the SM issue rate, 4 warp-instructions/cycle/SM."""
    try:
        d = json.loads((ROOT / "profiles" / "issue.json").read_text())
    except (OSError, ValueError):
        return None
    ent = {k: v for k, v in d.items() if k.startswith(prefix)}
    if not ent:
        return None
    top = max(ent.values(), key=lambda v: v["duration_us"])
    return {"bound": "issue", "kernel": top["kernel"], "frac": top["issue_active_frac"],
            "ipc_per_sm": top["ipc_per_sm"], "peak_ipc_per_sm": top["ipc_peak"],
            "fp64_pipe_frac": top["fp64_pipe_frac"], "source": "profiles/issue.json (ncu --set full)",
            "kernels": ent}


def rows(rng, B, n):
    r = rng.uniform(0.05, 1.0, size=(B, n))
    return (r / r.sum(axis=1, keepdims=True)).astype(np.float32)


# ------------------------------------------------------------------ configs[0]: Sum-2 train
def sum2_train(dev, iters=20, cpu=True, B=64):
    """LeNet (bf16 autocast, channels_last) on synthetic 28x28 digits -> 2 softmax blocks ->
    apply(+) (DAMP) -> loss_nll -> backward -> Adam.  The reference arm trains its own Mlp
    (it has no convolution primitive)."""
    torch.manual_seed(0)
    torch.backends.cudnn.benchmark = True
    model = LeNet(10).to(dev).to(memory_format=torch.channels_last)
    opt = torch.optim.Adam(model.parameters(), lr=1e-3, capturable=True)
    rng = np.random.default_rng(0)
    labels = rng.integers(0, 10, size=(2, B))
    centers = rng.normal(size=(10, 28 * 28))
    imgs_h = (centers[labels] * (5.0 / 28) + rng.normal(size=(2, B, 28 * 28))).astype(np.float32)
    imgs_h = torch.tensor(imgs_h.reshape(2 * B, 1, 28, 28))
    tgt_h = torch.tensor(labels.sum(axis=0))
    imgs = imgs_h.to(dev).to(memory_format=torch.channels_last)
    targets = tgt_h.to(dev)

    def step_on(x, t):
        opt.zero_grad(set_to_none=False)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            probs = model(x).float().view(2, B, 10)
        ctx = sg.ProgramContext(sg.Damp(), device=dev)
        out = P.sum_n(ctx, [sg.make_distribution(ctx, probs[i], range(10)) for i in range(2)])
        loss = loss_nll(sg.get_probs(out), t)
        loss.backward()
        opt.step()
        return loss

    flush = Flusher(dev)
    ms, mode = graph_time(lambda: step_on(imgs, targets), dev, iters, flush)
    alg, by = ledger(lambda: step_on(imgs, targets))
    pin_x, pin_t = imgs_h.pin_memory(), tgt_h.pin_memory()

    def host_step():
        x = pin_x.to(dev, non_blocking=True).to(memory_format=torch.channels_last)
        loss = step_on(x, pin_t.to(dev, non_blocking=True))
        return loss.item()

    e2e_ms = e2e_time(host_step, dev, iters)
    g_ms = graphed_e2e(lambda x, t: step_on(x, t), [imgs, targets], [imgs_h.to(memory_format=torch.channels_last),
                                                                     tgt_h], dev, iters)
    hbm, src = hbm_peak()
    res = {"config": "MNIST Sum-2 train: synthetic 28x28 digits, random-init LeNet, DAMP, B=64 (BASELINE configs[0])",
           "metric": "train samples/s", "batch": B,
           "device": {"ms_per_step": ms, "value": B / (ms * 1e-3), "mode": mode},
           "e2e": e2e_entry(g_ms, e2e_ms, B, pin_x.numel() * 4 + B * 8, 8,
                            "LeNet -> make_distribution -> sum_n -> get_probs -> loss_nll -> backward -> Adam"),
           "roofline": roofline(alg, by, ms, hbm, src) | {"note": "symbolic kernels only; the step is launch-bound "
                                                                  "(LeNet + Adam dominate)"}}
    if cpu:
        res["cpu"] = cpu_reference("sum2train", B, steps=10, warmup=2, procs=1)
    return res


# ------------------------------------------------------------------ configs[2]: HWF-7
def hwf7(dev, iters=20, cpu=True, B=64):
    rng = np.random.default_rng(1)
    xs_h = torch.tensor(np.stack([rows(rng, B, 14) for _ in range(7)]))
    xs = [xs_h[i].to(dev).requires_grad_(True) for i in range(7)]
    t0 = time.perf_counter()
    ctx = sg.ProgramContext(sg.DtkpAm(3), device=dev)
    out = P.hwf(ctx, [sg.make_distribution(ctx, x, P.TOKEN_ALPHABET) for x in xs], 7)
    torch.cuda.synchronize(dev)
    first = time.perf_counter() - t0
    n_out = len(out)
    del out, ctx
    tgt_h = torch.tensor(rng.integers(0, n_out, size=B))
    targets = tgt_h.to(dev)

    def step_on(xl, t):
        c = sg.ProgramContext(sg.DtkpAm(3), device=dev)
        o = P.hwf(c, [sg.make_distribution(c, x, P.TOKEN_ALPHABET) for x in xl], 7)
        loss = loss_nll(sg.get_probs(o), t)
        return loss, torch.autograd.grad(loss, xl)

    flush = Flusher(dev)
    ms, mode = graph_time(lambda: step_on(xs, targets), dev, iters, flush)
    alg, by = ledger(lambda: step_on(xs, targets))
    pin_x, pin_t = xs_h.pin_memory(), tgt_h.pin_memory()

    def host_step():
        xd = pin_x.to(dev, non_blocking=True)
        loss, _ = step_on([xd[i].requires_grad_(True) for i in range(7)], pin_t.to(dev, non_blocking=True))
        return loss.item()

    e2e_ms = e2e_time(host_step, dev, max(3, iters // 2))
    g_ms = graphed_e2e(lambda *a: step_on(list(a[:7]), a[7]), xs + [targets], [xs_h[i] for i in range(7)] + [tgt_h],
                       dev, iters)
    hbm, src = hbm_peak()
    combos = sum(int(np.prod(s)) for s in HWF7_SIZES)
    cand = by.get("dtkp_apply", {}).get("units", 0)
    res = {"config": "HWF-7 formula eval, DTKP k=3, B=64 (BASELINE configs[2])", "metric": "samples/s (symbolic "
           "fwd+loss+bwd)", "batch": B, "output_symbols": n_out,
           "device": {"ms_per_step": ms, "value": B / (ms * 1e-3), "symbol_combos_per_s": B * combos / (ms * 1e-3),
                      "candidate_rows_per_s": cand / (ms * 1e-3), "mode": mode},
           "e2e": e2e_entry(g_ms, e2e_ms, B, pin_x.numel() * 4 + B * 8, 8,
                            "programs.hwf (memoised plans) + loss_nll + autograd.grad"),
           "first_call_s_incl_host_plans": first,
           "roofline": roofline(alg, by, ms, hbm, src), "issue_ceiling": issue_ceiling("hwf7_")}
    if cpu:
        res["cpu"] = cpu_reference("hwf7", B, steps=1, warmup=0)
    return res


# ------------------------------------------------------------------ configs[3]: CLUTRR-style
def clutrr(dev, iters=20, cpu=True, B=4096, n_entities=5, k=5):
    from paper_2410_03348_b200.kinship import story_facts

    rng = np.random.default_rng(2)
    facts = story_facts(n_entities)
    x_h = torch.tensor(rng.uniform(0.05, 0.95, size=(B, len(facts))).astype(np.float32))
    x = x_h.to(dev).requires_grad_(True)
    ctx = sg.ProgramContext(sg.DtkpAm(k), device=dev)
    out = P.clutrr_closure(ctx, sg.make_distribution(ctx, x, facts))
    n_derived = len(out)
    del out, ctx
    tgt_h = torch.tensor(rng.integers(0, n_derived, size=B))
    targets = tgt_h.to(dev)

    def step_on(xv, t):
        c = sg.ProgramContext(sg.DtkpAm(k), device=dev)
        o = P.clutrr_closure(c, sg.make_distribution(c, xv, facts))
        loss = loss_nll(sg.get_probs(o), t)
        return loss, torch.autograd.grad(loss, [xv])

    flush = Flusher(dev)
    ms, mode = graph_time(lambda: step_on(x, targets), dev, iters, flush)
    alg, by = ledger(lambda: step_on(x, targets))
    pin_x, pin_t = x_h.pin_memory(), tgt_h.pin_memory()

    def host_step():
        loss, _ = step_on(pin_x.to(dev, non_blocking=True).requires_grad_(True), pin_t.to(dev, non_blocking=True))
        return loss.item()

    e2e_ms = e2e_time(host_step, dev, iters)
    g_ms = graphed_e2e(lambda xv, t: step_on(xv, t), [x, targets], [x_h, tgt_h], dev, iters)
    hbm, src = hbm_peak()
    cand = by.get("dtkp_apply", {}).get("units", 0)
    res = {"config": f"CLUTRR-style kinship closure, {n_entities} entities x 20 relations, DTKP k={k}, B={B} "
                     "(BASELINE configs[3])", "metric": "samples/s (symbolic fwd+loss+bwd)", "batch": B,
           "derived_facts": n_derived,
           "device": {"ms_per_step": ms, "value": B / (ms * 1e-3), "candidate_rows_per_s": cand / (ms * 1e-3),
                      "mode": mode},
           "e2e": e2e_entry(g_ms, e2e_ms, B, pin_x.numel() * 4 + B * 8, 8,
                            "clutrr_closure (fixpoint.closure) + loss_nll + autograd.grad"),
           "roofline": roofline(alg, by, ms, hbm, src), "issue_ceiling": issue_ceiling("clutrr_")}
    if cpu:
        res["cpu"] = cpu_reference("clutrr", B, steps=1, warmup=0)
    return res


# ------------------------------------------------------------------ configs[4]: sweep
SWEEP = [(2, 10, 65536), (2, 10, 16384), (2, 100, 16384), (2, 1000, 16384), (3, 10, 16384), (3, 100, 16384)]
# reference sample batch (and worker processes) per sweep point; the reference's dense
# group_disj matrix G (provenance.py:248-251) is C x N_out fp64 per apply: 2.4 GB at arity
# 3 |S|=100 (few processes), 16 GB at arity 2 |S|=1000 (infeasible)
SWEEP_CPU_BATCH = {(2, 10): (16384, 0), (2, 100): (2048, 0), (3, 10): (2048, 0), (3, 100): (16, 4)}
SWEEP_CPU_INFEASIBLE = {(2, 1000): "reference dense G = 1e6 x 1999 fp64 = 16 GB per apply (provenance.py:248-251)"}


def sweep_point(dev, arity, size, B, iters=20, cpu=True, provenance="damp"):
    rng = np.random.default_rng(size + B)
    xs_h = torch.tensor(np.stack([rows(rng, B, size) for _ in range(arity)]))
    xs = [xs_h[i].to(dev).requires_grad_(True) for i in range(arity)]
    syms = list(range(size))
    f = (lambda a, b: a + b) if arity == 2 else (lambda a, b, c: a + b + c)
    n_out = arity * (size - 1) + 1
    w_h = torch.tensor(rng.uniform(-1, 1, size=(B, n_out)).astype(np.float32))
    w = w_h.to(dev)
    prov = sg.Damp if provenance == "damp" else sg.DampMax

    def step_on(xl, wv):  # d(sum probs * w)/dx: the upstream gradient w goes straight in
        c = sg.ProgramContext(prov(), device=dev)
        p = sg.get_probs(sg.apply(f, *[sg.make_distribution(c, x, syms) for x in xl]))
        return p, torch.autograd.grad(p, xl, grad_outputs=wv)

    def fwd_only():
        c = sg.ProgramContext(prov(), device=dev)
        return sg.get_probs(sg.apply(f, *[sg.make_distribution(c, x.detach(), syms) for x in xs]))

    flush = Flusher(dev)
    ms_f, mode = graph_time(fwd_only, dev, iters, flush)
    ms, _ = graph_time(lambda: step_on(xs, w), dev, iters, flush)
    alg, by = ledger(lambda: step_on(xs, w))
    alg_f, _ = ledger(fwd_only)
    pin_x, pin_w = xs_h.pin_memory(), w_h.pin_memory()
    out_h = torch.empty((B, n_out), dtype=torch.float32).pin_memory()

    def host_step():
        xd = pin_x.to(dev, non_blocking=True)
        p, _ = step_on([xd[i].requires_grad_(True) for i in range(arity)], pin_w.to(dev, non_blocking=True))
        out_h.copy_(p.detach(), non_blocking=True)  # the step's result back to the host
        torch.cuda.current_stream(dev).synchronize()

    e2e_ms = e2e_time(host_step, dev, iters)
    g_ms = graphed_e2e(lambda *a: step_on(list(a[:arity]), a[arity]), xs + [w], [xs_h[i] for i in range(arity)] + [w_h],
                       dev, iters)
    C = size ** arity
    kp = sg.plan.build_plan(f, None, [tuple(syms)] * arity).kernel_plan()
    hbm, src = hbm_peak()
    res = {"config": f"sweep arity {arity} |S|={size} f=sum B={B} ({provenance}, BASELINE configs[4])",
           "metric": "symbol-combos/s (fwd+bwd)", "batch": B, "path": "toeplitz" if kp.conv else "generic segmented",
           "bound": "hbm" if (arity, size) == (2, 10) else "issue/FMA (SURVEY 8(d): >= 4 combos/byte)",
           "device": {"ms_per_step": ms, "value": B * C / (ms * 1e-3), "fwd_ms": ms_f,
                      "fwd_combos_per_s": B * C / (ms_f * 1e-3), "mode": mode,
                      "fwd_hbm_frac": alg_f / (ms_f * 1e-3) / 1e9 / hbm},
           "e2e": e2e_entry(g_ms, e2e_ms, B * C, pin_x.numel() * 4 + pin_w.numel() * 4, out_h.numel() * 4,
                            "make_distribution/apply/get_probs + autograd.grad(grad_outputs=w), probs D2H"),
           "roofline": roofline(alg, by, ms, hbm, src)}
    if cpu and provenance == "damp":
        cb = SWEEP_CPU_BATCH.get((arity, size))
        if cb:
            res["cpu"] = cpu_reference("sweep", cb[0], steps=2, warmup=1, procs=cb[1], arity=arity, size=size)
        elif (arity, size) in SWEEP_CPU_INFEASIBLE:
            res["cpu"] = {"value": None, "infeasible": SWEEP_CPU_INFEASIBLE[(arity, size)]}
    del xs, w
    torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------------ max/DAMP variant, Sum-15
def max_sum15(dev, iters=20, B=16384):
    """The north star's max/DAMP variant on the headline shape: Sum-15 chain under DampMax
    (fused sg_maxchain_fwd/bwd) + loss_nll, fwd + bwd, B=16384."""
    rng = np.random.default_rng(15)
    xs_h = torch.tensor(np.stack([rows(rng, B, 10) for _ in range(15)]))
    xs = [xs_h[i].to(dev).requires_grad_(True) for i in range(15)]
    tgt_h = torch.tensor(rng.integers(0, 136, size=B))
    targets = tgt_h.to(dev)

    def step_on(xl, t):
        c = sg.ProgramContext(sg.DampMax(), device=dev)
        o = P.sum_n(c, [sg.make_distribution(c, x, list(range(10))) for x in xl])
        loss = loss_nll(sg.get_probs(o), t)
        return loss, torch.autograd.grad(loss, xl)

    flush = Flusher(dev)
    ms, mode = graph_time(lambda: step_on(xs, targets), dev, iters, flush)
    alg, by = ledger(lambda: step_on(xs, targets))
    pin_x, pin_t = xs_h.pin_memory(), tgt_h.pin_memory()

    def host_step():
        xd = pin_x.to(dev, non_blocking=True)
        loss, _ = step_on([xd[i].requires_grad_(True) for i in range(15)], pin_t.to(dev, non_blocking=True))
        return loss.item()

    e2e_ms = e2e_time(host_step, dev, iters)
    g_ms = graphed_e2e(lambda *a: step_on(list(a[:15]), a[15]), xs + [targets], [xs_h[i] for i in range(15)] + [tgt_h],
                       dev, iters)
    hbm, src = hbm_peak()
    return {"config": "max/DAMP variant: Sum-15 chain (14 max-product applies) + loss_nll, fwd+bwd, B=16384",
            "metric": "symbol-combos/s", "batch": B,
            "device": {"ms_per_step": ms, "value": B * 9590 / (ms * 1e-3), "mode": mode},
            "e2e": e2e_entry(g_ms, e2e_ms, B * 9590, pin_x.numel() * 4 + B * 8, 8,
                             "sum_n under DampMax + loss_nll + autograd.grad"),
            "roofline": roofline(alg, by, ms, hbm, src)}


def all_configs(dev, iters=20, cpu=True, only=("sum2", "hwf7", "clutrr", "sweep", "max15")):
    out = {}
    if "sum2" in only:
        out["sum2_train"] = sum2_train(dev, iters, cpu)
    if "hwf7" in only:
        out["hwf7"] = hwf7(dev, iters, cpu)
    if "clutrr" in only:
        out["clutrr"] = clutrr(dev, iters, cpu)
    if "sweep" in only:
        for a, s, b in SWEEP:
            out[f"sweep_a{a}_s{s}_b{b}"] = sweep_point(dev, a, s, b, iters, cpu)
    if "max15" in only:
        out["max_sum15"] = max_sum15(dev, iters)
    if "maxsweep" in only:
        for a, s, b in [(2, 10, 65536), (2, 100, 16384), (3, 10, 16384)]:
            out[f"max_sweep_a{a}_s{s}_b{b}"] = sweep_point(dev, a, s, b, iters, False, provenance="max")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="sum2,hwf7,clutrr,sweep,max15")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    res = all_configs(dev, args.iters, not args.no_cpu, tuple(args.only.split(",")))
    for k, v in res.items():
        print(json.dumps({"key": k, **v}), flush=True)


if __name__ == "__main__":
    main()
