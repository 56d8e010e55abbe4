"""ORACLE — TEST INFRASTRUCTURE ONLY.  A float64 CPU mini-runtime of the reference API.

``OContext`` / ``ODist`` restate make_distribution / apply_if / filter / union /
get_probs (distribution.py:196-306) on top of oracle.algebra, with a tiny reverse sweep
for DAMP gradients (clamp pass-through, tensor.py:287) and the closed-form DTKP probs
gradient.  The program drivers below follow programs.py:42-196 and take the user symbol
functions (the workload definition) from the product's ``programs`` module, so both
sides evaluate exactly the same black-box functions.
"""

from __future__ import annotations

import numpy as np

from . import algebra as A


class OContext:
    def __init__(self, prov: str, k: int | None = None, undefined=None):
        if undefined is None:
            from paper_2410_03348_b200.plan import UNDEFINED as undefined  # the marker object only
        self.prov = prov
        self.k = k
        self.undefined = undefined
        self.blocks = []  # (B_i, n_i) float64 input probabilities
        self.width = 0
        self.nodes = []  # DAMP tape: (kind, payload)

    # --- registry
    def p(self):
        B = max(b.shape[0] for b in self.blocks)
        return np.concatenate([np.broadcast_to(b, (B, b.shape[1])) for b in self.blocks], axis=1)

    def _node(self, kind, payload, value):
        self.nodes.append((kind, payload, value))
        return len(self.nodes) - 1


class ODist:
    def __init__(self, ctx, symbols, tag, node=None):
        self.ctx = ctx
        self.symbols = tuple(symbols)
        self.tag = tag  # DAMP: (B, n) float64 ; DTKP: (member u8, present u8)
        self.node = node

    def __len__(self):
        return len(self.symbols)

    @property
    def batch(self):
        return self.tag.shape[0] if self.ctx.prov in ("damp", "max") else self.tag[0].shape[0]

    def filter(self, pred):
        keep = [i for i, s in enumerate(self.symbols) if pred(s)]
        syms = [self.symbols[i] for i in keep]
        if self.ctx.prov in ("damp", "max"):
            val = self.tag[:, keep]
            return ODist(self.ctx, syms, val, self.ctx._node("gather", (self.node, keep, self.tag.shape[1]), val))
        return ODist(self.ctx, syms, A.dtkp_gather(self.tag, keep))


def make_distribution(ctx: OContext, probs, symbols) -> ODist:
    probs = np.asarray(probs, dtype=np.float64)
    start = ctx.width
    ctx.blocks.append(probs)
    ctx.width += probs.shape[1]
    if ctx.prov in ("damp", "max"):
        return ODist(ctx, symbols, probs, ctx._node("input", len(ctx.blocks) - 1, probs))
    return ODist(ctx, symbols, A.dtkp_input_tags(start, probs.shape[1], ctx.width, probs.shape[0], ctx.k))


def _empty(ctx, batch):
    if ctx.prov in ("damp", "max"):
        v = np.zeros((batch, 0))
        return ODist(ctx, (), v, ctx._node("const", None, v))
    return ODist(ctx, (), (np.zeros((batch, 0, ctx.k, ctx.width), np.uint8), np.zeros((batch, 0, ctx.k), np.uint8)))


def apply_if(f, cond, *dists) -> ODist:
    ctx = dists[0].ctx
    batch = max(d.batch for d in dists)
    if any(len(d) == 0 for d in dists):
        return _empty(ctx, batch)
    syms, combos, out_idx = A.map_shuffle(f, cond, [d.symbols for d in dists], ctx.undefined)
    if len(out_idx) == 0:
        return _empty(ctx, batch)
    if ctx.prov == "damp":
        val = A.damp_apply([d.tag for d in dists], combos, out_idx, len(syms))
        node = ctx._node("apply", ([d.node for d in dists], combos, out_idx, [d.tag for d in dists]), val)
        return ODist(ctx, syms, val, node)
    if ctx.prov == "max":
        val, arg = A.max_apply([d.tag for d in dists], combos, out_idx, len(syms))
        node = ctx._node("apply_max", ([d.node for d in dists], combos, arg, [d.tag for d in dists]), val)
        return ODist(ctx, syms, val, node)
    tags = [A.pad_width(d.tag, ctx.width) for d in dists]
    return ODist(ctx, syms, A.dtkp_apply(tags, combos, out_idx, len(syms), ctx.p(), ctx.k))


def apply(f, *dists):
    return apply_if(f, None, *dists)


def union(d1: ODist, d2: ODist) -> ODist:
    ctx = d1.ctx
    if len(d1) == 0:
        return d2
    if len(d2) == 0:
        return d1
    symbols = list(d1.symbols)
    index = {s: i for i, s in enumerate(d1.symbols)}
    groups = [[i] for i in range(len(d1.symbols))]
    for j, s in enumerate(d2.symbols):
        pos = index.get(s)
        if pos is None:
            symbols.append(s)
            groups.append([len(d1.symbols) + j])
        else:
            groups[pos].append(len(d1.symbols) + j)
    if ctx.prov == "damp":
        n1 = len(d1.symbols)
        ia = [g[0] if g[0] < n1 else -1 for g in groups]
        ib = [(g[-1] - n1) if g[-1] >= n1 else -1 for g in groups]
        val = A.damp_union(d1.tag, d2.tag, ia, ib)
        return ODist(ctx, symbols, val, ctx._node("union", (d1.node, d2.node, ia, ib, d1.tag, d2.tag), val))
    if ctx.prov == "max":
        n1 = len(d1.symbols)
        ia = [g[0] if g[0] < n1 else -1 for g in groups]
        ib = [(g[-1] - n1) if g[-1] >= n1 else -1 for g in groups]
        val, which = A.max_union(d1.tag, d2.tag, ia, ib)
        return ODist(ctx, symbols, val,
                     ctx._node("union_max", (d1.node, d2.node, ia, ib, d1.tag, d2.tag, which), val))
    both = A.dtkp_concat([A.pad_width(d1.tag, ctx.width), A.pad_width(d2.tag, ctx.width)])
    return ODist(ctx, symbols, A.dtkp_group_disj(both, groups, ctx.p(), ctx.k))


def _encode_symbol(s) -> bytes:
    """distribution.py:64-86 (canonical byte encoding; sample_symbols tie-break only)."""
    import struct
    from fractions import Fraction

    if isinstance(s, bool):
        return b"b1" if s else b"b0"
    if isinstance(s, int):
        return b"i%d" % s
    if isinstance(s, Fraction):
        return b"q%d/%d" % (s.numerator, s.denominator)
    if isinstance(s, float):
        return b"f" + repr(s).encode()
    if isinstance(s, str):
        return b"s" + s.encode("utf-8")
    if s is None:
        return b"n"
    if isinstance(s, tuple):
        return b"t" + b"".join(struct.pack(">I", len(e)) + e for e in map(_encode_symbol, s))
    raise TypeError(type(s).__name__)


def _gather_cols(d: ODist, src, symbols) -> ODist:
    """Column gather with -1 = zero column: Damp/DtkpAm gather (provenance.py:233,
    :320-326) and placed (:264-268, :425-433)."""
    ctx = d.ctx
    src = np.asarray(src, dtype=np.int64)
    if ctx.prov in ("damp", "max"):
        val = np.where(src[None, :] >= 0, d.tag[:, np.maximum(src, 0)], 0.0)
        return ODist(ctx, symbols, val, ctx._node("placed", (d.node, src, d.tag.shape[1]), val))
    m, pr = A.pad_width(d.tag, ctx.width)
    om = np.where((src >= 0)[None, :, None, None], m[:, np.maximum(src, 0)], 0).astype(np.uint8)
    op = np.where((src >= 0)[None, :, None], pr[:, np.maximum(src, 0)], 0).astype(np.uint8)
    return ODist(ctx, symbols, (om, op))


def sample_symbols(d: ODist, m: int, seed=None, strategy="top") -> ODist:
    """distribution.py:309-342: keep m symbols by batch-mean probability (ties by the
    canonical encoding) or by a seeded categorical draw; original order is kept."""
    if m < 1:
        raise ValueError(m)
    if m >= len(d):
        return d
    mean = get_probs(d).mean(axis=0)
    n = len(d)
    if strategy == "top":
        keep = set(sorted(range(n), key=lambda i: (-mean[i], _encode_symbol(d.symbols[i])))[:m])
    else:
        total = mean.sum()
        w = mean / total if total > 0 else np.full(n, 1.0 / n)
        keep = set(np.random.default_rng(seed).choice(n, size=m, replace=False, p=w).tolist())
    idx = [i for i in range(n) if i in keep]
    return _gather_cols(d, idx, [d.symbols[i] for i in idx])


def stack(parts) -> ODist:
    """distribution.py:345-369: align symbol sets by first appearance (missing symbols get
    zero tags), then concatenate along the batch."""
    ctx = parts[0].ctx
    symbols, index = [], {}
    for part in parts:
        for s in part.symbols:
            if s not in index:
                index[s] = len(symbols)
                symbols.append(s)
    placed = []
    for part in parts:
        src = np.full(len(symbols), -1, dtype=np.int64)
        for i, s in enumerate(part.symbols):
            src[index[s]] = i
        placed.append(_gather_cols(part, src, symbols))
    if ctx.prov in ("damp", "max"):
        val = np.concatenate([p.tag for p in placed], axis=0)
        return ODist(ctx, symbols, val, ctx._node("stack", ([p.node for p in placed], [p.tag.shape[0] for p in placed]),
                                                  val))
    ms = [A.pad_width(p.tag, ctx.width) for p in placed]
    return ODist(ctx, symbols, (np.concatenate([m for m, _ in ms], axis=0), np.concatenate([r for _, r in ms], axis=0)))


def get_probs(d: ODist) -> np.ndarray:
    if d.ctx.prov in ("damp", "max"):
        return d.tag
    return A.dtkp_probs(A.pad_width(d.tag, d.ctx.width), d.ctx.p())


def grad_inputs(d: ODist, g: np.ndarray):
    """Gradient of sum(g * get_probs(d)) w.r.t. every registered input block."""
    ctx = d.ctx
    if ctx.prov == "dtkp":
        gp = A.dtkp_probs_grad(A.pad_width(d.tag, ctx.width), ctx.p(), g)
        out, col = [], 0
        for b in ctx.blocks:
            gb = gp[:, col: col + b.shape[1]]
            if b.shape[0] == 1 and gb.shape[0] > 1:
                gb = gb.sum(axis=0, keepdims=True)
            out.append(gb)
            col += b.shape[1]
        return out
    grads = {d.node: g}
    block_grads = [np.zeros_like(b) for b in ctx.blocks]
    for node in range(len(ctx.nodes) - 1, -1, -1):
        gn = grads.pop(node, None)
        if gn is None:
            continue
        kind, payload, _ = ctx.nodes[node]
        if kind == "input":
            gb = gn
            if ctx.blocks[payload].shape[0] == 1 and gb.shape[0] > 1:
                gb = gb.sum(axis=0, keepdims=True)
            block_grads[payload] = block_grads[payload] + gb
        elif kind == "apply":
            parents, combos, out_idx, vals = payload
            for parent, gi in zip(parents, A.damp_apply_grad(vals, combos, out_idx, gn)):
                grads[parent] = grads.get(parent, 0) + gi
        elif kind == "apply_max":
            parents, combos, arg, vals = payload
            for parent, gi in zip(parents, A.max_apply_grad(vals, combos, arg, gn)):
                grads[parent] = grads.get(parent, 0) + gi
        elif kind == "union_max":
            n1_node, n2_node, ia, ib, a, b, which = payload
            ga = np.zeros((gn.shape[0], a.shape[1]))
            gb = np.zeros((gn.shape[0], b.shape[1]))
            for r, (i, j) in enumerate(zip(ia, ib)):
                if i >= 0:
                    ga[:, i] += np.where(which[:, r] == 0, gn[:, r], 0.0)
                if j >= 0:
                    gb[:, j] += np.where(which[:, r] == 1, gn[:, r], 0.0)
            if a.shape[0] == 1 and ga.shape[0] > 1:
                ga = ga.sum(axis=0, keepdims=True)
            if b.shape[0] == 1 and gb.shape[0] > 1:
                gb = gb.sum(axis=0, keepdims=True)
            grads[n1_node] = grads.get(n1_node, 0) + ga
            grads[n2_node] = grads.get(n2_node, 0) + gb
        elif kind == "placed":
            parent, src, n = payload
            buf = np.zeros((gn.shape[0], n))
            keep = np.nonzero(src >= 0)[0]
            np.add.at(buf.T, src[keep], gn[:, keep].T)
            grads[parent] = grads.get(parent, 0) + buf
        elif kind == "stack":
            parents, sizes = payload
            off = 0
            for parent, bsz in zip(parents, sizes):
                grads[parent] = grads.get(parent, 0) + gn[off: off + bsz]
                off += bsz
        elif kind == "gather":
            parent, keep, n = payload
            buf = np.zeros((gn.shape[0], n))
            np.add.at(buf.T, keep, gn.T)
            grads[parent] = grads.get(parent, 0) + buf
        elif kind == "union":
            n1_node, n2_node, ia, ib, a, b = payload
            ga = np.zeros((gn.shape[0], a.shape[1]))
            gb = np.zeros((gn.shape[0], b.shape[1]))
            for r, (i, j) in enumerate(zip(ia, ib)):
                if i >= 0:
                    ga[:, i] += gn[:, r]
                if j >= 0:
                    gb[:, j] += gn[:, r]
            if a.shape[0] == 1 and ga.shape[0] > 1:
                ga = ga.sum(axis=0, keepdims=True)
            if b.shape[0] == 1 and gb.shape[0] > 1:
                gb = gb.sum(axis=0, keepdims=True)
            grads[n1_node] = grads.get(n1_node, 0) + ga
            grads[n2_node] = grads.get(n2_node, 0) + gb
    return block_grads


# ------------------------------------------------------------------ program drivers
def sum_n(dists):
    from paper_2410_03348_b200.programs import _add

    res = dists[0]
    for d in dists[1:]:
        res = apply(_add, res, d)
    return res


def product_n(dists):
    from paper_2410_03348_b200.programs import _mul

    res = dists[0]
    for d in dists[1:]:
        res = apply(_mul, res, d)
    return res


def hwf(ctx, slots, length):
    from paper_2410_03348_b200 import programs as P

    length = min(length, len(slots))
    b = slots[0].batch
    slots = list(slots)
    for i in range(length, len(slots)):
        slots[i] = make_distribution(ctx, np.ones((b, 1)), [P.PAD])
    for i in range(length):
        slots[i] = slots[i].filter(P._is_digit if i % 2 == 0 else P._is_operator)
    res = apply(P._singleton, slots[0])
    for slot in slots[1:]:
        res = apply(P._concat_symbol, res, slot)
    return apply(P._eval_chain, res)


def closure(derived, facts, f, cond):
    """path_closure / clutrr_closure fixpoint (programs.py:177-196)."""
    while True:
        new = apply_if(f, cond, derived, facts)
        merged = union(derived, new)
        if set(merged.symbols) == set(derived.symbols):
            return merged
        derived = merged
