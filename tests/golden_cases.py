"""Golden workloads, written once against an abstract API so the SAME program runs on
the reference (tools/make_golden.py), on the CPU oracle (tests/test_oracle.py) and on
the CUDA path (tests/test_gpu_golden.py).

``api`` provides apply / apply_if / union / UNDEFINED; ``P`` provides sum_n / hwf /
path_closure with the reference signatures (programs.py:42-196).
"""

from __future__ import annotations

import numpy as np

DIGITS = list(range(10))
TOKENS = [str(d) for d in range(10)] + ["+", "-", "*", "/"]


def rows(rng, n, cols):
    r = rng.uniform(0.05, 1.0, size=(n, cols))
    r = r / r.sum(axis=1, keepdims=True)
    return r.astype(np.float32).astype(np.float64)


def _sum(api, P, ctx, d):
    return P.sum_n(ctx, d)


def _apply_sum(api, P, ctx, d):
    return api.apply(lambda *xs: sum(xs), *d)


def _apply_prod(api, P, ctx, d):
    return api.apply(lambda x, y: x * y, *d)


def _mod_cond(api, P, ctx, d):
    return api.apply_if(lambda x, y: api.UNDEFINED if (x + y) % 4 == 3 else (x * y) % 7, lambda x, y: x != y, *d)


def _mod3(api, P, ctx, d):
    return api.apply(lambda x, y, z: (x * y + z) % 5, *d)


def _relabel(api, P, ctx, d):
    return api.apply(lambda x: x % 3, *d)


def _bcast_reuse(api, P, ctx, d):
    x = api.apply(lambda u, v: u + v, d[0], d[1])
    return api.apply(lambda u, v: u * v, x, d[0])


def _union_filter(api, P, ctx, d):
    e = d[0].filter(lambda s: s % 2 == 0)
    return api.union(api.apply(lambda x: x * 2, e), d[1])


def _hwf(length):
    def prog(api, P, ctx, d):
        return P.hwf(ctx, d, length)

    return prog


def _path(api, P, ctx, d):
    return P.path_closure(ctx, d[0])


def _clutrr(api, P, ctx, d):
    """CLUTRR-style kinship closure (BASELINE config 4 pattern) written against the
    reference API: apply_if(kinship_compose, chain_link) + union to a fixpoint."""
    from paper_2410_03348_b200.programs import _chain_link, kinship_compose_with

    compose = kinship_compose_with(api.UNDEFINED)
    derived = facts = d[0]
    while True:
        new = api.apply_if(compose, _chain_link, derived, facts)
        merged = api.union(derived, new)
        if set(merged.symbols) == set(derived.symbols):
            return merged
        derived = merged


def clutrr_facts(n_entities, rels=None):
    from paper_2410_03348_b200.programs import KINSHIP_RELATIONS, Fact

    rels = KINSHIP_RELATIONS if rels is None else rels
    return [Fact(i, i + 1, r) for i in range(n_entities - 1) for r in rels]


def _sample(m, strategy, seed=None):
    """sum of two lists, then sample_symbols (distribution.py:309-342), then one more
    apply so the gather's backward is exercised through a downstream op."""

    def prog(api, P, ctx, d):
        out = api.apply(lambda x, y: x + y, d[0], d[1])
        kept = api.sample_symbols(out, m, seed=seed, strategy=strategy)
        return api.apply(lambda s: s % 5, kept)

    return prog


def _stack_parts(api, P, ctx, d):
    """Per-sample parts with DIFFERENT symbol sets (each a batch-1 apply of a part with
    itself), aligned by stack (distribution.py:345-369, placed/stack_parts
    provenance.py:264-271, :425-440), then a batched apply over the stacked result."""
    parts = [api.apply(lambda x, y: x + y, di, di) for di in d]
    out = api.stack(parts)
    return api.apply(lambda s: s // 2, out)


def _stack_inputs(n_parts, width):
    def make(rng):
        return [rows(rng, 1, width) for _ in range(n_parts)]

    return make


def _edges(seed, nodes, prob):
    rng = np.random.default_rng(seed)
    return [(i, j) for i in range(nodes) for j in range(nodes) if i != j and rng.uniform() < prob]


# name: (provenance, k, program, symbol-list builder, input builder)
def _digit_inputs(n, B):
    def make(rng):
        return [rows(rng, B, 10) for _ in range(n)]

    return make


def _sized_inputs(arity, size, B):
    def make(rng):
        return [rows(rng, B, size) for _ in range(arity)]

    return make


CASES = {
    "damp_sum2": ("damp", None, _sum, lambda P: [DIGITS] * 2, _digit_inputs(2, 16), 0),
    "damp_sum4": ("damp", None, _sum, lambda P: [DIGITS] * 4, _digit_inputs(4, 8), 1),
    "damp_sum15": ("damp", None, _sum, lambda P: [DIGITS] * 15, _digit_inputs(15, 4), 2),
    "damp_sweep_a2_s10": ("damp", None, _apply_sum, lambda P: [list(range(10))] * 2, _sized_inputs(2, 10, 16), 3),
    "damp_sweep_a2_s37": ("damp", None, _apply_sum, lambda P: [list(range(37))] * 2, _sized_inputs(2, 37, 8), 4),
    "damp_sweep_a3_s7": ("damp", None, _apply_sum, lambda P: [list(range(7))] * 3, _sized_inputs(3, 7, 8), 5),
    "damp_prod_a2_s10": ("damp", None, _apply_prod, lambda P: [list(range(10))] * 2, _sized_inputs(2, 10, 8), 6),
    "damp_mod_cond_a2": ("damp", None, _mod_cond, lambda P: [list(range(9))] * 2, _sized_inputs(2, 9, 8), 7),
    "damp_mod_a3": ("damp", None, _mod3, lambda P: [list(range(6))] * 3, _sized_inputs(3, 6, 8), 8),
    "damp_a1_relabel": ("damp", None, _relabel, lambda P: [list(range(12))], _sized_inputs(1, 12, 8), 9),
    "damp_bcast_reuse": ("damp", None, _bcast_reuse, lambda P: [list(range(5)), list(range(4))],
                         lambda rng: [rows(rng, 6, 5), rows(rng, 1, 4)], 10),
    "damp_union_filter": ("damp", None, _union_filter, lambda P: [list(range(6)), list(range(3, 8))],
                          lambda rng: [rows(rng, 8, 6), rows(rng, 8, 5)], 11),
    "dtkp_hwf3": ("dtkp", 3, _hwf(3), lambda P: [TOKENS] * 3, _sized_inputs(3, 14, 6), 12),
    "dtkp_hwf5": ("dtkp", 3, _hwf(5), lambda P: [TOKENS] * 5, _sized_inputs(5, 14, 3), 13),
    "dtkp_hwf3_k1": ("dtkp", 1, _hwf(3), lambda P: [TOKENS] * 3, _sized_inputs(3, 14, 4), 14),
    "dtkp_hwf3_k7": ("dtkp", 7, _hwf(3), lambda P: [TOKENS] * 3, _sized_inputs(3, 14, 4), 15),
    "dtkp_sum3_k2": ("dtkp", 2, _sum, lambda P: [DIGITS] * 3, _digit_inputs(3, 5), 16),
    "dtkp_sum4_k5": ("dtkp", 5, _sum, lambda P: [DIGITS] * 4, _digit_inputs(4, 3), 17),
    "dtkp_path_k3": ("dtkp", 3, _path, lambda P: [[P.Coord(*e) for e in _edges(20, 5, 0.45)]],
                     lambda rng: [rng.uniform(0.05, 0.95, size=(4, len(_edges(20, 5, 0.45)))).astype(np.float32)
                                  .astype(np.float64)], 18),
    "dtkp_path_k5": ("dtkp", 5, _path, lambda P: [[P.Coord(*e) for e in _edges(21, 5, 0.45)]],
                     lambda rng: [rng.uniform(0.05, 0.95, size=(4, len(_edges(21, 5, 0.45)))).astype(np.float32)
                                  .astype(np.float64)], 19),
    "dtkp_clutrr_k5": ("dtkp", 5, _clutrr, lambda P: [clutrr_facts(4)],
                       lambda rng: [rng.uniform(0.05, 0.95, size=(3, 60)).astype(np.float32).astype(np.float64)], 21),
    # BASELINE configs[2] / [3] at their full program shape (small batch: the reference
    # runs them in minutes): HWF-7 k=3 (8 applies, step 7 = 30712 x 10 -> 208767 symbols,
    # eval -> 8332) and the benchmarked CLUTRR closure, 5 entities x 20 relations, k=5
    "dtkp_hwf7": ("dtkp", 3, _hwf(7), lambda P: [TOKENS] * 7, _sized_inputs(7, 14, 4), 23),
    "dtkp_clutrr_e5_r20_k5": ("dtkp", 5, _clutrr, lambda P: [clutrr_facts(5)],
                              lambda rng: [rng.uniform(0.05, 0.95, size=(6, 80)).astype(np.float32)
                                           .astype(np.float64)], 24),
    "dtkp_clutrr_k3_e5": ("dtkp", 3, _clutrr, lambda P: [clutrr_facts(5, ("father", "mother", "son", "daughter",
                                                                          "brother", "sister", "husband", "wife"))],
                          lambda rng: [rng.uniform(0.05, 0.95, size=(2, 32)).astype(np.float32).astype(np.float64)], 22),
    # sample_symbols (top / seeded categorical) and stack over parts with different
    # symbol sets; the reference's own examples are test_distribution.py:329-392
    "damp_sample_top": ("damp", None, _sample(7, "top"), lambda P: [list(range(8)), list(range(6))],
                        lambda rng: [rows(rng, 6, 8), rows(rng, 6, 6)], 25),
    "damp_sample_cat": ("damp", None, _sample(5, "categorical", seed=7), lambda P: [list(range(8)), list(range(6))],
                        lambda rng: [rows(rng, 6, 8), rows(rng, 6, 6)], 26),
    "dtkp_sample_top_k3": ("dtkp", 3, _sample(6, "top"), lambda P: [list(range(7)), list(range(5))],
                           lambda rng: [rows(rng, 5, 7), rows(rng, 5, 5)], 27),
    "damp_stack": ("damp", None, _stack_parts, lambda P: [list(range(i, i + 3 + i % 2)) for i in range(4)],
                   lambda rng: [rows(rng, 1, 3 + i % 2) for i in range(4)], 28),
    "dtkp_stack_k3": ("dtkp", 3, _stack_parts, lambda P: [list(range(i, i + 3 + i % 2)) for i in range(4)],
                      lambda rng: [rows(rng, 1, 3 + i % 2) for i in range(4)], 29),
    # the max-product ("max/DAMP") variant: fixtures from the reference's Tensor primitives
    # (tools/make_golden_max.py), since the reference has no max provenance
    "max_sum2": ("max", None, _sum, lambda P: [DIGITS] * 2, _digit_inputs(2, 16), 30),
    "max_sum4": ("max", None, _sum, lambda P: [DIGITS] * 4, _digit_inputs(4, 8), 31),
    "max_mod_cond_a2": ("max", None, _mod_cond, lambda P: [list(range(9))] * 2, _sized_inputs(2, 9, 8), 32),
    "max_mod_a3": ("max", None, _mod3, lambda P: [list(range(6))] * 3, _sized_inputs(3, 6, 8), 33),
    "max_bcast_reuse": ("max", None, _bcast_reuse, lambda P: [list(range(5)), list(range(4))],
                        lambda rng: [rows(rng, 6, 5), rows(rng, 1, 4)], 34),
    "max_union_filter": ("max", None, _union_filter, lambda P: [list(range(6)), list(range(3, 8))],
                         lambda rng: [rows(rng, 8, 6), rows(rng, 8, 5)], 35),
    "max_path": ("max", None, _path, lambda P: [[P.Coord(*e) for e in _edges(23, 4, 0.5)]],
                 lambda rng: [rng.uniform(0.05, 0.9, size=(4, len(_edges(23, 4, 0.5)))).astype(np.float32)
                              .astype(np.float64)], 36),
    "damp_path": ("damp", None, _path, lambda P: [[P.Coord(*e) for e in _edges(22, 4, 0.5)]],
                  lambda rng: [rng.uniform(0.05, 0.5, size=(4, len(_edges(22, 4, 0.5)))).astype(np.float32)
                               .astype(np.float64)], 20),
}


def case_inputs(name):
    prov, k, prog, syms, make, seed = CASES[name]
    return make(np.random.default_rng(1000 + seed))


def loss_weights(name, shape):
    prov, k, prog, syms, make, seed = CASES[name]
    return np.random.default_rng(5000 + seed).uniform(-1.0, 1.0, size=shape)
