"""CPU: the host map/shuffle stage (plan builder) and the device work-list layout.

The plan must be bit-exact with the reference's apply_if host part
(distribution.py:244-260) — checked against the oracle restatement and the golden
symbol orders — and the segmented work lists must cover every record exactly once.
"""

import numpy as np
import pytest

import golden_cases as G
from runners import load_golden


def plan_mod():
    from paper_2410_03348_b200 import plan

    return plan


def test_plan_matches_oracle_map_shuffle():
    P = plan_mod()
    from oracle.algebra import map_shuffle

    cases = [
        (lambda x, y: x + y, None, [tuple(range(10))] * 2),
        (lambda x, y: P.UNDEFINED if (x * y) % 5 == 3 else (x - y) % 4, lambda x, y: x != y, [tuple(range(9)), tuple(range(7))]),
        (lambda x, y, z: (x, y % 2, z > 1), None, [tuple("abc"), tuple(range(4)), tuple(range(3))]),
        (lambda s: s % 2, None, [(3, 1, 2, 0)]),
    ]
    for f, cond, lists in cases:
        plan = P.build_plan(f, cond, lists)
        syms, combos, idx = map_shuffle(f, cond, lists, P.UNDEFINED)
        assert plan.out_symbols == syms
        np.testing.assert_array_equal(plan.combos, combos)
        np.testing.assert_array_equal(plan.out_idx, idx)
    assert P.build_plan(lambda s: s % 2, None, [(3, 1, 2, 0)]).out_symbols == (1, 0)  # first derivation


@pytest.mark.parametrize("name", [n for n in G.CASES if n.startswith("damp_sum") or n.startswith("damp_sweep")])
def test_plan_output_order_matches_reference_golden(name):
    P = plan_mod()
    from paper_2410_03348_b200 import programs as PR

    gold = load_golden(name)
    prov, k, prog, syms_fn, _, _ = G.CASES[name]
    lists = syms_fn(PR)
    if name.startswith("damp_sum"):
        res = tuple(lists[0])
        for s in lists[1:]:
            res = P.build_plan(PR._add, None, [res, tuple(s)]).out_symbols
        got = res
    else:
        got = P.build_plan(lambda *xs: sum(xs), None, [tuple(s) for s in lists]).out_symbols
    assert [repr(s) for s in got] == gold["symbols"]


def test_table_and_undefined():
    P = plan_mod()
    plan = P.build_plan(lambda x, y: P.UNDEFINED if x == y else x * y, None, [tuple(range(3))] * 2)
    t = plan.table.reshape(3, 3)
    assert (np.diag(t) == -1).all()
    assert t[1, 2] == plan.out_symbols.index(2)
    assert plan.n_kept == 6 and plan.n_enumerated == 9


def test_symbol_function_errors_carry_the_tuple():
    P = plan_mod()
    with pytest.raises(P.SymbolFunctionError) as err:
        P.build_plan(lambda x, y: x / y, None, [(0, 1), (0, 1)])
    assert err.value.symbols == (0, 0)


def test_memo_hits_same_code_and_closure():
    P = plan_mod()
    P.plan_cache_clear()

    def make(k):
        return lambda x, y: (x + y) % k

    lists = [tuple(range(5))] * 2
    a = P.build_plan(make(3), None, lists)
    b = P.build_plan(make(3), None, [tuple(range(5)), tuple(range(5))])
    c = P.build_plan(make(4), None, lists)
    assert a is b and a is not c
    info = P.plan_cache_info()
    assert info["hits"] == 1 and info["misses"] == 2
    # typed symbol keys: 1 and 1.0 are different input lists
    d = P.build_plan(lambda x: type(x).__name__, None, [(1, 2)])
    e = P.build_plan(lambda x: type(x).__name__, None, [(1.0, 2.0)])
    assert d.out_symbols == ("int",) and e.out_symbols == ("float",)


def test_plan_outputs_are_canonical_for_chaining():
    P = plan_mod()
    from paper_2410_03348_b200.programs import _add

    p1 = P.build_plan(_add, None, [tuple(range(10))] * 2)
    p2 = P.build_plan(_add, None, [p1.out_symbols, tuple(range(10))])
    p2b = P.build_plan(_add, None, [p1.out_symbols, tuple(range(10))])
    assert p2 is p2b
    assert P.canonical_symbols(p1.out_symbols) is p1.out_symbols


def test_toeplitz_detection():
    P = plan_mod()
    kp = P.build_plan(lambda x, y: x + y, None, [tuple(range(30)), tuple(range(10))]).kernel_plan()
    assert kp.conv and kp.conv_short == 1
    kp = P.build_plan(lambda x, y: x + y, None, [tuple(range(4)), tuple(range(30))]).kernel_plan()
    assert kp.conv and kp.conv_short == 0
    assert not P.build_plan(lambda x, y: x * y, None, [tuple(range(4))] * 2).kernel_plan().conv
    assert P.build_plan(lambda x, y: x + y, None, [tuple(range(40))] * 2).kernel_plan().conv == 2  # both long
    assert not P.build_plan(lambda x, y: x + y, None, [(0, 2, 1), (0, 1)]).kernel_plan().conv  # not index-additive


@pytest.mark.parametrize("max_item", [1, 3, 128])
def test_segsum_items_cover_every_record_once(max_item):
    P = plan_mod()
    rng = np.random.default_rng(max_item)
    n_seg = 50
    lens = rng.integers(0, 400, size=n_seg)
    lens[3] = 0
    off = np.concatenate([[0], np.cumsum(lens)])
    recs = rng.integers(0, 1000, size=(off[-1], 3)).astype(np.int32)
    h = P.HostSegsum(off, recs, max_item)
    vals = rng.uniform(size=off[-1])
    out = np.full(n_seg, np.nan)
    partial = np.zeros(h.n_partial)
    seen = np.zeros(off[-1], dtype=int)
    for seg, rb, re, dest in h.items:
        seen[rb:re] += 1
        v = vals[rb:re].sum()
        if dest < 0:
            out[seg] = v
        else:
            partial[dest] = v
    for seg, pb, pe in h.split:
        out[seg] = partial[pb:pe].sum()
    assert (seen == 1).all()
    ref = np.array([vals[off[i]:off[i + 1]].sum() for i in range(n_seg)])
    np.testing.assert_allclose(out, ref)
    for nb in (1, 2, 7, 64):
        blk = h.blocks(nb)
        assert blk[0] == 0 and blk[-1] == len(h.items) and (np.diff(blk) >= 0).all()


# ------------------------------------------------------------------ native host planner
def _plans_equal(a, b):
    assert a.out_symbols == b.out_symbols
    assert [type(s) for s in a.out_symbols] == [type(s) for s in b.out_symbols]
    np.testing.assert_array_equal(a.combos, b.combos)
    np.testing.assert_array_equal(a.out_idx, b.out_idx)
    assert a.n_enumerated == b.n_enumerated


@pytest.mark.parametrize("case", range(7))
def test_native_planner_equals_interpreted_loop(case):
    """csrc/planner.cpp (the product path) against the interpreted restatement of
    distribution.py:244-260: same symbols (and their types), combos, output order."""
    P = plan_mod()
    f, cond, lists = [
        (lambda x, y: x + y, None, [tuple(range(10))] * 2),
        (lambda x, y: P.UNDEFINED if (x * y) % 5 == 3 else (x - y) % 4, lambda x, y: x != y,
         [tuple(range(9)), tuple(range(7))]),
        (lambda x, y, z: (x, y % 2, z > 1), None, [tuple("abc"), tuple(range(4)), tuple(range(3))]),
        # 1 == 1.0 == True collide in the bucket dict: the first derivation's object wins
        (lambda x: [1, 1.0, True, 2, 2.0][x], None, [tuple(range(5))]),
        (lambda x, y: x, None, [(), (1, 2)]),            # an empty input list: nothing enumerated
        (lambda: 7, None, []),                            # arity 0: one empty combination
        (lambda x, y: P.UNDEFINED, lambda x, y: x < y, [tuple(range(4))] * 2),  # everything dropped
    ][case]
    canon = [P.canonical_symbols(tuple(s)) for s in lists]
    _plans_equal(P._map_shuffle(f, cond, canon), P._map_shuffle_py(f, cond, canon))


def test_native_planner_errors():
    P = plan_mod()

    def bad(x, y):
        if (x, y) == (2, 1):
            raise ZeroDivisionError("boom")
        return x

    with pytest.raises(P.SymbolFunctionError) as ei:
        P._map_shuffle(bad, None, [tuple(range(3)), tuple(range(3))])
    assert ei.value.symbols == (2, 1)
    assert isinstance(ei.value.__cause__, ZeroDivisionError)
    with pytest.raises(P.SymbolFunctionError) as ei:  # cond errors are wrapped the same way
        P._map_shuffle(lambda x: x, lambda x: 1 / (x - 1), [tuple(range(3))])
    assert ei.value.symbols == (1,)
    with pytest.raises(TypeError):  # an unhashable result fails in the bucket dict, unwrapped
        P._map_shuffle(lambda x: [x], None, [tuple(range(2))])


def test_fused_dtkp_host_plan_keeps_intermediates_whole():
    """The fused conj -> group_disj work list (sg_dtkp_apply_desc.inner_arity): per output
    segment, the conj records of its intermediate symbols in (segment ordinal, conj
    ordinal) order, bit 31 on each intermediate's last record, items of whole
    intermediates, split segments listed for the merge pass."""
    import numpy as np

    from paper_2410_03348_b200 import programs as P
    from paper_2410_03348_b200.plan import build_plan

    d = tuple(P.DIGIT_TOKENS)
    o = tuple(P.OPERATOR_TOKENS)
    s1 = build_plan(P._singleton, None, [d])
    s2 = build_plan(P._concat_symbol, None, [s1.out_symbols, o])
    s3 = build_plan(P._concat_symbol, None, [s2.out_symbols, d])  # the binary apply (inner)
    ev = build_plan(P._eval_chain, None, [s3.out_symbols])          # the arity-1 apply (outer)
    inner, outer = s3.kernel_plan(), ev.kernel_plan()
    h = outer.dtkp_fused_host(inner)
    ih = inner.dtkp_host()
    flat = h.recs[:, :2].view(np.uint32).astype(np.int64)
    last = (flat[:, 1] >> 31) == 1
    rows = np.stack([flat[:, 0], flat[:, 1] & 0x7FFFFFFF], axis=1)
    # expected sequence, straight from the two plans
    exp, exp_last = [], []
    for seg in range(outer.n_out):
        for mid in outer.records[outer.out_idx == seg, 0]:
            a, b = ih.seg_off[mid], ih.seg_off[mid + 1]
            exp.extend((ih.recs[a:b, :2].astype(np.int64) & 0x7FFFFFFF).tolist())
            exp_last.extend([False] * (b - a - 1) + [True])
    np.testing.assert_array_equal(rows, np.asarray(exp))
    np.testing.assert_array_equal(last, np.asarray(exp_last))
    for seg, rb, re, dest in h.items:
        assert rb == re or last[re - 1]               # items end on an intermediate boundary
        assert rb == h.seg_off[seg] or last[rb - 1]  # ... and start on one
    split = np.bincount(h.items[:, 0], minlength=h.n_seg) > 1
    assert h.n_partial == int(split[h.items[:, 0]].sum()) == int((h.items[:, 3] >= 0).sum())


def test_packed_dtkp_items_cover_every_segment_once():
    """Packed DTKP work lists (sg_dtkp_apply_desc.seg_packed): items are runs of whole
    short segments (bit 31 on each segment's last record) or pieces of split long ones;
    every record is covered once, every segment is closed exactly once."""
    import numpy as np

    from paper_2410_03348_b200.plan import HostSegsum

    rng = np.random.default_rng(0)
    lens = rng.choice([0, 1, 1, 2, 3, 5, 47, 48, 49, 130], size=400)
    off = np.concatenate([[0], np.cumsum(lens)])
    recs = rng.integers(0, 1000, size=(int(off[-1]), 2)).astype(np.int32)
    h = HostSegsum(off, recs, 48, pack=40)
    assert h.packed
    flags = h.recs[:, 0] < 0
    np.testing.assert_array_equal(h.recs[:, 0] & 0x7FFFFFFF, recs[:, 0])
    np.testing.assert_array_equal(np.nonzero(flags)[0], off[1:][lens > 0] - 1)
    from paper_2410_03348_b200.plan import dtkp_pack_size

    assert dtkp_pack_size(307120, 64) == 43 and dtkp_pack_size(2000, 4096) == 18 and dtkp_pack_size(100, 4096) == 0
    covered = np.zeros(len(recs), dtype=int)
    closed = np.zeros(len(lens), dtype=int)
    for seg, rb, re, dest in h.items:
        covered[rb:re] += 1
        assert re - rb <= 48
        assert re - rb <= 40 or dest >= 0 or lens[seg] == re - rb  # packed run, split piece or one whole segment
        if dest < 0:
            assert rb == off[seg]
            if rb == re:
                closed[seg] += 1
            else:
                closed[seg: seg + int(flags[rb:re].sum())] += 1
                assert flags[re - 1]
        else:
            assert lens[seg] > 48
    for sp_seg, pb, pe in h.split:
        closed[sp_seg] += 1
        assert pe - pb == -(-lens[sp_seg] // 48)
    assert (covered == 1).all() and (closed == 1).all()
