"""Host map/shuffle stage of ``apply_if`` and the memoised device plans it feeds.

``build_plan`` restates ``apply_if``'s host part (distribution.py:244-260): the
symbol function runs once per combination of input symbols, in ``itertools.product``
order (last input fastest), ``cond`` before ``f``, ``UNDEFINED`` dropped, and output
symbols numbered in first-derivation order.  The result is an int32 combination ->
output-symbol table plus CSR views of it; it is memoised on the function's code and
closure and on the identity of the input symbol lists, so a training loop calls the
black-box function only once per distinct plan (sum_n builds a new lambda per fold step,
programs.py:48, which this keying recognises as the same function).

``KernelPlan`` turns (records, output index) pairs into the device work lists consumed by
the CUDA library: a forward segmented problem (segments = outputs), one backward
problem per input (segments = that input's positions), and the Toeplitz flag for tables
with T[s0][s1] == s0 + s1.
"""

from __future__ import annotations

import os

import itertools
from collections import OrderedDict

import numpy as np
import torch

from . import _native as N

__all__ = [
    "UNDEFINED",
    "SymbolFunctionError",
    "SymbolPlan",
    "KernelPlan",
    "build_plan",
    "plan_cache_clear",
    "plan_cache_info",
    "canonical_symbols",
]


class _Undefined:
    """Marker a mapping function returns for combinations with no result."""

    __slots__ = ()

    def __repr__(self):
        return "UNDEFINED"

    def __reduce__(self):
        return (_undefined_singleton, ())


def _undefined_singleton():
    return UNDEFINED


UNDEFINED = _Undefined()


class SymbolFunctionError(RuntimeError):
    """A user-supplied symbol function raised; carries the offending tuple."""

    def __init__(self, message, symbols):
        super().__init__(message)
        self.symbols = symbols


def call_user(fn, syms):
    """distribution.py:179-185: wrap user errors with the offending symbol tuple."""
    try:
        return fn(*syms)
    except Exception as exc:  # noqa: BLE001 - re-raised with context
        raise SymbolFunctionError(f"symbol function failed on {syms!r}: {exc}", syms) from exc


# ----------------------------------------------------------------------------- keys
def _typed(s):
    # 1, 1.0, True and Fraction(1) compare equal but may map differently under f
    if isinstance(s, tuple):
        return (type(s), tuple(_typed(x) for x in s))
    return (type(s), s)


class _SymbolIntern:
    """Canonical symbol-tuple objects so plan keys are cheap identity lookups.

    Plan outputs are canonical by construction; user-made lists are interned by a
    type-aware value key (bounded LRU)."""

    def __init__(self, limit=8192, large_limit=256):
        self.by_id = {}  # id(tuple) -> tuple (holds a reference so ids stay unique)
        self.by_value = OrderedDict()
        self.large = OrderedDict()  # id -> tuple for lists too long for a value key (LRU)
        self.limit = limit
        self.large_limit = large_limit

    def canon(self, symbols: tuple) -> tuple:
        hit = self.by_id.get(id(symbols))
        if hit is symbols:
            if id(symbols) in self.large:
                self.large.move_to_end(id(symbols))
            return symbols
        key = _typed(symbols) if len(symbols) <= 4096 else None
        if key is not None:
            c = self.by_value.get(key)
            if c is not None:
                self.by_value.move_to_end(key)
                return c
        self.adopt(symbols, key)
        return symbols

    def adopt(self, symbols: tuple, key=None):
        self.by_id[id(symbols)] = symbols
        if key is None and len(symbols) <= 4096:
            key = _typed(symbols)
        if key is not None:
            self.by_value[key] = symbols
            while len(self.by_value) > self.limit:
                _, old = self.by_value.popitem(last=False)
                self.by_id.pop(id(old), None)
        else:
            # long lists (e.g. fresh sample_symbols subsets of HWF's 8332 outputs) are
            # known by identity only; bound them separately so they cannot accumulate
            self.large[id(symbols)] = symbols
            self.large.move_to_end(id(symbols))
            while len(self.large) > self.large_limit:
                oid, old = self.large.popitem(last=False)
                if self.by_id.get(oid) is old:
                    del self.by_id[oid]


_INTERN = _SymbolIntern()


def canonical_symbols(symbols: tuple) -> tuple:
    return _INTERN.canon(symbols)


def _fn_key(fn):
    """Hashable identity of a pure symbol function, or None when uncachable."""
    if fn is None:
        return ("none",)
    code = getattr(fn, "__code__", None)
    try:
        if code is None:
            hash(fn)
            return ("obj", fn)
        cells = getattr(fn, "__closure__", None)
        contents = tuple(c.cell_contents for c in cells) if cells else ()
        kw = getattr(fn, "__kwdefaults__", None)
        key = (
            "fn",
            code,
            getattr(fn, "__defaults__", None),
            tuple(sorted(kw.items())) if kw else None,
            contents,
            getattr(fn, "__self__", None),
        )
        hash(key)
        return key
    except (TypeError, ValueError):
        return None


# ----------------------------------------------------------------------------- plans
class SymbolPlan:
    """Result of the host map + shuffle stage for one apply_if call.

    combos   int32 [C+, arity]  input positions of every kept combination, ordinal order
    out_idx  int32 [C+]         output symbol of each kept combination (first derivation)
    table    int32 [prod S_i]   dense combination -> output index table, -1 = dropped
    """

    __slots__ = ("out_symbols", "sizes", "combos", "out_idx", "n_enumerated", "_kplan", "_table")

    def __init__(self, out_symbols, sizes, combos, out_idx, n_enumerated):
        self.out_symbols = out_symbols
        self.sizes = tuple(sizes)
        self.combos = combos
        self.out_idx = out_idx
        self.n_enumerated = n_enumerated
        self._kplan = None
        self._table = None

    @property
    def arity(self):
        return len(self.sizes)

    @property
    def n_out(self):
        return len(self.out_symbols)

    @property
    def n_kept(self):
        return int(self.combos.shape[0])

    @property
    def table(self) -> np.ndarray:
        if self._table is None:
            t = np.full(self.n_enumerated, -1, dtype=np.int32)
            if self.n_kept:
                flat = np.ravel_multi_index(tuple(self.combos.T.astype(np.int64)), self.sizes)
                t[flat] = self.out_idx
            self._table = t
        return self._table

    def groups(self):
        """Bucket member lists (ordinals) in output order, as the reference builds them."""
        order = np.argsort(self.out_idx, kind="stable")
        bounds = np.searchsorted(self.out_idx[order], np.arange(self.n_out + 1))
        return [order[bounds[i] : bounds[i + 1]].tolist() for i in range(self.n_out)]

    def kernel_plan(self) -> "KernelPlan":
        if self._kplan is None:
            self._kplan = KernelPlan(self.combos, self.out_idx, self.n_out, self.sizes, clamp=True)
        return self._kplan


_PLAN_CACHE: "OrderedDict[tuple, SymbolPlan]" = OrderedDict()
_PLAN_CACHE_LIMIT = 1024
_stats = {"hits": 0, "misses": 0, "uncachable": 0, "f_calls": 0}


def plan_cache_clear():
    _PLAN_CACHE.clear()
    for k in _stats:
        _stats[k] = 0


def plan_cache_info() -> dict:
    return dict(_stats, size=len(_PLAN_CACHE))


def build_plan(f, cond, symbol_lists) -> SymbolPlan:
    """Memoised host map/shuffle (distribution.py:244-260); bit-exact plan semantics."""
    canon = [canonical_symbols(tuple(s)) for s in symbol_lists]
    fk, ck = _fn_key(f), _fn_key(cond)
    key = None
    if fk is not None and ck is not None:
        key = (fk, ck, tuple(id(s) for s in canon))
        hit = _PLAN_CACHE.get(key)
        if hit is not None:
            _PLAN_CACHE.move_to_end(key)
            _stats["hits"] += 1
            return hit[0]
        _stats["misses"] += 1
    else:
        _stats["uncachable"] += 1
    plan = _map_shuffle(f, cond, canon)
    if key is not None:
        # the value keeps the canonical input tuples alive so their ids stay valid
        _PLAN_CACHE[key] = (plan, canon)
        while len(_PLAN_CACHE) > _PLAN_CACHE_LIMIT:
            _PLAN_CACHE.popitem(last=False)
    return plan


def _planner():
    """The native map/shuffle loop (csrc/planner.cpp, built by _build.build())."""
    global _PLANNER
    if _PLANNER is None:
        try:
            from . import _planner as mod
        except ImportError as exc:  # the product path has no interpreted fallback
            raise N.NativeError("native host planner _planner missing: run paper_2410_03348_b200._build") from exc
        _PLANNER = mod
    return _PLANNER


_PLANNER = None


def _map_shuffle(f, cond, symbol_lists) -> SymbolPlan:
    sizes = [len(s) for s in symbol_lists]
    n_enum = int(np.prod(sizes, dtype=np.int64)) if sizes else 0
    res = _planner().map_shuffle(f, cond, symbol_lists, UNDEFINED)
    if len(res) == 3 and res[0] == "error":
        _, syms, exc = res
        raise SymbolFunctionError(f"symbol function failed on {syms!r}: {exc}", syms) from exc
    out_symbols, kept_b, idx_b, calls = res
    _stats["f_calls"] += calls
    return _make_symbol_plan(out_symbols, sizes, np.frombuffer(kept_b, dtype=np.int64),
                             np.frombuffer(idx_b, dtype=np.int32).copy(), n_enum)


def _map_shuffle_py(f, cond, symbol_lists) -> SymbolPlan:
    """Interpreted restatement of the same loop (test reference for the native planner)."""
    sizes = [len(s) for s in symbol_lists]
    n_enum = int(np.prod(sizes, dtype=np.int64)) if sizes else 0
    kept = []
    out_idx = []
    buckets = {}
    calls = 0
    for ordinal, syms in enumerate(itertools.product(*symbol_lists)):
        if cond is not None:
            calls += 1
            if not call_user(cond, syms):
                continue
        calls += 1
        value = call_user(f, syms)
        if value is UNDEFINED:
            continue
        idx = buckets.get(value)
        if idx is None:
            idx = len(buckets)
            buckets[value] = idx
        kept.append(ordinal)
        out_idx.append(idx)
    _stats["f_calls"] += calls
    return _make_symbol_plan(tuple(buckets.keys()), sizes, np.asarray(kept, dtype=np.int64),
                             np.asarray(out_idx, dtype=np.int32), n_enum)


def _make_symbol_plan(out_symbols, sizes, kept, out_idx, n_enum) -> SymbolPlan:
    _INTERN.adopt(out_symbols)
    if len(kept) and sizes:
        combos = np.stack(np.unravel_index(kept, sizes), axis=1).astype(np.int32)
    elif len(kept):
        combos = np.zeros((len(kept), 0), dtype=np.int32)
    else:
        combos = np.zeros((0, len(sizes)), dtype=np.int32)
    return SymbolPlan(out_symbols, sizes, combos, out_idx, n_enum)


# ----------------------------------------------------------------------------- device plans
def _rec_words(n_ops: int) -> int:
    for w in (1, 2, 4, 8):
        if n_ops <= w:
            return w
    raise ValueError(f"arity {n_ops} exceeds the supported maximum of {N.MAX_ARITY}")


class HostSegsum:
    """One segmented problem: records grouped into segments, cut into bounded items."""

    __slots__ = ("n_seg", "rec_words", "recs", "items", "split", "n_partial", "work", "seg_off", "packed")

    def __init__(self, seg_off: np.ndarray, recs: np.ndarray, max_item: int, cut_points: np.ndarray | None = None,
                 cut_seg: np.ndarray | None = None, pack: int = 0):
        """Items hold at most ``max_item`` records.  With ``cut_points`` (record offsets of
        groups that must stay whole — one intermediate symbol's conj records in a fused
        conj -> group_disj — and ``cut_seg``, the segment of each group) items are made of
        whole groups and close before they would exceed ``max_item`` records (at least one
        group each)."""
        seg_off = np.asarray(seg_off, dtype=np.int64)
        n_seg = len(seg_off) - 1
        nrec, nops = recs.shape if recs.ndim == 2 else (recs.shape[0], 1)
        rw = _rec_words(max(nops, 1))
        packed = np.zeros((nrec, rw), dtype=np.int32)
        packed[:, :nops] = recs.reshape(nrec, nops)
        lens = np.diff(seg_off)
        self.packed = pack > 1
        if self.packed:
            # runs of whole short segments (<= pack records) per item; word 0 of every
            # segment's last record carries bit 31 (sg_dtkp_apply_desc.seg_packed); long
            # segments are split at max_item as usual
            seg_of, rb, re, pieces = self._pack(seg_off, lens, int(max_item), int(pack))
            n_items = len(seg_of)
            nz = np.nonzero(lens > 0)[0]
            packed[seg_off[nz + 1] - 1, 0] |= np.int32(-2**31)
        elif cut_points is None:
            pieces = np.maximum(1, -(-lens // max_item))
            n_items = int(pieces.sum())
            seg_of = np.repeat(np.arange(n_seg, dtype=np.int64), pieces)
            first = np.repeat(np.cumsum(pieces) - pieces, pieces)
            piece = np.arange(n_items, dtype=np.int64) - first
            rb = seg_off[seg_of] + piece * max_item
            re = np.minimum(rb + max_item, seg_off[seg_of + 1])
            re = np.maximum(re, rb)
        else:
            cp = np.asarray(cut_points, dtype=np.int64)
            gseg_off = np.searchsorted(np.asarray(cut_seg, dtype=np.int64), np.arange(n_seg + 1), side="left")
            seg_of, gb, ge = self._group_pieces(gseg_off, np.diff(cp), int(max_item))
            rb, re = cp[gb], cp[ge]
            pieces = np.bincount(seg_of, minlength=n_seg)
            n_items = len(seg_of)
        is_split = pieces[seg_of] > 1
        dest = np.full(n_items, -1, dtype=np.int64)
        n_partial = int(is_split.sum())
        dest[is_split] = np.arange(n_partial)
        items = np.stack([seg_of, rb, re, dest], axis=1).astype(np.int32)
        split_segs = np.nonzero(pieces > 1)[0]
        if len(split_segs):
            cnt = pieces[split_segs]
            pb = np.cumsum(cnt) - cnt
            split = np.stack([split_segs, pb, pb + cnt], axis=1).astype(np.int32)
        else:
            split = np.zeros((0, 3), dtype=np.int32)
        self.n_seg = n_seg
        self.rec_words = rw
        self.recs = packed
        self.items = items
        self.split = split
        self.n_partial = n_partial
        self.work = (re - rb) + 2  # records + per-item overhead
        self.seg_off = seg_off

    @staticmethod
    def _pack(seg_off, lens, max_item, pack):
        """(first segment, begin, end, pieces-per-segment) of packed items: whole segments
        gathered while the item holds at most `pack` records, segments longer than
        max_item split."""
        seg_of, rb, re = [], [], []
        pieces = np.ones(len(lens), dtype=np.int64)
        cur_s, cur_b, cur_n = -1, 0, 0
        for sgi, ln in enumerate(lens.tolist()):
            a = int(seg_off[sgi])
            if ln > max_item or ln == 0 or ln > pack:
                if cur_s >= 0:
                    seg_of.append(cur_s), rb.append(cur_b), re.append(cur_b + cur_n)
                    cur_s = -1
                if ln == 0:
                    seg_of.append(sgi), rb.append(a), re.append(a)
                    continue
                if ln <= max_item:  # a whole segment too long to pack: its own item
                    seg_of.append(sgi), rb.append(a), re.append(a + ln)
                    continue
                k = -(-ln // max_item)
                pieces[sgi] = k
                for p in range(k):
                    seg_of.append(sgi), rb.append(a + p * max_item), re.append(min(a + (p + 1) * max_item, a + ln))
                continue
            if cur_s >= 0 and cur_n + ln > pack:
                seg_of.append(cur_s), rb.append(cur_b), re.append(cur_b + cur_n)
                cur_s = -1
            if cur_s < 0:
                cur_s, cur_b, cur_n = sgi, a, 0
            cur_n += ln
        if cur_s >= 0:
            seg_of.append(cur_s), rb.append(cur_b), re.append(cur_b + cur_n)
        return (np.asarray(seg_of, dtype=np.int64), np.asarray(rb, dtype=np.int64), np.asarray(re, dtype=np.int64),
                pieces)

    @staticmethod
    def _group_pieces(gseg_off, gsize, max_w):
        """Per segment, runs of whole groups of at most max_w records (>= 1 group each);
        an empty segment still gets one (empty) item -> (segment, first group, end group)."""
        seg_of, gb, ge = [], [], []
        for sgi in range(len(gseg_off) - 1):
            a, b = int(gseg_off[sgi]), int(gseg_off[sgi + 1])
            start, acc = a, 0
            for g in range(a, b):
                if acc > 0 and acc + gsize[g] > max_w:
                    seg_of.append(sgi)
                    gb.append(start)
                    ge.append(g)
                    start, acc = g, 0
                acc += int(gsize[g])
            seg_of.append(sgi)
            gb.append(start)
            ge.append(b)
        return (np.asarray(seg_of, dtype=np.int64), np.asarray(gb, dtype=np.int64), np.asarray(ge, dtype=np.int64))

    def blocks(self, n_blocks: int) -> np.ndarray:
        """Item ranges of n_blocks contiguous CTA chunks balanced by work."""
        n_items = len(self.items)
        n_blocks = max(1, min(n_blocks, n_items))
        cum = np.concatenate([[0], np.cumsum(self.work)])
        targets = cum[-1] * np.arange(1, n_blocks) / n_blocks
        cuts = np.searchsorted(cum, targets, side="left")
        blk = np.concatenate([[0], cuts, [n_items]]).astype(np.int32)
        return np.maximum.accumulate(blk)


class DeviceSegsum:
    """HostSegsum uploaded to one device, with per-grid block partitions cached."""

    def __init__(self, host: HostSegsum, device, staged: bool, min_chunk_work: int, target_ctas: int = 2 * 148):
        self.host = host
        self.device = device
        self.staged = staged
        self.min_chunk_work = min_chunk_work
        self.target_ctas = target_ctas
        self.recs = torch.from_numpy(np.ascontiguousarray(host.recs.reshape(-1))).to(device)
        self.items = torch.from_numpy(np.ascontiguousarray(host.items.reshape(-1))).to(device)
        self.split = torch.from_numpy(np.ascontiguousarray(host.split.reshape(-1))).to(device)
        self.total_work = int(host.work.sum()) if len(host.work) else 0
        self._blk = {}

    def struct(self, B: int) -> N.SgSegsum:
        tiles = max(1, -(-B // 32))
        want = max(1, -(-self.target_ctas // tiles))
        cap = max(1, self.total_work // max(1, self.min_chunk_work))
        nb = 1
        while nb < min(want, cap):
            nb *= 2
        nb = min(nb, max(1, len(self.host.items)), 65535)
        blk = self._blk.get(nb)
        if blk is None:
            blk = torch.from_numpy(self.host.blocks(nb)).to(self.device)
            self._blk[nb] = blk
        s = N.SgSegsum()
        h = self.host
        s.n_seg = h.n_seg
        s.rec_words = h.rec_words
        s.n_items = len(h.items)
        s.n_blocks = int(blk.numel()) - 1
        s.n_split = len(h.split)
        s.n_partial = h.n_partial
        s.staged = 1 if self.staged else 0
        s.n_recs = len(h.recs)
        s.recs = self.recs.data_ptr() if self.recs.numel() else None
        s.items = self.items.data_ptr() if self.items.numel() else None
        s.blk = blk.data_ptr()
        s.split = self.split.data_ptr() if self.split.numel() else None
        return s


def csr(keys: np.ndarray, n_seg: int):
    """Stable CSR grouping: (order, seg_off) with records sorted by (key, position)."""
    order = np.argsort(keys, kind="stable")
    counts = np.bincount(keys, minlength=n_seg) if len(keys) else np.zeros(n_seg, dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return order, off


DAMP_MAX_ITEM = 128
DTKP_MAX_ITEM = 48
DTKP_PACK = os.environ.get("SG_DTKP_PACK", "1") != "0"  # runs of short segments per item
DTKP_RESIDENT_WARPS = 148 * 6 * 4  # one resident wave of 4-warp apply CTAs at 6 per SM


def dtkp_pack_size(n_rec: int, B: int) -> int:
    """Records per packed item: as many short segments per item as keeps ~4 items per
    resident warp of each 32-sample column (HWF-7 step 7 at B=64: 43; the CLUTRR closure
    at B=4096: its segments stay ~whole), so packing removes per-item overhead without
    starving the grid."""
    if not DTKP_PACK:
        return 0
    gx = max(1, -(-B // 32))
    target = max(1, 4 * DTKP_RESIDENT_WARPS // gx)
    p = min(DTKP_MAX_ITEM, n_rec // target)
    return p if p > 1 else 0


def dtkp_item_size(n_rec: int, B: int) -> int:
    """Records per piece of a long segment.  48 while the problem fills the resident warps
    several times over; a small problem with one long segment (HWF-7 step 4: 11,037
    records, one 101-record segment, ~6 records per resident warp) is cut finer, because
    its longest item is the launch's critical path — the two-level merge absorbs the
    extra partial lists."""
    gx = max(1, -(-B // 32))
    per_warp = n_rec * gx / DTKP_RESIDENT_WARPS
    if per_warp >= DTKP_MAX_ITEM / 2:
        return DTKP_MAX_ITEM
    return int(min(DTKP_MAX_ITEM, max(8, 2 * -(-int(per_warp * 2) // 2))))


DTKP_FUSED_ITEM = int(os.environ.get("SG_DTKP_FUSED_ITEM", "48"))  # conj records per fused item
DTKP_MERGE_ITEM = 8  # partial lists per first-level merge item (two-level merge)
STAGE_BYTES = 200 * 1024


class KernelPlan:
    """Device-ready form of a (records -> outputs) sum-of-products structure.

    records  int32 [n_rec, arity]: row of operand i used by record r
    out_idx  int32 [n_rec]:        output row the record contributes to
    """

    def __init__(self, records: np.ndarray, out_idx: np.ndarray, n_out: int, sizes, clamp: bool):
        self.records = np.ascontiguousarray(records, dtype=np.int32).reshape(len(out_idx), len(sizes))
        self.out_idx = np.ascontiguousarray(out_idx, dtype=np.int32)
        self.n_out = int(n_out)
        self.sizes = tuple(int(s) for s in sizes)
        self.arity = len(self.sizes)
        self.clamp = bool(clamp)
        if self.arity > N.MAX_ARITY:
            raise ValueError(f"apply arity {self.arity} exceeds {N.MAX_ARITY}")
        self.conv, self.conv_short = self._detect_toeplitz()
        self._fwd_host = None
        self._bwd_host = {}
        self._dtkp_host = None
        self._dev = {}

    # T[s0][s1] == s0 + s1 for every combination, no drops: a 1-D convolution per sample.
    # conv = 1: the short operand (<= 16 symbols) in registers (k_conv_*, fused chains);
    # conv = 2: both operands long (k_lconv, an FMA-bound direct convolution).
    # conv = 3: f = a + b + c over three lists, run as (a (*) b) (*) c (no clamp in between).
    def _detect_toeplitz(self):
        if self.arity == 3 and self.clamp:
            s0, s1, s2 = self.sizes
            if (len(self.out_idx) == s0 * s1 * s2 and self.n_out == s0 + s1 + s2 - 2
                    and np.array_equal(self.out_idx, self.records.sum(axis=1))):
                return 3, 0
            return 0, 0
        if self.arity != 2 or not self.clamp:
            return 0, 0
        s0, s1 = self.sizes
        if len(self.out_idx) != s0 * s1 or self.n_out != s0 + s1 - 1:
            return 0, 0
        if not np.array_equal(self.out_idx, self.records[:, 0] + self.records[:, 1]):
            return 0, 0
        if min(s0, s1) > 16:
            return 2, 0
        return 1, (1 if s1 <= s0 else 0)

    @property
    def n_rec(self):
        return len(self.out_idx)

    def fwd_host(self) -> HostSegsum:
        if self._fwd_host is None:
            order, off = csr(self.out_idx, self.n_out)
            self._fwd_host = HostSegsum(off, self.records[order], DAMP_MAX_ITEM)
        return self._fwd_host

    def bwd_host(self, k: int) -> HostSegsum:
        h = self._bwd_host.get(k)
        if h is None:
            order, off = csr(self.records[:, k], self.sizes[k])
            cols = [self.out_idx[order]] + [self.records[order, j] for j in range(self.arity) if j != k]
            h = HostSegsum(off, np.stack(cols, axis=1), DAMP_MAX_ITEM)
            self._bwd_host[k] = h
        return h

    def dtkp_host(self, pack: int = 0, item: int = DTKP_MAX_ITEM) -> HostSegsum:
        """DTKP work list; pack > 1 gathers runs of whole short segments of up to `pack`
        records per item (sg_dtkp_apply_desc.seg_packed); long segments are cut into
        pieces of `item` records."""
        if self._dtkp_host is None:
            self._dtkp_host = {}
        h = self._dtkp_host.get((pack, item))
        if h is None:
            order, off = csr(self.out_idx, self.n_out)
            h = HostSegsum(off, self.records[order], item, pack=pack)
            self._dtkp_host[(pack, item)] = h
        return h

    def dtkp_fused_host(self, inner: "KernelPlan") -> HostSegsum:
        """Fused conj -> group_disj (this plan arity 1 over ``inner``'s outputs, inner arity
        2): segments = this plan's outputs; records = for each of its records (an inner
        output s, ordinal order) the inner conj records of s in their ordinal order, the
        last one flagged by bit 31 of its second word (sg_dtkp_apply_desc.inner_arity).
        Items hold whole intermediate symbols, ~DTKP_FUSED_ITEM conj records each."""
        cache = self.__dict__.setdefault("_fused_hosts", {})
        hit = cache.get(id(inner))
        if hit is not None and hit[0] is inner:
            return hit[1]
        if self.arity != 1 or inner.arity != 2:
            raise ValueError("fused DTKP apply needs an arity-1 plan over an arity-2 plan")
        ih = inner.dtkp_host()
        ioff = np.asarray(ih.seg_off, dtype=np.int64)
        irecs = ih.recs[:, :2].astype(np.int64) & 0x7FFFFFFF  # (segment-end flags of a packed inner)
        order, off = csr(self.out_idx, self.n_out)
        mids = self.records[order, 0].astype(np.int64)
        lens = ioff[mids + 1] - ioff[mids]
        # flat conj records of every intermediate, in this plan's segment order
        starts = np.repeat(ioff[mids], lens)
        within = np.arange(int(lens.sum()), dtype=np.int64) - np.repeat(np.cumsum(lens) - lens, lens)
        flat = irecs[starts + within].copy()
        last = np.cumsum(lens) - 1
        flat[last, 1] |= np.int64(1) << 31
        flat = flat.astype(np.uint32).view(np.int32).reshape(-1, 2)
        # segment offsets and item cuts in flat-record units, at intermediate boundaries
        mid_off = np.concatenate([[0], np.cumsum(lens)])
        seg_off = mid_off[off]
        seg_of_mid = np.repeat(np.arange(self.n_out), np.diff(off))
        h = HostSegsum(seg_off, flat, DTKP_FUSED_ITEM, cut_points=mid_off, cut_seg=seg_of_mid)
        cache[id(inner)] = (inner, h)
        return h

    def maxprod_host(self) -> "dict[str, np.ndarray]":
        """CSR arrays of the max-product apply (sg_maxprod_plan): records grouped by output
        in first-derivation order, and per input the records using each row."""
        h = getattr(self, "_maxprod_host", None)
        if h is None:
            order, off = csr(self.out_idx, self.n_out)
            recs = self.records[order]
            h = {"seg_off": off.astype(np.int32), "recs": np.ascontiguousarray(recs, dtype=np.int32),
                 "rec_out": np.ascontiguousarray(self.out_idx[order], dtype=np.int32)}
            for k, n in enumerate(self.sizes):
                o, ko = csr(recs[:, k], n)
                h[f"in_off{k}"] = ko.astype(np.int32)
                h[f"in_recs{k}"] = o.astype(np.int32)
            self._maxprod_host = h
        return h

    def device(self, device) -> "DevicePlan":
        key = torch.device(device)
        dp = self._dev.get(key)
        if dp is None:
            dp = DevicePlan(self, key)
            self._dev[key] = dp
        return dp


class DevicePlan:
    """Per-device uploaded work lists of a KernelPlan (lazily, per direction)."""

    def __init__(self, kp: KernelPlan, device):
        self.kp = kp
        self.device = device
        self._fwd = None
        self._bwd = {}
        self._dtkp = None
        self._dtkp_merge = None
        self._dtkp_merge2 = None

    def _staged(self, rows: int) -> bool:
        return rows * 32 * 4 <= STAGE_BYTES

    def fwd(self) -> DeviceSegsum:
        if self._fwd is None:
            rows = sum(self.kp.sizes)
            self._fwd = DeviceSegsum(self.kp.fwd_host(), self.device, self._staged(rows), max(512, 2 * rows))
        return self._fwd

    def bwd(self, k: int) -> DeviceSegsum:
        d = self._bwd.get(k)
        if d is None:
            rows = self.kp.n_out + sum(s for j, s in enumerate(self.kp.sizes) if j != k)
            d = DeviceSegsum(self.kp.bwd_host(k), self.device, self._staged(rows), max(512, 2 * rows))
            self._bwd[k] = d
        return d

    def _dtkp_levels(self, host: HostSegsum):
        """(items, merge, merge2) device work lists of a DTKP segmented problem."""
        # DTKP items are latency-bound per warp: ask for ~8 resident CTAs per SM
        seg = DeviceSegsum(host, self.device, True, 16, target_ctas=148 * 8)
        merge = merge2 = None
        if len(host.split):
            # merge of the split segments' partial lists, itself cut into pieces of
            # DTKP_MERGE_ITEM partials whose lists a second level merges: the serial
            # chain of a 3868-record segment drops from 48 + 81 to 48 + 8 + 11 records
            off = np.concatenate([[0], host.split[:, 2]]).astype(np.int64)
            merge_recs = np.arange(host.n_partial, dtype=np.int32).reshape(-1, 1)
            mh = HostSegsum(off, merge_recs, DTKP_MERGE_ITEM)
            # merge items that finish a segment write the original output segment
            mh.items[:, 0] = host.split[mh.items[:, 0], 0]
            merge = DeviceSegsum(mh, self.device, True, 16, target_ctas=148 * 8)
            if len(mh.split):
                off2 = np.concatenate([[0], mh.split[:, 2]]).astype(np.int64)
                m2 = HostSegsum(off2, np.arange(mh.n_partial, dtype=np.int32).reshape(-1, 1), 1 << 30)
                m2.items[:, 0] = host.split[mh.split[m2.items[:, 0], 0], 0]
                merge2 = DeviceSegsum(m2, self.device, True, 16, target_ctas=148 * 8)
        return seg, merge, merge2

    def dtkp(self, B: int = 0):
        """(items, merge, merge2) for batch B (the packing granularity depends on B)."""
        pack = dtkp_pack_size(self.kp.n_rec, B) if B else 0
        item = dtkp_item_size(self.kp.n_rec, B) if B else DTKP_MAX_ITEM
        if self._dtkp is None:
            self._dtkp = {}
        hit = self._dtkp.get((pack, item))
        if hit is None:
            hit = self._dtkp_levels(self.kp.dtkp_host(pack, item))
            self._dtkp[(pack, item)] = hit
        return hit

    def dtkp_fused(self, inner: "KernelPlan"):
        """(items, merge, merge2) of the fused conj -> group_disj over ``inner``."""
        cache = self.__dict__.setdefault("_fused", {})
        hit = cache.get(id(inner))
        if hit is None or hit[0] is not inner:
            hit = (inner, self._dtkp_levels(self.kp.dtkp_fused_host(inner)))
            cache[id(inner)] = hit
        return hit[1]

    def maxprod_struct(self) -> N.SgMaxprodPlan:
        d = getattr(self, "_maxprod", None)
        if d is None:
            d = {k: torch.from_numpy(v).to(self.device) for k, v in self.kp.maxprod_host().items()}
            self._maxprod = d
        kp = self.kp
        s = N.SgMaxprodPlan()
        s.arity = kp.arity
        s.n_out = kp.n_out
        s.n_recs = len(kp.out_idx)
        for i, n in enumerate(kp.sizes):
            s.sizes[i] = n
            s.in_off[i] = d[f"in_off{i}"].data_ptr()
            s.in_recs[i] = d[f"in_recs{i}"].data_ptr() if d[f"in_recs{i}"].numel() else None
        s.seg_off = d["seg_off"].data_ptr()
        s.recs = d["recs"].data_ptr() if d["recs"].numel() else None
        s.rec_out = d["rec_out"].data_ptr() if d["rec_out"].numel() else None
        return s

    def damp_struct(self, B: int, need_bwd=()) -> N.SgDampPlan:
        kp = self.kp
        s = N.SgDampPlan()
        s.arity = kp.arity
        s.n_out = kp.n_out
        for i, n in enumerate(kp.sizes):
            s.sizes[i] = n
        s.conv = int(kp.conv)
        s.conv_short = kp.conv_short
        if not kp.conv:
            s.fwd = self.fwd().struct(B)
            for k in need_bwd:
                s.bwd[k] = self.bwd(k).struct(B)
        return s
