"""Provenance semirings over batched device tags (the plugin API of provenance.py).

``Damp`` and ``DtkpAm`` keep the reference's duck-typed protocol (provenance.py:217-457):
``input_tags, zero, one, gather, conj, disj, group_disj, concat_syms, probs,
forward_probs, placed, stack_parts`` (+ ``tags_from_proofs`` for DTKP), and add the fused
entry points the new ``apply_if`` / ``union`` always call: ``apply_plan`` and
``union_tags``.  All tag work runs in the sm_100a kernels of ``libsgb200.so``.

Tag storage (symbol-major, batch innermost — see include/sgb200.h):
  DampTags   ``sm``   float32 [n][B]  (``.value`` is the (B, n) transposed view)
  DtkpTags   ``pm``   int64   [n][K][W][B]  packed u64 proof bitmasks
             ``pp``   uint8   [n][K][B]     present flags
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import ops
from .plan import KernelPlan, SymbolPlan

__all__ = [
    "ProvenanceError",
    "InputRegistry",
    "Damp",
    "DampMax",
    "DtkpAm",
    "DampTags",
    "DtkpTags",
    "wmc_exact",
    "provenance_from_name",
]


class ProvenanceError(ValueError):
    """Registry misuse or incompatible tags."""


def _default_device():
    if not torch.cuda.is_available():
        raise ops.N.NativeError("no CUDA device: the Dolphin hot path runs only on the GPU")
    return torch.device("cuda", torch.cuda.current_device())


def _as_probs(probs, device) -> torch.Tensor:
    if isinstance(probs, torch.Tensor):
        t = probs if probs.is_cuda else probs.to(device)
    else:
        t = torch.as_tensor(np.asarray(probs, dtype=np.float64), device=device)
    if t.dtype not in (torch.float32, torch.float64, torch.float16, torch.bfloat16):
        t = t.double()
    return t


class InputRegistry:
    """Ordered universe of input symbols and their probability leaves (provenance.py:66-137).

    Blocks are kept as the caller's (b, n) tensors plus their symbol-major fp32 copies;
    ``prob_values`` / ``prob_tensor`` give the registry as one [I][B] fp32 tensor.
    """

    def __init__(self, device=None):
        self.ids = []
        self._parts = []  # symbol-major [n][b] fp32 tensors (autograd-connected)
        self._frozen = False
        self._prob_cache = None
        self._value_cache = None
        self.device = torch.device(device) if device is not None else None

    @property
    def size(self) -> int:
        return len(self.ids)

    @property
    def frozen(self) -> bool:
        return self._frozen

    def freeze(self):
        self._frozen = True

    def _dev(self):
        if self.device is None:
            self.device = _default_device()
        return self.device

    def add_block(self, ids, probs_sm: torch.Tensor) -> int:
        """Append a block of columns given as symbol-major [n][b]; returns its first column."""
        if self._frozen:
            raise ProvenanceError("cannot register inputs after the registry is frozen")
        if probs_sm.ndim != 2 or probs_sm.shape[0] != len(ids):
            raise ProvenanceError(
                f"probability block shape {tuple(probs_sm.shape[::-1])} does not match {len(ids)} input symbols"
            )
        start = len(self.ids)
        self.ids.extend(ids)
        self._parts.append(probs_sm)
        self._value_cache = None
        self._prob_cache = None
        return start

    @property
    def batch(self) -> int:
        return max((p.shape[1] for p in self._parts), default=1)

    def prob_tensor(self) -> torch.Tensor:
        """Differentiable [I][B] fp32 view of all registered probabilities."""
        if self._frozen and self._prob_cache is not None:
            return self._prob_cache
        if not self._parts:
            raise ProvenanceError("registry holds no input symbols")
        b = self.batch
        parts = [ops.expand_batch(p, b) for p in self._parts]
        out = parts[0].contiguous() if len(parts) == 1 else torch.cat(parts, dim=0)
        if self._frozen:
            self._prob_cache = out
        return out

    def prob_values(self) -> torch.Tensor:
        """[I][B] fp32 probabilities without autograd (ranking keys)."""
        if self._value_cache is None:
            if not self._parts:
                self._value_cache = torch.zeros((0, 1), device=self._dev(), dtype=torch.float32)
            else:
                b = self.batch
                with torch.no_grad():
                    parts = [p.detach().expand(p.shape[0], b) for p in self._parts]
                    self._value_cache = torch.cat(parts, dim=0).contiguous()
        return self._value_cache


# ================================================================================== DAMP
class _ConvChain:
    """A pending left fold of Toeplitz applies (every Sum-N fold step).

    ``Damp.apply_plan`` extends the chain instead of launching a kernel per apply; the
    first consumer of the values (``get_probs``, another non-Toeplitz op, a host read)
    materialises it with ONE fused forward launch, and autograd runs ONE fused backward
    (ops.ConvChainFn).  Results equal the per-apply kernels step for step."""

    __slots__ = ("base", "filters", "kf", "B", "n_out", "first_plan", "kind")
    MAX_STEPS = 32

    @staticmethod
    def max_rows(kf: int, kind: str = "sum") -> int:
        """Longest state (rows) whose fwd/bwd shared-memory working set fits one CTA."""
        return ops.chain_max_rows(kf) if kind == "sum" else ops.maxchain_max_rows(kf)

    def __init__(self, base, filters, kf, B, n_out, first_plan, kind="sum"):
        self.base, self.filters, self.kf, self.B, self.n_out = base, filters, kf, B, n_out
        self.first_plan = first_plan
        self.kind = kind

    def can_extend(self, kf: int, B: int, n_out: int, kind: str = "sum") -> bool:
        return (kind == self.kind and kf == self.kf and B == self.B and len(self.filters) < self.MAX_STEPS
                and n_out <= self.max_rows(kf, kind) and n_out == self.n_out + kf - 1)

    def extend(self, short_sm: torch.Tensor, n_out: int) -> "_ConvChain":
        return _ConvChain(self.base, self.filters + [short_sm], self.kf, self.B, n_out, self.first_plan, self.kind)

    def materialize(self) -> torch.Tensor:
        if len(self.filters) == 1:  # a single apply: the per-apply kernel
            ops_ = _conv_operands(self.first_plan, self.base, self.filters[0])
            if self.kind == "max":
                return ops.maxprod_apply(self.first_plan, ops_, self.B)
            return ops.damp_apply(self.first_plan, ops_, self.B)
        fn = ops.ConvChainFn if self.kind == "sum" else ops.MaxChainFn
        return fn.apply(self.base.shape[0], self.kf, self.B, ops.expand_batch(self.base, self.B),
                        *[ops.expand_batch(f, self.B) for f in self.filters])


def _conv_operands(kp, long_sm, short_sm):
    ops_ = [None, None]
    ops_[kp.conv_short] = short_sm
    ops_[1 - kp.conv_short] = long_sm
    return ops_


class DampTags:
    """Probability tags for a whole symbol list: symbol-major fp32 [n][b] on the device
    (possibly a pending Toeplitz chain, materialised on first access of ``sm``)."""

    __slots__ = ("_sm", "_chain")

    def __init__(self, value=None, *, sm: torch.Tensor | None = None, chain: _ConvChain | None = None):
        if sm is None and chain is None:
            v = _as_probs(value, _default_device())
            if v.ndim != 2:
                raise ValueError("DampTags value must be (batch, n)")
            sm = ops.symbol_view(v)
        self._sm = sm
        self._chain = chain

    @property
    def sm(self) -> torch.Tensor:
        if self._sm is None:
            self._sm = self._chain.materialize()
            self._chain = None
        return self._sm

    @property
    def pending(self) -> bool:
        return self._sm is None

    @property
    def value(self) -> torch.Tensor:
        return self.sm.t()

    @property
    def batch(self) -> int:
        return self._chain.B if self._sm is None else self._sm.shape[1]

    @property
    def count(self) -> int:
        return self._chain.n_out if self._sm is None else self._sm.shape[0]


def _damp(sm: torch.Tensor) -> DampTags:
    return DampTags(sm=sm)


class Damp:
    """Add-mult probabilities: conj = product, disj = clamped sum (provenance.py:217-271)."""

    name = "damp"
    k = None

    def input_tags(self, registry, ids, probs) -> DampTags:
        """The classifier block is read in place as an (n, B) view — no layout copy."""
        sm = ops.symbol_view(_as_probs(probs, registry._dev()))
        registry.add_block(ids, sm)
        return _damp(sm)

    def zero(self, registry, b: int = 1, n: int = 1) -> DampTags:
        return _damp(torch.zeros((n, b), device=registry._dev(), dtype=torch.float32))

    def one(self, registry, b: int = 1, n: int = 1) -> DampTags:
        return _damp(torch.ones((n, b), device=registry._dev(), dtype=torch.float32))

    def gather(self, tags: DampTags, indices) -> DampTags:
        rng = _as_range(indices)
        if rng is not None:  # e.g. HWF's digit / operator filters: a zero-copy row view
            return _damp(tags.sm[rng[0]:rng[1]])
        return _damp(ops.damp_apply(ops.gather_plan(indices, tags.count), [tags.sm], tags.batch))

    def conj(self, a: DampTags, b: DampTags) -> DampTags:
        B = max(a.batch, b.batch)
        return _damp(ops.damp_apply(_colwise_conj_plan(a.count, b.count), [a.sm, b.sm], B))

    def disj(self, a: DampTags, b: DampTags) -> DampTags:
        n = max(a.count, b.count)
        B = max(a.batch, b.batch)
        ia = np.arange(n) if a.count == n else np.zeros(n, dtype=np.int64)
        ib = np.arange(n) if b.count == n else np.zeros(n, dtype=np.int64)
        dev = a.sm.device
        return _damp(
            ops.DampRowsAdd.apply(
                ops.expand_batch(a.sm, B), ops.expand_batch(b.sm, B), ops.index_map(ia, a.count, dev),
                ops.index_map(ib, b.count, dev), True,
            )
        )

    def group_disj(self, tags: DampTags, groups) -> DampTags:
        """Bucket disjunction: clamp01 of the per-group sum (provenance.py:242-253)."""
        kp = _group_plan(groups, tags.count)
        return _damp(ops.damp_apply(kp, [tags.sm], tags.batch))

    def concat_syms(self, parts) -> DampTags:
        B = max(p.batch for p in parts)
        return _damp(torch.cat([ops.expand_batch(p.sm, B) for p in parts], dim=0))

    def probs(self, tags: DampTags) -> torch.Tensor:
        return tags.value

    def forward_probs(self, tags: DampTags) -> np.ndarray:
        return tags.sm.detach().t().double().cpu().numpy()

    def placed(self, tags: DampTags, placement: np.ndarray) -> DampTags:
        return _damp(ops.damp_apply(ops.gather_plan(_placement_src(placement), tags.count), [tags.sm], tags.batch))

    def stack_parts(self, parts) -> DampTags:
        return _damp(torch.cat([p.sm for p in parts], dim=1))

    # ---- fused entry points ---------------------------------------------------------
    fuse_chains = os.environ.get("SG_FUSE_CHAINS", "1") != "0"

    def apply_plan(self, tags_list, plan: SymbolPlan, batch: int) -> DampTags:
        """K1 (+K2 through autograd): gather -> conj fold -> group_disj in one kernel.

        Toeplitz applies whose long operand is the previous apply's output are deferred
        into a fused chain (``_ConvChain``) and run as one launch each way."""
        kp = plan.kernel_plan()
        if self.fuse_chains and kp.conv == 1 and len(tags_list) == 2:
            long_t, short_t = tags_list[1 - kp.conv_short], tags_list[kp.conv_short]
            kf = kp.sizes[kp.conv_short]
            if short_t.batch in (1, batch) and long_t.batch in (1, batch) and kp.n_out <= _ConvChain.max_rows(kf):
                ch = long_t._chain
                if ch is not None and ch.can_extend(kf, batch, kp.n_out):
                    return DampTags(chain=ch.extend(short_t.sm, kp.n_out))
                if ch is None or not ch.can_extend(kf, batch, kp.n_out):
                    return DampTags(chain=_ConvChain(long_t.sm, [short_t.sm], kf, batch, kp.n_out, kp))
        return _damp(ops.damp_apply(kp, [t.sm for t in tags_list], batch))

    def union_tags(self, a: DampTags, b: DampTags, uplan) -> DampTags:
        B = max(a.batch, b.batch)
        dev = a.sm.device
        return _damp(
            ops.DampRowsAdd.apply(
                ops.expand_batch(a.sm, B), ops.expand_batch(b.sm, B), ops.index_map(uplan.ia, a.count, dev),
                ops.index_map(uplan.ib, b.count, dev), True,
            )
        )


class DampMax(Damp):
    """Max-product probabilities: the north star's "max/DAMP variant" of kernel (1).

    There is no max provenance in the reference, so it is assembled from the
    reference's primitives: conj is the DAMP product (provenance.py:236), disj is
    tensor.py's reduce "max" (tensor.py:319-325: gradient to the FIRST maximal entry, here
    the earliest record in first-derivation order), followed by DAMP's clamp01 (pass-through
    gradient, tensor.py:287).  Every operator runs on sg_maxprod_fwd / sg_maxprod_bwd;
    tags are the same symbol-major fp32 [n][b] as Damp's."""

    name = "max"

    def gather(self, tags: DampTags, indices) -> DampTags:
        rng = _as_range(indices)
        if rng is not None:
            return _damp(tags.sm[rng[0]:rng[1]])
        return _damp(ops.maxprod_apply(ops.gather_plan(indices, tags.count), [tags.sm], tags.batch))

    def conj(self, a: DampTags, b: DampTags) -> DampTags:
        B = max(a.batch, b.batch)
        return _damp(ops.maxprod_apply(_colwise_conj_plan(a.count, b.count), [a.sm, b.sm], B))

    def _pairwise_max(self, a: DampTags, b: DampTags, ia, ib) -> DampTags:
        """out[s] = clamp01(max(a[ia[s]], b[ib[s]])), -1 = absent; ties go to a."""
        B = max(a.batch, b.batch)
        kp = _pairwise_max_plan(np.asarray(ia, dtype=np.int32), np.asarray(ib, dtype=np.int32), a.count, b.count)
        both = torch.cat([ops.expand_batch(a.sm, B), ops.expand_batch(b.sm, B)], dim=0)
        return _damp(ops.maxprod_apply(kp, [both], B))

    def disj(self, a: DampTags, b: DampTags) -> DampTags:
        n = max(a.count, b.count)
        ia = np.arange(n) if a.count == n else np.zeros(n, dtype=np.int64)
        ib = np.arange(n) if b.count == n else np.zeros(n, dtype=np.int64)
        return self._pairwise_max(a, b, ia, ib)

    def group_disj(self, tags: DampTags, groups) -> DampTags:
        kp = _group_plan(groups, tags.count)
        return _damp(ops.maxprod_apply(kp, [tags.sm], tags.batch))

    def placed(self, tags: DampTags, placement: np.ndarray) -> DampTags:
        return _damp(ops.maxprod_apply(ops.gather_plan(_placement_src(placement), tags.count), [tags.sm],
                                       tags.batch))

    def apply_plan(self, tags_list, plan: SymbolPlan, batch: int) -> DampTags:
        """gather -> product fold -> max bucket (+clamp) in one sg_maxprod_fwd launch;
        Toeplitz applies whose long operand (input 0, so records are ordered by it) is the
        previous apply's output fold into one fused max chain (sg_maxchain_*)."""
        kp = plan.kernel_plan()
        if self.fuse_chains and kp.conv == 1 and kp.conv_short == 1 and len(tags_list) == 2:
            long_t, short_t = tags_list[0], tags_list[1]
            kf = kp.sizes[1]
            if short_t.batch in (1, batch) and long_t.batch in (1, batch) and \
                    kp.n_out <= _ConvChain.max_rows(kf, "max"):
                ch = long_t._chain
                if ch is not None and ch.can_extend(kf, batch, kp.n_out, "max"):
                    return DampTags(chain=ch.extend(short_t.sm, kp.n_out))
                return DampTags(chain=_ConvChain(long_t.sm, [short_t.sm], kf, batch, kp.n_out, kp, "max"))
        return _damp(ops.maxprod_apply(kp, [t.sm for t in tags_list], batch))

    def union_tags(self, a: DampTags, b: DampTags, uplan) -> DampTags:
        return self._pairwise_max(a, b, uplan.ia, uplan.ib)


_GROUPS: "dict[tuple, KernelPlan]" = {}


def _group_plan(groups, n_src: int) -> KernelPlan:
    """group_disj's bucket plan (records in (group, ordinal) order), memoised by content."""
    recs = np.asarray([c for g in groups for c in g], dtype=np.int32).reshape(-1, 1)
    out = np.asarray([s for s, g in enumerate(groups) for _ in g], dtype=np.int32)
    key = (int(n_src), len(groups), recs.tobytes(), out.tobytes())
    kp = _GROUPS.get(key)
    if kp is None:
        kp = KernelPlan(recs, out, len(groups), (int(n_src),), clamp=True)
        if len(_GROUPS) > 4096:
            _GROUPS.clear()
        _GROUPS[key] = kp
    return kp


_COLWISE: "dict[tuple, KernelPlan]" = {}


def _colwise_conj_plan(na: int, nb: int) -> KernelPlan:
    """Column-wise product plan of conj (provenance.py:236: a batch-1 / single-column side
    broadcasts).  Memoised like every other plan: its device tables are uploaded once, so
    a CUDA graph captured over conj never references freed plan memory."""
    key = (na, nb)
    kp = _COLWISE.get(key)
    if kp is None:
        n = max(na, nb)
        ia = np.arange(n) if na == n else np.zeros(n, dtype=np.int64)
        ib = np.arange(n) if nb == n else np.zeros(n, dtype=np.int64)
        kp = KernelPlan(np.stack([ia, ib], axis=1), np.arange(n), n, (na, nb), clamp=False)
        if len(_COLWISE) > 4096:
            _COLWISE.clear()
        _COLWISE[key] = kp
    return kp


_PAIRMAX: "dict[tuple, KernelPlan]" = {}


def _pairwise_max_plan(ia: np.ndarray, ib: np.ndarray, na: int, nb: int) -> KernelPlan:
    """out[s] = max over {a[ia[s]], b[ib[s]]} (records: a's row first, then b's), memoised
    by (ia, ib, counts)."""
    key = (na, nb, ia.tobytes(), ib.tobytes())
    kp = _PAIRMAX.get(key)
    if kp is None:
        recs, outs = [], []
        for s in range(len(ia)):
            if ia[s] >= 0:
                recs.append(int(ia[s]))
                outs.append(s)
            if ib[s] >= 0:
                recs.append(na + int(ib[s]))
                outs.append(s)
        kp = KernelPlan(np.asarray(recs, dtype=np.int32).reshape(-1, 1), np.asarray(outs, dtype=np.int32), len(ia),
                        (na + nb,), clamp=True)
        if len(_PAIRMAX) > 4096:
            _PAIRMAX.clear()
        _PAIRMAX[key] = kp
    return kp


def _as_range(indices):
    """(start, stop) when indices are one ascending contiguous run (gather = a view)."""
    idx = np.asarray(indices, dtype=np.int64).reshape(-1)
    if idx.size == 0:
        return None
    a = int(idx[0])
    if a >= 0 and np.array_equal(idx, np.arange(a, a + idx.size)):
        return a, a + idx.size
    return None


def _placement_src(placement: np.ndarray) -> np.ndarray:
    placement = np.asarray(placement)
    src = np.full(placement.shape[1], -1, dtype=np.int32)
    s, d = np.nonzero(placement)
    src[d] = s
    return src


# ================================================================================== DTKP
def _words(I: int) -> int:
    return (I + 63) // 64


def pack_member(member_u8: np.ndarray) -> np.ndarray:
    """u8 [b, n, k, I] -> u64 bit pattern (as int64) [n, k, W, b]; bit j%64 of word j//64."""
    b, n, k, I = member_u8.shape
    W = _words(I)
    bits = np.packbits((np.asarray(member_u8) != 0).astype(np.uint8), axis=-1, bitorder="little")
    pad = np.zeros((b, n, k, W * 8), dtype=np.uint8)
    pad[..., : bits.shape[-1]] = bits
    words = pad.view("<u8").reshape(b, n, k, W)
    return np.ascontiguousarray(words.transpose(1, 2, 3, 0)).view(np.int64)


def unpack_member(pm: np.ndarray, I: int) -> np.ndarray:
    """int64 [n, k, W, b] -> u8 [b, n, k, I]."""
    n, k, W, b = pm.shape
    words = np.ascontiguousarray(pm.transpose(3, 0, 1, 2)).view("<u8")
    bits = np.unpackbits(words.view(np.uint8).reshape(b, n, k, W * 8), axis=-1, bitorder="little")
    return np.ascontiguousarray(bits[..., :I])


class DtkpTags:
    """Proof-matrix tags for a whole symbol list (packed on the device).

    The constructor also accepts the reference layout — ``member`` uint8 (b, n, k, I) and
    ``present`` uint8 (b, n, k) host arrays — and packs it.
    """

    __slots__ = ("_pm", "_pp", "registry", "_pending", "ranked")

    def __init__(self, member, present, registry, pending: "_PendingConj | None" = None, ranked: bool | None = None):
        # ranked: every (symbol, sample) holds its present rows first, in non-increasing key
        # order — true for every tag the kernels, input_tags / zero / one and the row
        # gathers produce; hand-built reference-layout tags are not assumed ranked
        self._pending = pending
        if pending is not None:
            self._pm = self._pp = None
            self.ranked = True
        elif isinstance(member, torch.Tensor) and member.dtype == torch.int64 and member.ndim == 4:
            self._pm = member
            self._pp = present
            self.ranked = True if ranked is None else bool(ranked)
        else:
            self.ranked = False if ranked is None else bool(ranked)
            m = np.asarray(member.cpu() if isinstance(member, torch.Tensor) else member, dtype=np.uint8)
            pr = np.asarray(present.cpu() if isinstance(present, torch.Tensor) else present, dtype=np.uint8)
            dev = registry._dev()
            self._pm = torch.as_tensor(pack_member(m), device=dev)
            self._pp = torch.as_tensor(np.ascontiguousarray(pr.transpose(1, 2, 0)), device=dev)
        self.registry = registry

    # A binary-conj apply may be left pending: its consumer, if it is a group_disj-shaped
    # apply (an arity-1 apply_plan), fuses both into one launch and the intermediate tag
    # never exists; every other access materialises it with the plain apply kernel.
    def _materialise(self):
        pm, pp = self._pending.run()
        self._pm, self._pp, self._pending = pm, pp, None

    @property
    def pm(self) -> torch.Tensor:
        if self._pending is not None:
            self._materialise()
        return self._pm

    @pm.setter
    def pm(self, v):
        self._pm = v

    @property
    def pp(self) -> torch.Tensor:
        if self._pending is not None:
            self._materialise()
        return self._pp

    @pp.setter
    def pp(self, v):
        self._pp = v

    @property
    def pending(self) -> "_PendingConj | None":
        return self._pending

    @property
    def batch(self) -> int:
        return self._pending.B if self._pending is not None else self._pm.shape[3]

    @property
    def count(self) -> int:
        return self._pending.kp.n_out if self._pending is not None else self._pm.shape[0]

    @property
    def k(self) -> int:
        return self._pending.K if self._pending is not None else self._pm.shape[1]

    @property
    def W(self) -> int:
        return self._pending.W if self._pending is not None else self._pm.shape[2]

    def aligned(self) -> "DtkpTags":
        """Pad the word axis to the registry width (provenance.py:185-192)."""
        W = _words(self.registry.size)
        if self.pm.shape[2] < W:
            n, k, w, b = self.pm.shape
            pm = torch.zeros((n, k, W, b), device=self.pm.device, dtype=torch.int64)
            pm[:, :, :w] = self.pm
            self.pm = pm
        return self

    # ---- reference-layout host views (debug / tests) ----------------------------------
    @property
    def member(self) -> np.ndarray:
        return unpack_member(self.pm.cpu().numpy(), self.registry.size)

    @property
    def present(self) -> np.ndarray:
        return np.ascontiguousarray(self.pp.cpu().numpy().transpose(2, 0, 1))

    def aligned_member(self) -> np.ndarray:
        return self.member

    def to_matrix(self) -> np.ndarray:
        member = self.member.astype(bool)
        present = self.present.astype(bool)
        p = self.registry.prob_values().t().double().cpu().numpy()
        out = np.where(member, p[:, None, None, :], np.inf)
        return np.where(present[..., None], out, -np.inf)

    def proof_sets(self, col: int = 0):
        member = self.member
        present = self.present
        out = []
        for m in range(self.batch):
            proofs = set()
            for r in range(self.k):
                if present[m, col, r]:
                    proofs.add(frozenset(np.flatnonzero(member[m, col, r]).tolist()))
            out.append(proofs)
        return out


class _PendingConj:
    """A deferred binary-conj DTKP apply (plan, operands and registry state captured at
    call time, so later registrations cannot change what it computes)."""

    __slots__ = ("prov", "registry", "kp", "operands", "B", "K", "W", "I", "p")

    def __init__(self, prov, registry, kp, operands, B, p):
        self.prov, self.registry, self.kp, self.operands, self.B = prov, registry, kp, operands, B
        self.K = prov.k
        self.I = registry.size
        self.W = _words(self.I)
        self.p = p

    def run(self):
        dseg, dmerge, dmerge2 = self.kp.device(self.p.device).dtkp(self.B)
        return ops.dtkp_apply(self.kp, dseg, dmerge, self.operands, None, self.K, self.W, self.I, self.B, self.p, 2,
                              dmerge2)


def _bcast_dtkp(t: DtkpTags, B: int):
    pm, pp = t.pm, t.pp
    if pm.shape[3] != B:
        if pm.shape[3] != 1:
            raise ProvenanceError(f"cannot broadcast tag batch {pm.shape[3]} to {B}")
        pm = pm.expand(*pm.shape[:3], B).contiguous()
        pp = pp.expand(*pp.shape[:2], B).contiguous()
    return pm, pp


_WORDS_CACHE: "dict[tuple, torch.Tensor]" = {}


def _input_words(start: int, n: int, k: int, W: int, device) -> torch.Tensor:
    """Device template [n][k][W] of single-proof input tags (cached: no H2D per call,
    so programs stay CUDA-graph capturable)."""
    key = (start, n, k, W, torch.device(device))
    t = _WORDS_CACHE.get(key)
    if t is None:
        words = np.zeros((n, k, W), dtype=np.uint64)
        for i in range(n):
            j = start + i
            words[i, 0, j // 64] = np.uint64(1) << np.uint64(j % 64)
        t = torch.as_tensor(words.view(np.int64), device=device)
        if len(_WORDS_CACHE) > 4096:
            _WORDS_CACHE.clear()
        _WORDS_CACHE[key] = t
    return t


class _IdentityPlans:
    """Cached KernelPlans of the column-wise DTKP operators (conj / disj) per width n."""

    def __init__(self):
        self.conj = {}
        self.disj = {}

    def conj_plan(self, n):
        kp = self.conj.get(n)
        if kp is None:
            r = np.arange(n, dtype=np.int32)
            kp = KernelPlan(np.stack([r, r], axis=1), r, n, (n, n), clamp=True)
            self.conj[n] = kp
        return kp

    def disj_plan(self, n):
        kp = self.disj.get(n)
        if kp is None:
            r = np.arange(n, dtype=np.int32)
            recs = np.stack([r, r + n], axis=1).reshape(-1, 1)
            out = np.repeat(r, 2)
            kp = KernelPlan(recs, out, n, (2 * n,), clamp=True)
            self.disj[n] = kp
        return kp


_IDPLANS = _IdentityPlans()


class DtkpAm:
    """Top-k proof matrices with add-mult probability extraction (provenance.py:274-457)."""

    name = "dtkp"

    def __init__(self, k: int):
        if k < 1:
            raise ProvenanceError(f"top-k retention needs k >= 1, got {k}")
        if k > 8:
            raise ProvenanceError(f"the sm_100a top-k kernels support k <= 8, got {k}")
        self.k = int(k)

    # ---- construction ----------------------------------------------------------------
    def input_tags(self, registry, ids, probs) -> DtkpTags:
        sm = ops.symbol_view(_as_probs(probs, registry._dev()))
        start = registry.add_block(ids, sm)
        n, b = sm.shape
        W = _words(registry.size)
        words = _input_words(start, n, self.k, W, sm.device)
        pm = words[..., None].expand(n, self.k, W, b).contiguous()
        pp = torch.zeros((n, self.k, b), device=sm.device, dtype=torch.uint8)
        pp[:, 0] = 1
        return DtkpTags(pm, pp, registry)

    def zero(self, registry, b: int = 1, n: int = 1) -> DtkpTags:
        dev = registry._dev()
        W = _words(registry.size)
        return DtkpTags(torch.zeros((n, self.k, W, b), device=dev, dtype=torch.int64),
                        torch.zeros((n, self.k, b), device=dev, dtype=torch.uint8), registry)

    def one(self, registry, b: int = 1, n: int = 1) -> DtkpTags:
        t = self.zero(registry, b, n)
        t.pp[:, 0] = 1  # single empty proof
        return t

    def _check_registry(self, a: DtkpTags, b: DtkpTags):
        if a.registry is not b.registry:
            raise ProvenanceError("tags belong to different input registries")
        if a.count != b.count:
            raise ProvenanceError(f"columnwise tag operation on {a.count} vs {b.count} symbols")

    def _p(self, registry, B: int) -> torch.Tensor:
        p = registry.prob_values()
        if p.shape[1] == B:
            return p
        if p.shape[1] == 1:
            return p.expand(p.shape[0], B).contiguous()
        raise ProvenanceError(f"registry batch {p.shape[1]} does not match tag batch {B}")

    def _run(self, registry, kp: KernelPlan, operands, tail, arity: int, B: int, ranked: bool = True) -> DtkpTags:
        W = _words(registry.size)
        p = self._p(registry, B)
        dseg, dmerge, dmerge2 = kp.device(p.device).dtkp(B)
        pm, pp = ops.dtkp_apply(kp, dseg, dmerge, operands, tail, self.k, W, registry.size, B, p, arity, dmerge2,
                                ranked=ranked and ops.DTKP_RANKED)
        return DtkpTags(pm, pp, registry)

    # ---- protocol ----------------------------------------------------------------------
    def gather(self, tags: DtkpTags, indices) -> DtkpTags:
        rng = _as_range(indices)
        if rng is not None:  # contiguous symbol rows: a zero-copy view of both tensors
            return DtkpTags(tags.pm[rng[0]:rng[1]], tags.pp[rng[0]:rng[1]], tags.registry, ranked=tags.ranked)
        idx = ops.index_map(indices, tags.count, tags.pm.device).idx
        n = int(idx.numel())
        pm = torch.empty((n, *tags.pm.shape[1:]), device=tags.pm.device, dtype=torch.int64)
        pp = torch.empty((n, *tags.pp.shape[1:]), device=tags.pp.device, dtype=torch.uint8)
        ops.rows_gather(tags.pm, idx, pm)
        ops.rows_gather(tags.pp, idx, pp)
        return DtkpTags(pm, pp, tags.registry, ranked=tags.ranked)

    def conj(self, a: DtkpTags, b: DtkpTags) -> DtkpTags:
        """All row pairs OR-ed, dedup + top-k (provenance.py:328-341)."""
        self._check_registry(a, b)
        B = max(a.batch, b.batch)
        return self._run(a.registry, _IDPLANS.conj_plan(a.count), [_bcast_dtkp(a, B), _bcast_dtkp(b, B)], None, 2, B,
                         a.ranked and b.ranked)

    def disj(self, a: DtkpTags, b: DtkpTags) -> DtkpTags:
        """Rows of a then rows of b, dedup + top-k (provenance.py:343-350)."""
        self._check_registry(a, b)
        B = max(a.batch, b.batch)
        return self._run(a.registry, _IDPLANS.disj_plan(a.count), [_bcast_dtkp(a, B)], _bcast_dtkp(b, B), 1, B,
                         a.ranked and b.ranked)

    def group_disj(self, tags: DtkpTags, groups) -> DtkpTags:
        kp = _group_plan(groups, tags.count)
        B = tags.batch
        return self._run(tags.registry, kp, [_bcast_dtkp(tags, B)], None, 1, B, tags.ranked)

    def concat_syms(self, parts) -> DtkpTags:
        registry = parts[0].registry
        B = max(p.batch for p in parts)
        for p in parts:
            p.aligned()
        pms, pps = zip(*(_bcast_dtkp(p, B) for p in parts))
        return DtkpTags(torch.cat(pms, dim=0), torch.cat(pps, dim=0), registry, ranked=all(p.ranked for p in parts))

    def probs(self, tags: DtkpTags) -> torch.Tensor:
        """Differentiable add-mult probability of every tag, (B, n) (provenance.py:398-413)."""
        p = tags.registry.prob_tensor()
        B = max(tags.batch, p.shape[1])
        pm, pp = _bcast_dtkp(tags, B)
        # the kernels read p as contiguous [I][B]: a batch-1 registry (e.g. stack() of
        # per-sample parts) is materialised, and torch sums its gradient back over b
        p = ops.expand_batch(p, B).contiguous()
        return ops.DtkpProbs.apply(pm, pp, p).t()

    def forward_probs(self, tags: DtkpTags) -> np.ndarray:
        p = tags.registry.prob_values()
        B = max(tags.batch, p.shape[1])
        pm, pp = _bcast_dtkp(tags, B)
        with torch.no_grad():
            out = ops.DtkpProbs.apply(pm, pp, ops.expand_batch(p, B).contiguous())
        return out.t().double().cpu().numpy()

    def placed(self, tags: DtkpTags, placement: np.ndarray) -> DtkpTags:
        src = _placement_src(placement)
        idx = ops.index_map(src, tags.count, tags.pm.device).idx
        n = len(src)
        pm = torch.empty((n, *tags.pm.shape[1:]), device=tags.pm.device, dtype=torch.int64)
        pp = torch.empty((n, *tags.pp.shape[1:]), device=tags.pp.device, dtype=torch.uint8)
        ops.rows_gather(tags.pm, idx, pm)
        ops.rows_gather(tags.pp, idx, pp)
        return DtkpTags(pm, pp, tags.registry, ranked=tags.ranked)

    def stack_parts(self, parts) -> DtkpTags:
        registry = parts[0].registry
        for p in parts:
            p.aligned()
        return DtkpTags(torch.cat([p.pm for p in parts], dim=3), torch.cat([p.pp for p in parts], dim=2), registry,
                        ranked=all(p.ranked for p in parts))

    def tags_from_proofs(self, registry, proofs, b: int = 1) -> DtkpTags:
        """Single-symbol tag from explicit proof index sets, normalised like the operators."""
        proofs = list(proofs)
        width = registry.size
        rows = max(len(proofs), 1)
        member = np.zeros((b, rows, width), dtype=np.uint8)
        present = np.zeros((b, rows), dtype=np.uint8)
        for r, proof in enumerate(proofs):
            for j in proof:
                member[:, r, j] = 1
            present[:, r] = 1
        dev = registry._dev()
        pv = self._p(registry, b).t().double().contiguous()
        om, op = ops.dedup_topk(torch.as_tensor(member, device=dev), torch.as_tensor(present, device=dev), pv,
                                self.k)
        return DtkpTags(om.cpu().numpy()[:, None], op.cpu().numpy()[:, None], registry, ranked=True)

    # ---- fused entry points ---------------------------------------------------------
    # the fused conj -> group_disj launch is exact (tests/test_gpu_fused.py) but, as built,
    # slower than the two launches on HWF-7 (1.77 ms vs 1.45 ms, profiles/r02_dtkp_launches.md):
    # opt in with SG_DTKP_FUSE=1
    fuse_conj_group = os.environ.get("SG_DTKP_FUSE", "0") == "1"

    def apply_plan(self, tags_list, plan: SymbolPlan, batch: int) -> DtkpTags:
        """K3/K4: gather -> conj fold -> group_disj as one streaming top-k kernel.

        A binary apply is left pending; an arity-1 apply over a pending binary apply (HWF's
        eval over its last concat step) runs both as ONE fused kernel (conj ->
        group_disj), so the intermediate tag (208767 symbols at HWF-7) never reaches HBM."""
        registry = tags_list[0].registry
        kp = plan.kernel_plan()
        if self.fuse_conj_group and len(tags_list) == 1:
            src = tags_list[0]
            pend = src.pending
            if pend is not None and pend.registry is registry and pend.B == batch and pend.K == self.k:
                return self._run_fused(kp, pend, batch)
        ops_ = [_bcast_dtkp(t, batch) for t in tags_list]
        if self.fuse_conj_group and len(tags_list) == 2:
            p = self._p(registry, batch)
            return DtkpTags(None, None, registry, pending=_PendingConj(self, registry, kp, ops_, batch, p))
        return self._run(registry, kp, ops_, None, len(tags_list), batch, all(t.ranked for t in tags_list))

    def _run_fused(self, kp: KernelPlan, pend: "_PendingConj", B: int) -> DtkpTags:
        dseg, dmerge, dmerge2 = kp.device(pend.p.device).dtkp_fused(pend.kp)
        pm, pp = ops.dtkp_apply(kp, dseg, dmerge, [], None, self.k, pend.W, pend.I, B, pend.p, 1, dmerge2,
                                inner=(pend.kp, pend.operands))
        return DtkpTags(pm, pp, pend.registry)

    def union_tags(self, a: DtkpTags, b: DtkpTags, uplan) -> DtkpTags:
        B = max(a.batch, b.batch)
        return self._run(a.registry, uplan.kplan, [_bcast_dtkp(a, B)], _bcast_dtkp(b, B), 1, B, a.ranked and b.ranked)


def wmc_exact(proofs, weights) -> float:
    """Exact weighted model count of a proof set (test oracle, provenance.py:460-501)."""
    if isinstance(weights, InputRegistry):
        weights = weights.prob_values()[:, 0].double().cpu().numpy()
    w = np.asarray(weights, dtype=np.float64).ravel()
    n = w.size
    if n > 20:
        raise ProvenanceError(f"wmc_exact enumerates 2^|I| assignments; |I|={n} exceeds the guard of 20")
    proofs = [frozenset(p) for p in proofs]
    if not proofs:
        return 0.0
    for proof in proofs:
        for j in proof:
            if not 0 <= j < n:
                raise ProvenanceError(f"proof index {j} outside universe of {n}")
    involved = sorted(set().union(*proofs))
    pos = {j: i for i, j in enumerate(involved)}
    m = len(involved)
    assign = np.arange(1 << m, dtype=np.int64)
    sat = np.zeros(assign.size, dtype=bool)
    for proof in proofs:
        mask = sum(1 << pos[j] for j in proof)
        sat |= (assign & mask) == mask
    weight = np.ones(assign.size)
    for i, j in enumerate(involved):
        weight *= np.where((assign >> i) & 1, w[j], 1.0 - w[j])
    return float(weight[sat].sum())


def provenance_from_name(name: str, k: int = 1):
    if name == "damp":
        return Damp()
    if name == "dtkp":
        return DtkpAm(k)
    if name in ("max", "damp-max"):
        return DampMax()
    raise ProvenanceError(f"unknown provenance {name!r} (expected damp, dtkp or max)")
