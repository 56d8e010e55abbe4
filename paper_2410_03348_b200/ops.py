"""torch.autograd bindings of the C-ABI kernels (the thin layer between tags and CUDA).

Every function here runs on the current CUDA stream of the tensors' device and calls
into ``libsgb200.so``; there is no eager or CPU fallback.  DAMP tensors are symbol-major
``[rows][B]`` fp32; DTKP tags are ``member int64 [rows][K][W][B]`` (bit patterns of u64)
plus ``present uint8 [rows][K][B]``.

Gradient conventions follow the reference tape (tensor.py):
  * clamp backward is the identity everywhere (tensor.py:275-287) — the DAMP apply and
    disjunction backward pass ``g`` through unchanged;
  * reduce_prod backward is leave-one-out with the exact-zeros rule (tensor.py:302-318);
  * batch-1 operands broadcast and their gradient is summed over the batch
    (tensor.py:130-138) — done by expanding the operand before the kernel, so torch's
    expand-backward sums it.
"""

from __future__ import annotations

import ctypes
import functools

import numpy as np
import torch

from . import _native as N
from .plan import KernelPlan

F32 = torch.float32


def _lib():
    return N.load()


def _check_operand(t: torch.Tensor, what: str):
    N.require_cuda(t, what)
    if t.dtype != F32 or t.ndim != 2:
        raise N.NativeError(f"{what}: expected a float32 (rows, B) view, got {t.dtype} {tuple(t.shape)}")


# ------------------------------------------------------------------------ layout
class ToSymbolMajor(torch.autograd.Function):
    """(B, n) any float dtype/strides -> contiguous [n][B] fp32 (explicit re-layout)."""

    @staticmethod
    def forward(ctx, x: torch.Tensor):
        N.require_cuda(x, "probabilities")
        if x.dtype not in N.DTYPE_CODE:
            x = x.float()
        B, n = x.shape
        out = torch.empty((n, B), device=x.device, dtype=F32)
        rc = _lib().sg_to_symbol_major(x.data_ptr(), N.DTYPE_CODE[x.dtype], B, n, x.stride(0), x.stride(1),
                                       out.data_ptr(), N.stream_ptr(x.device))
        N.check(rc, "sg_to_symbol_major")
        ctx.in_dtype = x.dtype
        return out

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        g = g.contiguous().float()
        n, B = g.shape
        out = torch.empty((B, n), device=g.device, dtype=ctx.in_dtype)
        rc = _lib().sg_from_symbol_major(g.data_ptr(), B, n, out.data_ptr(), N.DTYPE_CODE[ctx.in_dtype], out.stride(0),
                                         out.stride(1), N.stream_ptr(g.device))
        N.check(rc, "sg_from_symbol_major")
        return out


def to_symbol_major(x: torch.Tensor) -> torch.Tensor:
    return ToSymbolMajor.apply(x)


def symbol_view(probs: torch.Tensor) -> torch.Tensor:
    """A user (B, n) block as the (n, B) operand view the kernels read in place (fp32)."""
    N.require_cuda(probs, "probabilities")
    if probs.dtype != F32:
        probs = probs.float()
    return probs.t()


def expand_batch(x: torch.Tensor, B: int) -> torch.Tensor:
    """(rows, 1) -> (rows, B) stride-0 view (torch sums the gradient back over the batch)."""
    if x.shape[1] == B:
        return x
    if x.shape[1] != 1:
        raise ValueError(f"cannot broadcast batch {x.shape[1]} to {B}")
    return x.expand(x.shape[0], B)


# ------------------------------------------------------------------------ DAMP apply
class DampApply(torch.autograd.Function):
    """K1/K2: fused gather -> conj fold -> group_disj (+clamp) and its backward."""

    @staticmethod
    def forward(ctx, kplan: KernelPlan, B: int, *inputs):
        dev = inputs[0].device
        for i, x in enumerate(inputs):
            _check_operand(x, f"apply input {i}")
        dplan = kplan.device(dev)
        out = torch.empty((kplan.n_out, B), device=dev, dtype=F32)
        st = N.stream_ptr(dev)
        ops_ = N.rows_array(inputs)
        if kplan.clamp:
            s = dplan.damp_struct(B)
            scratch = None
            if kplan.conv == 3:  # the unclamped a (*) b of a three-way sum
                scratch = torch.empty((kplan.sizes[0] + kplan.sizes[1] - 1, B), device=dev, dtype=F32)
            elif not kplan.conv and s.fwd.n_partial:
                scratch = torch.empty((s.fwd.n_partial, B), device=dev, dtype=F32)
            rc = _lib().sg_damp_apply_fwd(ctypes.byref(s), ops_, B, out.data_ptr(), N.ptr(scratch), st)
            N.check(rc, "sg_damp_apply_fwd")
        else:
            seg = dplan.fwd().struct(B)
            scratch = torch.empty((seg.n_partial, B), device=dev, dtype=F32) if seg.n_partial else None
            rows = (ctypes.c_int32 * N.MAX_ARITY)(*kplan.sizes)
            rc = _lib().sg_segsum_run(ctypes.byref(seg), ops_, rows, kplan.arity, B, 0, N.rows(out), N.ptr(scratch), st)
            N.check(rc, "sg_segsum_run")
        _ledger("damp_apply_fwd", 4 * B * (sum(kplan.sizes) + kplan.n_out) + 4 * kplan.n_rec * kplan.arity,
                B * kplan.n_rec)
        ctx.kplan = kplan
        ctx.B = B
        ctx.save_for_backward(*inputs)
        return out

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        inputs = ctx.saved_tensors
        kplan: KernelPlan = ctx.kplan
        B = ctx.B
        if kplan.conv == 1 and not conv_staged(kplan):  # the unstaged kernel reads contiguous rows
            g = g.contiguous()
        dev = g.device
        need = [i for i in range(len(inputs)) if ctx.needs_input_grad[2 + i]]
        grads = [None] * len(inputs)
        if need:
            dplan = kplan.device(dev)
            alloc = range(2) if kplan.conv == 1 else need  # the short-filter Toeplitz backward writes both
            for i in alloc:
                grads[i] = torch.empty_like(inputs[i])
            s = dplan.damp_struct(B, need_bwd=() if kplan.conv else need)
            n_partial = 0 if kplan.conv else max((s.bwd[i].n_partial for i in need), default=0)
            if kplan.conv == 3:
                n_partial = 2 * (kplan.sizes[0] + kplan.sizes[1] - 1)
            scratch = torch.empty((n_partial, B), device=dev, dtype=F32) if n_partial else None
            rc = _lib().sg_damp_apply_bwd(ctypes.byref(s), N.rows_array(inputs), N.rows(g), B,
                                          N.rows_array(grads), N.ptr(scratch), N.stream_ptr(dev))
            N.check(rc, "sg_damp_apply_bwd")
            _ledger("damp_apply_bwd", 4 * B * (kplan.n_out + sum(2 * kplan.sizes[i] for i in need))
                    + 4 * kplan.n_rec * kplan.arity, B * kplan.n_rec)
            if kplan.conv:
                grads = [gr if ctx.needs_input_grad[2 + i] else None for i, gr in enumerate(grads)]
        return (None, None, *grads)


def conv_staged(kplan: KernelPlan) -> bool:
    """Whether the short-filter Toeplitz backward reads the upstream gradient in place."""
    sh = kplan.conv_short
    return _conv_staged(kplan.sizes[sh], kplan.sizes[1 - sh], kplan.n_out)


@functools.lru_cache(maxsize=4096)
def _conv_staged(kf: int, n_long: int, n_out: int) -> bool:
    return bool(_lib().sg_damp_conv_staged(kf, n_long, n_out))


class MaxProdApply(torch.autograd.Function):
    """Max-product apply (the north star's max variant): per output the max over its
    records of the product of the inputs, gradient to the first maximal record
    (tensor.py:319-325); sg_maxprod_fwd / sg_maxprod_bwd."""

    @staticmethod
    def forward(ctx, kplan: KernelPlan, B: int, *inputs):
        dev = inputs[0].device
        for i, x in enumerate(inputs):
            _check_operand(x, f"max apply input {i}")
        s = kplan.device(dev).maxprod_struct()
        out = torch.empty((kplan.n_out, B), device=dev, dtype=F32)
        arg = torch.empty((kplan.n_out, B), device=dev, dtype=torch.int32)
        rc = _lib().sg_maxprod_fwd(ctypes.byref(s), N.rows_array(inputs), B, int(kplan.clamp), N.ptr(out),
                                   N.ptr(arg), N.stream_ptr(dev))
        N.check(rc, "sg_maxprod_fwd")
        _ledger("maxprod_fwd", 4 * B * (sum(kplan.sizes) + 2 * kplan.n_out) + 4 * kplan.n_rec * (kplan.arity + 1),
                B * kplan.n_rec)
        ctx.kplan = kplan
        ctx.B = B
        ctx.save_for_backward(arg, *inputs)
        ctx.mark_non_differentiable(arg)
        return out

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        arg, *inputs = ctx.saved_tensors
        kplan: KernelPlan = ctx.kplan
        grads = [torch.empty_like(x) if ctx.needs_input_grad[2 + i] else None for i, x in enumerate(inputs)]
        if any(gr is not None for gr in grads):
            dev = g.device
            s = kplan.device(dev).maxprod_struct()
            rc = _lib().sg_maxprod_bwd(ctypes.byref(s), N.rows_array(inputs), ctx.B, N.ptr(arg), N.rows(g),
                                       N.rows_array(grads), N.stream_ptr(dev))
            N.check(rc, "sg_maxprod_bwd")
            _ledger("maxprod_bwd", 4 * ctx.B * (2 * kplan.n_out + sum(2 * n for n in kplan.sizes))
                    + 4 * kplan.n_rec * (kplan.arity + 2), ctx.B * kplan.n_rec)
        return (None, None, *grads)


def maxprod_apply(kplan: KernelPlan, inputs, B: int) -> torch.Tensor:
    inputs = [expand_batch(x, B) for x in inputs]
    return MaxProdApply.apply(kplan, B, *inputs)


def damp_apply(kplan: KernelPlan, inputs, B: int) -> torch.Tensor:
    inputs = [expand_batch(x, B) for x in inputs]
    return DampApply.apply(kplan, B, *inputs)


# Opt-in algorithmic-traffic ledger (bench.py): while ALG_BYTES is a list, every launch
# below appends (kernel, compulsory HBM bytes, work units) with the SURVEY §8(d) formulas
# evaluated on the launch's shapes — inputs read once, outputs written once, plan tables
# read once per launch — so a step's roofline fraction is sum(bytes) / step time.
ALG_BYTES = None


def _ledger(kernel: str, nbytes: int, units: int = 0):
    if ALG_BYTES is not None:
        ALG_BYTES.append((kernel, int(nbytes), int(units)))


# Opt-in per-launch CUDA-event timers (bench.py): while LAUNCH_TIMERS is a dict, the
# launches below are bracketed by timing events on their stream — also inside a CUDA-graph
# capture, where they become event-record nodes replayed with the step.
LAUNCH_TIMERS = None


class launch_timer:
    __slots__ = ("name", "e0")

    def __init__(self, name):
        self.name = name
        self.e0 = None

    def __enter__(self):
        if LAUNCH_TIMERS is not None:
            self.e0 = torch.cuda.Event(enable_timing=True, external=True)
            self.e0.record()
        return self

    def __exit__(self, *exc):
        if self.e0 is not None:
            e1 = torch.cuda.Event(enable_timing=True, external=True)  # a timing node when captured
            e1.record()
            LAUNCH_TIMERS.setdefault(self.name, []).append((self.e0, e1))
        return False


@functools.lru_cache(maxsize=None)
def chain_max_rows(kf: int) -> int:
    return int(_lib().sg_chain_max_rows(kf))


class ConvChainFn(torch.autograd.Function):
    """A left fold of Toeplitz applies v_i = clamp01(v_{i-1} (*) S_i) as one fused forward
    and one fused backward launch (csrc/chain.cu); identical per-step arithmetic to
    DampApply on the Toeplitz path."""

    @staticmethod
    def forward(ctx, n0: int, kf: int, B: int, base, *filters):
        m = len(filters)
        dev = base.device
        _check_operand(base, "chain base")
        for f in filters:
            _check_operand(f, "chain filter")
        elems = int(_lib().sg_chain_states_elems(n0, kf, m, B))
        states = torch.empty((max(elems, 1),), device=dev, dtype=F32)
        out = torch.empty((n0 + m * (kf - 1), B), device=dev, dtype=F32)
        c = _chain_struct(n0, kf, B, base, filters, states)
        rowsum = torch.empty((B,), device=dev, dtype=torch.float64)
        with launch_timer("chain_fwd"):
            rc = _lib().sg_chain_fwd(ctypes.byref(c), out.data_ptr(), rowsum.data_ptr(), N.stream_ptr(dev))
        N.check(rc, "sg_chain_fwd")
        # what a directly following loss_nll needs to fuse its backward into the chain's
        # (ChainNllLoss): the chain operands and the forward's per-sample row sums
        out._sg_chain = (n0, kf, B, base, tuple(filters), states, rowsum, out._version)
        _ledger("chain_fwd", 4 * B * (n0 + m * kf + (elems // B if B else 0) + out.shape[0]) + 8 * B,
                B * sum((n0 + i * (kf - 1)) * kf for i in range(m)))
        out._sg_rowsum = (rowsum, out._version)  # for loss_nll on exactly these values
        ctx.meta = (n0, kf, B)
        ctx.save_for_backward(base, states, *filters)
        return out

    @staticmethod
    def backward(ctx, g):
        base, states, *filters = ctx.saved_tensors
        n0, kf, B = ctx.meta
        g = g.contiguous()
        gbase = torch.empty_like(base)
        gfilt = [torch.empty_like(f) for f in filters]
        c = _chain_struct(n0, kf, B, base, filters, states)
        arr = (N.SgRows * N.CHAIN_MAX_STEPS)()
        for i, t in enumerate(gfilt):
            arr[i] = N.rows(t)
        with launch_timer("chain_bwd"):
            rc = _lib().sg_chain_bwd(ctypes.byref(c), g.data_ptr(), N.rows(gbase), arr, N.stream_ptr(g.device))
        N.check(rc, "sg_chain_bwd")
        m = len(filters)
        _ledger("chain_bwd", 4 * B * (g.shape[0] + 2 * m * kf + states.numel() // max(B, 1) + 2 * n0),
                B * sum((n0 + i * (kf - 1)) * kf for i in range(m)))
        return (None, None, None, gbase, *gfilt)


@functools.lru_cache(maxsize=None)
def maxchain_max_rows(kf: int) -> int:
    return int(_lib().sg_maxchain_max_rows(kf))


class MaxChainFn(torch.autograd.Function):
    """The max/DAMP variant of ConvChainFn: a left fold of max-product Toeplitz applies in
    one forward and one backward launch (csrc/maxchain.cu), per step bit-identical to
    MaxProdApply (first-argmax gradient, pass-through clamp)."""

    @staticmethod
    def forward(ctx, n0: int, kf: int, B: int, base, *filters):
        m = len(filters)
        dev = base.device
        _check_operand(base, "max chain base")
        for f in filters:
            _check_operand(f, "max chain filter")
        states = torch.empty((max(int(_lib().sg_maxchain_states_elems(n0, kf, m, B)), 1),), device=dev, dtype=F32)
        argmax = torch.empty((max(int(_lib().sg_maxchain_argmax_bytes(n0, kf, m, B)), 1),), device=dev,
                             dtype=torch.uint8)
        out = torch.empty((n0 + m * (kf - 1), B), device=dev, dtype=F32)
        rowsum = torch.empty((B,), device=dev, dtype=torch.float64)
        c = _chain_struct(n0, kf, B, base, filters, states)
        with launch_timer("maxchain_fwd"):
            rc = _lib().sg_maxchain_fwd(ctypes.byref(c), out.data_ptr(), rowsum.data_ptr(), argmax.data_ptr(),
                                        N.stream_ptr(dev))
        N.check(rc, "sg_maxchain_fwd")
        _ledger("maxchain_fwd", 4 * B * (n0 + m * kf + states.numel() // max(B, 1) + out.shape[0]) + argmax.numel()
                + 8 * B, B * sum((n0 + i * (kf - 1)) * kf for i in range(m)))
        out._sg_rowsum = (rowsum, out._version)
        ctx.meta = (n0, kf, B)
        ctx.save_for_backward(base, states, argmax, *filters)
        return out

    @staticmethod
    def backward(ctx, g):
        base, states, argmax, *filters = ctx.saved_tensors
        n0, kf, B = ctx.meta
        g = g.contiguous()
        gbase = torch.empty_like(base)
        gfilt = [torch.empty_like(f) for f in filters]
        c = _chain_struct(n0, kf, B, base, filters, states)
        arr = (N.SgRows * N.CHAIN_MAX_STEPS)()
        for i, t in enumerate(gfilt):
            arr[i] = N.rows(t)
        with launch_timer("maxchain_bwd"):
            rc = _lib().sg_maxchain_bwd(ctypes.byref(c), argmax.data_ptr(), g.data_ptr(), N.rows(gbase), arr,
                                        N.stream_ptr(g.device))
        N.check(rc, "sg_maxchain_bwd")
        m = len(filters)
        _ledger("maxchain_bwd", 4 * B * (g.shape[0] + 2 * m * kf + states.numel() // max(B, 1) + 2 * n0)
                + argmax.numel(), B * sum((n0 + i * (kf - 1)) * kf for i in range(m)))
        return (None, None, None, gbase, *gfilt)


FUSE_CHAIN_NLL = True  # loss_nll directly on a fused chain's output: one fused backward


def known_chain(probs_nb: torch.Tensor):
    """The chain operands behind ``probs_nb`` if it is exactly a fused chain's (unmodified)
    output, else None."""
    base = probs_nb._base if probs_nb._base is not None else probs_nb
    tag = getattr(base, "_sg_chain", None)
    if tag is None or not FUSE_CHAIN_NLL:
        return None
    if (base._version != tag[-1] or probs_nb.data_ptr() != base.data_ptr() or probs_nb.shape != base.shape
            or probs_nb.stride() != base.stride()):
        return None
    return tag


class ChainNllLoss(torch.autograd.Function):
    """loss_nll (learn.py:92-119) of a fused Sum-N chain's output as ONE autograd node over
    the chain's operands: the forward reuses the chain forward's output and row sums
    (sg_nll_fwd_rowsum), the backward is a single sg_chain_bwd_nll launch whose upstream
    gradient rows are generated inside the kernel (bit-identical to sg_nll_bwd's), so the
    [n_out][B] loss gradient never exists.  The chain's own autograd node stays valid for
    any other use of the probabilities."""

    @staticmethod
    def forward(ctx, meta, probs_nb, targets, base, *filters):
        n0, kf, B, states, rowsum = meta
        n = probs_nb.shape[0]
        dev = probs_nb.device
        loss = torch.empty((), device=dev, dtype=torch.float64)
        scratch = _nll_scratch(dev, n, B)
        picked = torch.empty((B,), device=dev, dtype=torch.float64)
        rc = _lib().sg_nll_fwd_rowsum(N.rows(probs_nb), n, B, targets.data_ptr(), rowsum.data_ptr(), loss.data_ptr(),
                                      scratch.data_ptr(), picked.data_ptr(), N.stream_ptr(dev))
        N.check(rc, "sg_nll_fwd_rowsum")
        _ledger("nll_fwd", 4 * B + 24 * B, B * n)
        ctx.meta = (n0, kf, B)
        ctx.save_for_backward(targets, rowsum, picked, base, states, *filters)
        return loss

    @staticmethod
    def backward(ctx, gloss):
        targets, rowsum, picked, base, states, *filters = ctx.saved_tensors
        n0, kf, B = ctx.meta
        g = gloss.detach().to(torch.float64).reshape(()).contiguous()
        gbase = torch.empty_like(base)
        gfilt = [torch.empty_like(f) for f in filters]
        c = _chain_struct(n0, kf, B, base, filters, states)
        arr = (N.SgRows * N.CHAIN_MAX_STEPS)()
        for i, t in enumerate(gfilt):
            arr[i] = N.rows(t)
        with launch_timer("chain_bwd"):
            rc = _lib().sg_chain_bwd_nll(ctypes.byref(c), targets.data_ptr(), rowsum.data_ptr(), picked.data_ptr(),
                                         g.data_ptr(), N.rows(gbase), arr, N.stream_ptr(g.device))
        N.check(rc, "sg_chain_bwd_nll")
        m = len(filters)
        _ledger("chain_bwd", 4 * B * (2 * m * kf + states.numel() // max(B, 1) + 2 * n0) + 24 * B,
                B * sum((n0 + i * (kf - 1)) * kf for i in range(m)))
        return (None, None, None, gbase, *gfilt)


def _chain_struct(n0, kf, B, base, filters, states) -> N.SgChain:
    c = N.SgChain()
    c.base = N.rows(base)
    c.n0 = n0
    c.kf = kf
    c.m = len(filters)
    c.B = B
    for i, f in enumerate(filters):
        c.filters[i] = N.rows(f)
    c.states = states.data_ptr()
    return c


class _IndexMap:
    """Host index list -> device index tensor + the scatter-sum plan of its backward."""

    __slots__ = ("idx", "bwd", "n_src")

    def __init__(self, indices: np.ndarray, n_src: int, device):
        indices = np.asarray(indices, dtype=np.int32).reshape(-1)
        self.n_src = int(n_src)
        self.idx = torch.as_tensor(indices, device=device)
        keep = indices >= 0
        rec = np.nonzero(keep)[0].astype(np.int32).reshape(-1, 1)
        # backward: grad_src[s] = sum_{r: idx[r] == s} g[r]  (select_rows bw, tensor.py:386-391)
        self.bwd = KernelPlan(rec, indices[keep], self.n_src, (len(indices),), clamp=False)


_MAP_CACHE: "dict[tuple, _IndexMap]" = {}
_GATHER_CACHE: "dict[tuple, KernelPlan]" = {}


def index_map(indices, n_src: int, device) -> _IndexMap:
    arr = np.asarray(indices, dtype=np.int32).reshape(-1)
    key = (torch.device(device), int(n_src), arr.tobytes())
    m = _MAP_CACHE.get(key)
    if m is None:
        if len(_MAP_CACHE) > 4096:
            _MAP_CACHE.clear()
        m = _IndexMap(arr, n_src, device)
        _MAP_CACHE[key] = m
    return m


def gather_plan(indices, n_src: int) -> KernelPlan:
    """out[r] = src[idx[r]] (0 for idx -1) as an arity-1 segmented plan (backward: scatter-add)."""
    arr = np.asarray(indices, dtype=np.int32).reshape(-1)
    key = (int(n_src), arr.tobytes())
    kp = _GATHER_CACHE.get(key)
    if kp is None:
        if len(_GATHER_CACHE) > 4096:
            _GATHER_CACHE.clear()
        keep = np.nonzero(arr >= 0)[0].astype(np.int32)
        kp = KernelPlan(arr[keep].reshape(-1, 1), keep, len(arr), (int(n_src),), clamp=False)
        _GATHER_CACHE[key] = kp
    return kp


def scatter_rows_sum(g: torch.Tensor, imap: _IndexMap) -> torch.Tensor:
    return DampApply.apply(imap.bwd, g.shape[1], g.contiguous())


class DampRowsAdd(torch.autograd.Function):
    """out[r] = clamp01(A[ia[r]] + Bm[ib[r]]) — Damp.disj / union; clamp bw = identity."""

    @staticmethod
    def forward(ctx, A, Bm, ma: _IndexMap, mb: _IndexMap, clamp: bool):
        _check_operand(A, "disj lhs")
        _check_operand(Bm, "disj rhs")
        B = max(A.shape[1], Bm.shape[1])
        n = int(ma.idx.numel())
        out = torch.empty((n, B), device=A.device, dtype=F32)
        rc = _lib().sg_damp_rows_add(N.rows(A), ma.idx.data_ptr(), N.rows(Bm), mb.idx.data_ptr(), n, B,
                                     1 if clamp else 0, out.data_ptr(), N.stream_ptr(A.device))
        N.check(rc, "sg_damp_rows_add")
        _ledger("damp_rows_add", 4 * B * (A.shape[0] + Bm.shape[0] + n), B * n)
        ctx.maps = (ma, mb)
        return out

    @staticmethod
    def backward(ctx, g):
        ma, mb = ctx.maps
        ga = scatter_rows_sum(g, ma) if ctx.needs_input_grad[0] else None
        gb = scatter_rows_sum(g, mb) if ctx.needs_input_grad[1] else None
        return ga, gb, None, None, None


_NLL_SCRATCH: "dict[tuple, torch.Tensor]" = {}
_NLL_RETIRED: "list[torch.Tensor]" = []  # outgrown scratch a captured graph may still use


def _nll_scratch(dev, n: int, B: int) -> torch.Tensor:
    """Per-device zero-initialised scratch; the kernel resets its counter itself, so the
    buffer is reused across calls, streams and CUDA-graph replays without a memset (a
    buffer first created during a capture would put its memset into the graph).  Losses
    on one device must not run concurrently on two streams."""
    key = dev
    nbytes = int(_lib().sg_nll_scratch_bytes(n, B))
    buf = _NLL_SCRATCH.get(key)
    if buf is None or buf.numel() < nbytes:
        if buf is not None:
            # a CUDA graph captured earlier may still hold this address (its ticket counter
            # and partials): keep the outgrown buffer alive, never recycle it
            _NLL_RETIRED.append(buf)
        # under CUDA-graph capture this allocates from the graph pool (memset captured once)
        buf = torch.zeros(max(nbytes, 4096), device=dev, dtype=torch.uint8)
        _NLL_SCRATCH[key] = buf
    return buf


def known_rowsum(probs_nb: torch.Tensor):
    """Per-sample row sums a fused chain forward wrote beside ``probs_nb``'s values, if
    ``probs_nb`` is exactly that output and unmodified since (else None)."""
    base = probs_nb._base if probs_nb._base is not None else probs_nb
    tag = getattr(base, "_sg_rowsum", None)
    if tag is None:
        return None
    rowsum, version = tag
    if (base._version != version or probs_nb.data_ptr() != base.data_ptr() or probs_nb.shape != base.shape
            or probs_nb.stride() != base.stride()):
        return None
    return rowsum


class NllLoss(torch.autograd.Function):
    """Fused get_probs -> loss_nll (learn.py:92-119) over an (n, B) probability view."""

    @staticmethod
    def forward(ctx, probs_nb: torch.Tensor, targets: torch.Tensor):
        _check_operand(probs_nb, "loss probabilities")
        n, B = probs_nb.shape
        dev = probs_nb.device
        loss = torch.empty((), device=dev, dtype=torch.float64)
        scratch = _nll_scratch(dev, n, B)
        rowsum = known_rowsum(probs_nb)
        if rowsum is not None:  # a fused chain forward already summed these rows
            rc = _lib().sg_nll_fwd_rowsum(N.rows(probs_nb), n, B, targets.data_ptr(), rowsum.data_ptr(),
                                          loss.data_ptr(), scratch.data_ptr(), None, N.stream_ptr(dev))
            N.check(rc, "sg_nll_fwd_rowsum")
        else:
            rowsum = torch.empty((B,), device=dev, dtype=torch.float64)
            rc = _lib().sg_nll_fwd(N.rows(probs_nb), n, B, targets.data_ptr(), loss.data_ptr(), scratch.data_ptr(),
                                   rowsum.data_ptr(), N.stream_ptr(dev))
            N.check(rc, "sg_nll_fwd")
        _ledger("nll_fwd", 4 * B * n + 16 * B, B * n)
        ctx.save_for_backward(probs_nb, targets, rowsum)
        return loss

    @staticmethod
    def backward(ctx, gloss):
        probs_nb, targets, rowsum = ctx.saved_tensors
        n, B = probs_nb.shape
        g = gloss.detach().to(torch.float64).reshape(()).contiguous()
        grad = torch.empty_like(probs_nb)
        rc = _lib().sg_nll_bwd(N.rows(probs_nb), n, B, targets.data_ptr(), g.data_ptr(), rowsum.data_ptr(),
                               N.rows(grad), N.stream_ptr(probs_nb.device))
        N.check(rc, "sg_nll_bwd")
        _ledger("nll_bwd", 8 * B * n + 16 * B, B * n)
        return grad, None


def rows_gather(src: torch.Tensor, idx: torch.Tensor, out: torch.Tensor):
    """Copy whole contiguous symbol rows (DTKP tags): out[r] = src[idx[r]] or zeros for -1."""
    n = int(idx.numel())
    if n == 0 or out.numel() == 0:
        return out
    row_bytes = out[0].numel() * out.element_size()
    rc = _lib().sg_rows_gather(src.data_ptr() if src.numel() else None, idx.data_ptr(), n, row_bytes, out.data_ptr(),
                               N.stream_ptr(out.device))
    N.check(rc, "sg_rows_gather")
    _ledger("rows_gather", 2 * n * row_bytes, n)
    return out


def index_tensor(indices, device) -> torch.Tensor:
    return torch.as_tensor(np.asarray(indices, dtype=np.int32).reshape(-1), device=device)


# ------------------------------------------------------------------------ DTKP
_SCHED: "dict[tuple, torch.Tensor]" = {}
_SCHED_RETIRED: "list[torch.Tensor]" = []  # outgrown buffers a captured graph may still use
DTKP_DYNAMIC = True  # False: the static block partition (sched = NULL), kept for tests
DTKP_RANKED = True   # False: never use the ranked-rows early exit (A/B tests)


def dtkp_sched(device, n: int) -> torch.Tensor:
    """Zeroed work counters for sg_dtkp_apply's dynamic item schedule, one buffer per
    (device, stream): launches on one stream are ordered, and every launch leaves the
    counters zero again.  A buffer first made during CUDA-graph capture is zeroed by a
    captured memset, which is harmless on replay."""
    key = (torch.device(device), N.stream_ptr(device))
    t = _SCHED.get(key)
    if t is None or t.numel() < n:
        if t is not None:
            _SCHED_RETIRED.append(t)
        t = torch.zeros(max(n, 64), device=device, dtype=torch.int32)
        _SCHED[key] = t
    return t


def dtkp_apply(kplan_host, dseg, dmerge, operands, tail, K: int, W: int, I: int, B: int, p: torch.Tensor,
               arity: int, dmerge2=None, inner=None, ranked: bool = True):
    """Run sg_dtkp_apply; operands are (member, present) pairs with full batch B.
    ``inner`` = (inner_plan, [(member, present)] * 2) runs the fused conj -> group_disj
    (``dseg`` from DevicePlan.dtkp_fused): operand 0 is the never-materialised output of
    the binary apply ``inner_plan`` over those operands (``operands`` is then empty)."""
    dev = p.device
    n_out = dseg.host.n_seg
    out_m = torch.empty((n_out, K, W, B), device=dev, dtype=torch.int64)
    out_p = torch.empty((n_out, K, B), device=dev, dtype=torch.uint8)
    d = N.SgDtkpApplyDesc()
    d.arity = arity
    d.K = K
    d.W = W
    d.I = I
    d.B = B
    for i, (m, pr) in enumerate(operands):
        d.ops[i].member = m.data_ptr() if m.numel() else None
        d.ops[i].present = pr.data_ptr() if pr.numel() else None
        d.ops[i].rows = m.shape[0]
        d.ops[i].W = m.shape[2]
    if tail is not None:
        m, pr = tail
        d.op_tail.member = m.data_ptr() if m.numel() else None
        d.op_tail.present = pr.data_ptr() if pr.numel() else None
        d.op_tail.rows = m.shape[0]
        d.op_tail.W = m.shape[2]
    if inner is not None:
        ikp, iops = inner
        d.inner_arity = 2
        for i, (m, pr) in enumerate(iops):
            d.inner_ops[i].member = m.data_ptr() if m.numel() else None
            d.inner_ops[i].present = pr.data_ptr() if pr.numel() else None
            d.inner_ops[i].rows = m.shape[0]
            d.inner_ops[i].W = m.shape[2]
        d.ops[0].rows = ikp.n_out
        d.ops[0].W = W
    d.p = p.data_ptr() if p.numel() else None
    d.seg = dseg.struct(B)
    d.seg_packed = 1 if getattr(dseg.host, "packed", False) else 0
    d.rows_ranked = 1 if ranked else 0
    d.out_member = out_m.data_ptr() if out_m.numel() else None
    d.out_present = out_p.data_ptr() if out_p.numel() else None
    scr_m = scr_p = None
    if dseg.host.n_partial:
        scr_m = torch.empty((dseg.host.n_partial, K, W, B), device=dev, dtype=torch.int64)
        scr_p = torch.empty((dseg.host.n_partial, K, B), device=dev, dtype=torch.uint8)
        d.scratch_member = scr_m.data_ptr()
        d.scratch_present = scr_p.data_ptr()
        d.merge = dmerge.struct(B)
        if dmerge.host.n_partial:
            scr2_m = torch.empty((dmerge.host.n_partial, K, W, B), device=dev, dtype=torch.int64)
            scr2_p = torch.empty((dmerge.host.n_partial, K, B), device=dev, dtype=torch.uint8)
            d.scratch2_member = scr2_m.data_ptr()
            d.scratch2_present = scr2_p.data_ptr()
            d.merge2 = dmerge2.struct(B)
    d.sched = dtkp_sched(dev, -(-B // 32) + 1).data_ptr() if DTKP_DYNAMIC else None
    rc = _lib().sg_dtkp_apply(ctypes.byref(d), N.stream_ptr(dev))
    N.check(rc, "sg_dtkp_apply")
    if ALG_BYTES is not None:
        row = 8 * K * W + K  # one tag per sample: K rows of W words + K present bytes
        rows_in = sum(m.shape[0] for m, _ in operands) + (tail[0].shape[0] if tail is not None else 0)
        partial = dseg.host.n_partial + (dmerge.host.n_partial if dseg.host.n_partial else 0)
        n_rec = kplan_host.n_rec
        cand = n_rec * (K ** arity if arity >= 2 else K)  # candidate rows ranked (upper bound)
        if inner is not None:  # the inner conj's operands are read, its output never is
            rows_in = sum(m.shape[0] for m, _ in inner[1])
            n_rec += inner[0].n_rec * 2
            cand += inner[0].n_rec * K * K
        _ledger("dtkp_apply", B * (rows_in + n_out + 2 * partial) * row + 4 * B * I + 4 * n_rec * max(arity, 1),
                B * cand)
    return out_m, out_p


class DtkpProbs(torch.autograd.Function):
    """K5: clamp(sum_r present * prod_{j in r} p_j) and its leave-one-out backward."""

    @staticmethod
    def forward(ctx, member, present, p):
        Nn, K, W, B = member.shape
        I = p.shape[0]
        out = torch.empty((Nn, B), device=p.device, dtype=F32)
        rc = _lib().sg_dtkp_probs_fwd(member.data_ptr() if member.numel() else None,
                                      present.data_ptr() if present.numel() else None, Nn, K, W,
                                      p.data_ptr() if p.numel() else None, I, B, out.data_ptr() if out.numel() else None,
                                      N.stream_ptr(p.device))
        N.check(rc, "sg_dtkp_probs_fwd")
        _ledger("dtkp_probs_fwd", B * Nn * (8 * K * W + K) + 4 * B * I + 4 * B * Nn, B * Nn * K)
        ctx.save_for_backward(member, present, p)
        return out

    @staticmethod
    def backward(ctx, g):
        member, present, p = ctx.saved_tensors
        Nn, K, W, B = member.shape
        I = p.shape[0]
        g = g.contiguous()
        gp = torch.empty_like(p)
        nbytes = int(_lib().sg_dtkp_probs_bwd_scratch(Nn, I, B))
        scratch = torch.empty(max(nbytes, 8), device=p.device, dtype=torch.uint8)
        rc = _lib().sg_dtkp_probs_bwd(member.data_ptr() if member.numel() else None,
                                      present.data_ptr() if present.numel() else None, Nn, K, W, p.data_ptr(), I, B,
                                      g.data_ptr() if g.numel() else None, gp.data_ptr(), scratch.data_ptr(),
                                      N.stream_ptr(p.device))
        N.check(rc, "sg_dtkp_probs_bwd")
        _ledger("dtkp_probs_bwd", B * Nn * (8 * K * W + K) + 8 * B * I + 4 * B * Nn, B * Nn * K)
        return None, None, gp


def dedup_topk(member: torch.Tensor, present: torch.Tensor, p: torch.Tensor, k: int):
    """Device drop-in for _dtkpcore.dedup_topk: u8 [M,R,I], u8 [M,R], f64 [M,I] -> u8 [M,k,I], u8 [M,k]."""
    M, R, I = member.shape
    member = member.contiguous().to(torch.uint8)
    present = present.contiguous().to(torch.uint8)
    p = p.contiguous().to(torch.float64)
    om = torch.empty((M, k, I), device=member.device, dtype=torch.uint8)
    op = torch.empty((M, k), device=member.device, dtype=torch.uint8)
    if M == 0 or k == 0:
        return om.zero_(), op.zero_()
    rc = _lib().sg_dedup_topk(member.data_ptr() if member.numel() else None,
                              present.data_ptr() if present.numel() else None, p.data_ptr() if p.numel() else None,
                              M, R, I, k, om.data_ptr() if om.numel() else None, op.data_ptr(),
                              N.stream_ptr(member.device))
    N.check(rc, "sg_dedup_topk")
    return om, op
