"""ctypes binding of the sm_100a C-ABI library ``libsgb200.so`` (see include/sgb200.h).

The library is loaded from the package directory (built in-tree by ``_build.py``).  There
is no fallback: if the library is missing or a call returns a CUDA error, a
``NativeError`` is raised.  All buffers passed in are device tensors owned by PyTorch's
caching allocator; work is enqueued on the current torch stream.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, c_double, c_int32, c_int64, c_void_p
from pathlib import Path

import torch

MAX_ARITY = 8
# SGB200_LIB: an alternative build of the same library (A/B measurements, tools/ab_build.py)
LIB_PATH = Path(os.environ.get("SGB200_LIB") or Path(__file__).resolve().parent / "libsgb200.so")


class NativeError(RuntimeError):
    """The CUDA library is missing or a kernel launch failed."""


class SgSegsum(Structure):
    _fields_ = [
        ("n_seg", c_int32),
        ("rec_words", c_int32),
        ("n_items", c_int32),
        ("n_blocks", c_int32),
        ("n_split", c_int32),
        ("n_partial", c_int32),
        ("staged", c_int32),
        ("n_recs", c_int32),
        ("recs", c_void_p),
        ("items", c_void_p),
        ("blk", c_void_p),
        ("split", c_void_p),
    ]


class SgRows(Structure):
    _fields_ = [("ptr", c_void_p), ("stride_row", c_int64), ("stride_b", c_int64)]


CHAIN_MAX_STEPS = 32


class SgChain(Structure):
    _fields_ = [
        ("base", SgRows),
        ("n0", c_int32),
        ("kf", c_int32),
        ("m", c_int32),
        ("pad_", c_int32),
        ("B", c_int64),
        ("filters", SgRows * CHAIN_MAX_STEPS),
        ("states", c_void_p),
    ]


class SgDampPlan(Structure):
    _fields_ = [
        ("arity", c_int32),
        ("n_out", c_int32),
        ("sizes", c_int32 * MAX_ARITY),
        ("conv", c_int32),
        ("conv_short", c_int32),
        ("fwd", SgSegsum),
        ("bwd", SgSegsum * MAX_ARITY),
    ]


class SgDtkpOperand(Structure):
    _fields_ = [
        ("member", c_void_p),
        ("present", c_void_p),
        ("rows", c_int32),
        ("W", c_int32),
    ]


class SgDtkpApplyDesc(Structure):
    _fields_ = [
        ("arity", c_int32),
        ("K", c_int32),
        ("W", c_int32),
        ("I", c_int32),
        ("B", c_int64),
        ("ops", SgDtkpOperand * MAX_ARITY),
        ("op_tail", SgDtkpOperand),
        ("p", c_void_p),
        ("seg", SgSegsum),
        ("out_member", c_void_p),
        ("out_present", c_void_p),
        ("scratch_member", c_void_p),
        ("scratch_present", c_void_p),
        ("merge", SgSegsum),
        ("sched", c_void_p),
        ("merge2", SgSegsum),
        ("scratch2_member", c_void_p),
        ("scratch2_present", c_void_p),
        ("inner_arity", c_int32),
        ("seg_packed", c_int32),
        ("inner_ops", SgDtkpOperand * 2),
        ("rows_ranked", c_int32),
        ("rows_ranked_pad_", c_int32),
    ]


class SgMaxprodPlan(Structure):
    _fields_ = [
        ("arity", c_int32),
        ("n_out", c_int32),
        ("n_recs", c_int32),
        ("sizes", c_int32 * MAX_ARITY),
        ("seg_off", c_void_p),
        ("recs", c_void_p),
        ("rec_out", c_void_p),
        ("in_off", c_void_p * MAX_ARITY),
        ("in_recs", c_void_p * MAX_ARITY),
    ]


# (name, restype, argtypes) of every exported entry point in include/sgb200.h
EXPORTS = {
    "sg_version": (c_int32, []),
    "sg_launch_count": (c_int64, []),
    "sg_device_sm_count": (c_int32, [c_int32]),
    "sg_to_symbol_major": (c_int32, [c_void_p, c_int32, c_int64, c_int64, c_int64, c_int64, c_void_p, c_void_p]),
    "sg_from_symbol_major": (c_int32, [c_void_p, c_int64, c_int64, c_void_p, c_int32, c_int64, c_int64, c_void_p]),
    "sg_segsum_run": (
        c_int32,
        [POINTER(SgSegsum), POINTER(SgRows), POINTER(c_int32), c_int32, c_int64, c_int32, SgRows, c_void_p, c_void_p],
    ),
    "sg_damp_apply_fwd": (c_int32, [POINTER(SgDampPlan), POINTER(SgRows), c_int64, c_void_p, c_void_p, c_void_p]),
    "sg_damp_apply_bwd": (
        c_int32,
        [POINTER(SgDampPlan), POINTER(SgRows), SgRows, c_int64, POINTER(SgRows), c_void_p, c_void_p],
    ),
    "sg_damp_rows_add": (
        c_int32,
        [SgRows, c_void_p, SgRows, c_void_p, c_int64, c_int64, c_int32, c_void_p, c_void_p],
    ),
    "sg_chain_states_elems": (c_int64, [c_int32, c_int32, c_int32, c_int64]),
    "sg_chain_max_rows": (c_int32, [c_int32]),
    "sg_chain_fwd": (c_int32, [POINTER(SgChain), c_void_p, c_void_p, c_void_p]),
    "sg_chain_bwd": (c_int32, [POINTER(SgChain), c_void_p, SgRows, POINTER(SgRows), c_void_p]),
    "sg_chain_bwd_nll": (c_int32, [POINTER(SgChain), c_void_p, c_void_p, c_void_p, c_void_p, SgRows,
                                   POINTER(SgRows), c_void_p]),
    "sg_damp_conv_staged": (c_int32, [c_int32, c_int32, c_int32]),
    "sg_maxchain_states_elems": (c_int64, [c_int32, c_int32, c_int32, c_int64]),
    "sg_maxchain_argmax_bytes": (c_int64, [c_int32, c_int32, c_int32, c_int64]),
    "sg_maxchain_max_rows": (c_int32, [c_int32]),
    "sg_maxchain_fwd": (c_int32, [POINTER(SgChain), c_void_p, c_void_p, c_void_p, c_void_p]),
    "sg_maxchain_bwd": (c_int32, [POINTER(SgChain), c_void_p, c_void_p, SgRows, POINTER(SgRows), c_void_p]),
    "sg_nll_scratch_bytes": (c_int64, [c_int64, c_int64]),
    "sg_nll_fwd": (c_int32, [SgRows, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "sg_nll_bwd": (c_int32, [SgRows, c_int64, c_int64, c_void_p, c_void_p, c_void_p, SgRows, c_void_p]),
    "sg_nll_fwd_rowsum": (c_int32, [SgRows, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                    c_void_p]),
    "sg_maxprod_fwd": (c_int32, [POINTER(SgMaxprodPlan), POINTER(SgRows), c_int64, c_int32, c_void_p, c_void_p,
                                 c_void_p]),
    "sg_maxprod_bwd": (c_int32, [POINTER(SgMaxprodPlan), POINTER(SgRows), c_int64, c_void_p, SgRows, POINTER(SgRows),
                                 c_void_p]),
    "sg_rows_gather": (c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "sg_dtkp_apply": (c_int32, [POINTER(SgDtkpApplyDesc), c_void_p]),
    "sg_dtkp_probs_fwd": (
        c_int32,
        [c_void_p, c_void_p, c_int32, c_int32, c_int32, c_void_p, c_int32, c_int64, c_void_p, c_void_p],
    ),
    "sg_dtkp_probs_bwd_scratch": (c_int64, [c_int32, c_int32, c_int64]),
    "sg_dtkp_probs_bwd": (
        c_int32,
        [c_void_p, c_void_p, c_int32, c_int32, c_int32, c_void_p, c_int32, c_int64, c_void_p, c_void_p, c_void_p,
         c_void_p],
    ),
    "sg_dedup_topk": (
        c_int32,
        [c_void_p, c_void_p, c_void_p, c_int64, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p],
    ),
}

_lib = None
class _Lib:
    def __init__(self, cdll):
        self._cdll = cdll
        for name in EXPORTS:
            setattr(self, name, getattr(cdll, name))


def launch_count() -> int:
    """Kernels the library has enqueued so far (sg_launch_count; a captured graph's
    kernels count once, at capture)."""
    return int(load().sg_launch_count())


def load() -> "_Lib":
    """Load (once) and return the library; raises NativeError when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2410_03348_b200._build` "
            "(there is no CPU fallback for the probabilistic hot path)"
        )
    lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_LOCAL | getattr(os, "RTLD_NOW", 2))
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = _Lib(lib)
    return _lib


_CUDA_ERR = {1: "cudaErrorInvalidValue", 2: "cudaErrorMemoryAllocation", 98: "cudaErrorInvalidDeviceFunction",
             209: "cudaErrorNoKernelImageForDevice", 801: "cudaErrorNotSupported"}


def check(rc: int, what: str):
    if rc != 0:
        raise NativeError(f"{what} failed with CUDA error {rc} ({_CUDA_ERR.get(rc, 'see cudaError_t')})")


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def rows(t) -> SgRows:
    """A (rows, B) float32 tensor view as an sg_rows operand (any strides; NULL for None)."""
    r = SgRows()
    if t is not None:
        r.ptr = t.data_ptr() if t.numel() else None
        r.stride_row = t.stride(0)
        r.stride_b = t.stride(1) if t.shape[1] > 1 else 0
    return r


def rows_array(tensors) -> ctypes.Array:
    arr = (SgRows * MAX_ARITY)()
    for i, t in enumerate(tensors):
        if t is not None:
            arr[i] = rows(t)
    return arr


def ptr_array(tensors) -> ctypes.Array:
    arr = (c_void_p * MAX_ARITY)()
    for i, t in enumerate(tensors):
        arr[i] = None if t is None else t.data_ptr()
    return arr


DTYPE_CODE = {torch.float32: 0, torch.float64: 1, torch.float16: 2, torch.bfloat16: 3}


def require_cuda(t: torch.Tensor, what: str = "tensor"):
    if not t.is_cuda:
        raise NativeError(f"{what} must live on a CUDA device (the hot path has no CPU implementation)")
