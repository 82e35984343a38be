"""Saturating lane kernels on 128-bit blocks -- drop-in for semimat.kernels.

Same functions, arguments, list-in/list-out contract and error messages as
the reference (pkg/src/semimat/kernels.py:41-204).  The lanes are computed by
the device kernel ``smx_lane_op`` (csrc/lanes.cu) with the same packed u16x2
instructions the semiring GEMM uses (u8 lanes widened into 16-bit lanes);
there is no numpy or pure-Python path.

Path selection: the reference picks numpy or pure Python per call
(``use_vector``, ``SEMIMAT_FORCE_SCALAR``, ``forced_scalar`` /
``forced_vector``, kernels.py:53-88) and guarantees the two are
bit-identical.  This package keeps those names and their state so code that
queries or pins a path still runs, but every call executes the device kernel
whichever path is pinned (no second backend).
"""

from __future__ import annotations

import os
import platform
from contextlib import contextmanager

import numpy as np
import torch

from . import _native
from .scalars import sat_limit

BLOCK_BITS = 128
FORCE_SCALAR_ENV = "SEMIMAT_FORCE_SCALAR"

_DTYPES = {8: np.uint8, 16: np.uint16, 32: np.uint32}
_SIMD_MACHINES = {"x86_64", "amd64", "i386", "i686", "aarch64", "arm64", "ppc64le"}
OP_SUBSAT, OP_ADDSAT, OP_MAX, OP_MIN, OP_ABSDIFF, OP_CLONENOT = range(6)

_forced = None  # None, "scalar" or "vector" (reported only; see module doc)


def lane_count(width: int) -> int:
    """Lanes per 128-bit block: 16, 8 or 4 (kernels.py:41-44)."""
    sat_limit(width)
    return BLOCK_BITS // width


def dtype_for(width: int):
    """numpy dtype matching a lane width (kernels.py:47-50)."""
    sat_limit(width)
    return _DTYPES[width]


def vector_supported() -> bool:
    """kernels.py:53-55: whether the host ISA has 128-bit integer SIMD."""
    return platform.machine().lower() in _SIMD_MACHINES


def use_vector() -> bool:
    """The reference's path flag (kernels.py:58-64); the device kernels run either way."""
    if _forced is not None:
        return _forced == "vector"
    if os.environ.get(FORCE_SCALAR_ENV, "0") not in ("", "0"):
        return False
    return vector_supported()


@contextmanager
def forced_scalar():
    global _forced
    previous = _forced
    _forced = "scalar"
    try:
        yield
    finally:
        _forced = previous


@contextmanager
def forced_vector():
    global _forced
    previous = _forced
    _forced = "vector"
    try:
        yield
    finally:
        _forced = previous


def _lanes(seq, width: int) -> np.ndarray:
    """Coerce a flat sequence to the lane dtype, refusing silent wraparound
    (the checks and messages of kernels.py:91-104)."""
    limit = sat_limit(width)
    dtype = _DTYPES[width]
    arr = np.asarray(seq)
    if arr.dtype != dtype:
        if arr.size and (arr.min() < 0 or arr.max() > limit):
            raise ValueError(f"lane value outside [0, {limit}]")
        arr = arr.astype(dtype)
    if arr.ndim != 1 or arr.size % lane_count(width):
        raise ValueError(f"expected a flat sequence of a multiple of {lane_count(width)} lanes")
    return np.ascontiguousarray(arr)


def _device_op(x: torch.Tensor, y: torch.Tensor | None, op: int) -> torch.Tensor:
    """Run smx_lane_op on flat CUDA tensors of whole 128-bit blocks."""
    out = torch.empty_like(x)
    _native.check(_native.lib().smx_lane_op(
        x.data_ptr(), (y if y is not None else x).data_ptr(), out.data_ptr(), x.numel(),
        x.element_size(), op, _native.stream_ptr(x.device)), "smx_lane_op")
    return out


def _run(x: np.ndarray, y: np.ndarray | None, op: int) -> np.ndarray:
    if x.size == 0:
        return x.copy()
    dev = _native.require_cuda()
    tx = torch.from_numpy(x).to(dev)
    ty = torch.from_numpy(y).to(dev) if y is not None else None
    return _device_op(tx, ty, op).cpu().numpy()


def _pair_op(a, b, width: int, op: int) -> list[int]:
    x, y = _lanes(a, width), _lanes(b, width)
    if len(x) != len(y):
        raise ValueError(f"lane count mismatch: {len(x)} vs {len(y)}")
    return _run(x, y, op).tolist()


def clonenot(value: int, width: int = 8, count: int | None = None) -> list[int]:
    """Width-complement of ``value`` copied into every lane (kernels.py:129-144)."""
    limit = sat_limit(width)
    block = lane_count(width)
    n = block if count is None else count
    if n <= 0 or n % block:
        raise ValueError(f"count must be a positive multiple of {block}, got {count}")
    if not 0 <= value <= limit:
        raise ValueError(f"lane value {value} outside [0, {limit}]")
    return _run(np.full(n, value, dtype=_DTYPES[width]), None, OP_CLONENOT).tolist()


def subsat(a, b, width: int = 8) -> list[int]:
    """Lanewise saturating subtraction max(a - b, 0) (kernels.py:147-152)."""
    return _pair_op(a, b, width, OP_SUBSAT)


def addsat(a, b, width: int = 8) -> list[int]:
    """Lanewise saturating addition min(a + b, S) (kernels.py:155-161)."""
    return _pair_op(a, b, width, OP_ADDSAT)


def maxlanes(a, b, width: int = 8) -> list[int]:
    return _pair_op(a, b, width, OP_MAX)


def minlanes(a, b, width: int = 8) -> list[int]:
    return _pair_op(a, b, width, OP_MIN)


def absdiff(a, b, width: int = 8) -> list[int]:
    """Lanewise |a - b| (kernels.py:180-189)."""
    return _pair_op(a, b, width, OP_ABSDIFF)


# ---- array-level forms (kernels.py:195-204), on the device -----------------

def _array_op(a, b, op: int):
    """Broadcast a and b, run the lane kernel on the device.  numpy in ->
    numpy out; CUDA tensors in -> CUDA tensor out (stays in HBM)."""
    if isinstance(a, torch.Tensor) or isinstance(b, torch.Tensor):
        ta = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))
        tb = b if isinstance(b, torch.Tensor) else torch.as_tensor(np.asarray(b))
        dev = ta.device if ta.is_cuda else tb.device
        if dev.type != "cuda":
            dev = _native.require_cuda()
        if ta.dtype != tb.dtype or ta.dtype not in (torch.uint8, torch.uint16, torch.uint32):
            raise TypeError(f"lane operands must share an unsigned dtype, got {ta.dtype} and {tb.dtype}")
        xa, xb = torch.broadcast_tensors(ta.to(dev), tb.to(dev))
        shape = xa.shape
        return _flat_device(xa.reshape(-1), xb.reshape(-1), op).reshape(shape)
    xa, xb = np.broadcast_arrays(np.asarray(a), np.asarray(b))
    dt = np.result_type(xa, xb)
    if dt not in (np.uint8, np.uint16, np.uint32):
        raise TypeError(f"lane operands must carry an unsigned dtype, got {dt}")
    shape = xa.shape
    dev = _native.require_cuda()
    ta = torch.from_numpy(np.ascontiguousarray(xa, dtype=dt).reshape(-1)).to(dev)
    tb = torch.from_numpy(np.ascontiguousarray(xb, dtype=dt).reshape(-1)).to(dev)
    return _flat_device(ta, tb, op).cpu().numpy().reshape(shape)


def _flat_device(x: torch.Tensor, y: torch.Tensor, op: int) -> torch.Tensor:
    n = x.numel()
    per = 16 // x.element_size()
    padded = -(-n // per) * per
    if padded == 0:
        return x.clone()
    if padded != n or not x.is_contiguous() or not y.is_contiguous():
        xp = torch.zeros(padded, dtype=x.dtype, device=x.device)
        yp = torch.zeros(padded, dtype=y.dtype, device=y.device)
        xp[:n] = x
        yp[:n] = y
        x, y = xp, yp
    return _device_op(x, y, op)[:n]


def np_subsat(a, b):
    """max(a, b) - b, broadcast (kernels.py:195-196)."""
    return _array_op(a, b, OP_SUBSAT)


def np_addsat(a, b, limit):
    """min(a, limit - b) + b, broadcast (kernels.py:199-200).  ``limit`` is
    the lane limit S of the operands' dtype, as at every reference call site."""
    dt = a.dtype if hasattr(a, "dtype") else np.asarray(a).dtype
    bits = {np.dtype(np.uint8): 8, np.dtype(np.uint16): 16, np.dtype(np.uint32): 32,
            torch.uint8: 8, torch.uint16: 16, torch.uint32: 32}.get(dt)
    if bits is None or int(limit) != (1 << bits) - 1:
        raise ValueError(f"np_addsat: limit {limit} is not the lane limit of {dt}")
    return _array_op(a, b, OP_ADDSAT)


def np_absdiff(a, b):
    """(a -sat b) | (b -sat a), broadcast (kernels.py:203-204)."""
    return _array_op(a, b, OP_ABSDIFF)
