"""Many small products and closures in one launch.

The reference computes one matrix per call (pkg/src/semimat/boolmat.py:151-189,
antidist.py:226-350).  Workloads of many small graphs -- its own acceptance
suite runs 262,144 3x3 Boolean products and 1,500 closures of <= 64-vertex
graphs (pkg/tests/test_acceptance.py:28-85) -- would be bound by one launch
(and one host round trip) per matrix on a GPU, so this module stacks
same-shaped matrices and runs the batched kernels of csrc/lanes.cu:

* ``bool_mul_many(As, Bs)``     BoolMatrix products      (smx_bool_mul_tc_batched on the
                                tensor cores for 128-multiple shapes, else
                                smx_bool_mul_batched)
* ``bool_closure_many(Ms)``     Warshall, n <= 512       (smx_bool_warshall_batched)
* ``closure_many(Ms)``          Floyd-Warshall of AntidistMatrix / DistMatrix,
                                n <= 128                 (smx_fw_batched)

Results equal the per-matrix calls bit for bit (the same sweep per matrix).
Shapes outside the batched kernels' limits fall back to the per-matrix
device calls -- still the GPU, never the CPU.  The ``*_stacked`` functions
take and return stacked device tensors in the classes' storage layouts.
"""

from __future__ import annotations

import torch

from . import _native
from .antidist import AntidistMatrix, DistMatrix, _LaneMatrix
from .boolmat import BoolMatrix

FW_BATCH_MAX = 128
WARSHALL_BATCH_MAX = 512


def bool_mul_stacked(a_words: torch.Tensor, b_words: torch.Tensor, inner: int, cols: int) -> torch.Tensor:
    """(batch, M, lda_w) x (batch, inner, ldb_w) packed rows -> (batch, M, ldc_w),
    ldc_w = the BoolMatrix stride for ``cols`` columns."""
    from .boolmat import _stride_words
    batch, m = a_words.shape[0], a_words.shape[1]
    if b_words.shape[0] != batch or b_words.shape[1] != inner:
        raise ValueError("stacked operands disagree in batch or inner size")
    a_words, b_words = a_words.contiguous(), b_words.contiguous()
    out = torch.empty((batch, m, _stride_words(cols)), dtype=torch.int32, device=a_words.device)
    _native.check(_native.lib().smx_bool_mul_batched(
        a_words.data_ptr(), b_words.data_ptr(), out.data_ptr(), batch, m, cols, inner, a_words.shape[2],
        b_words.shape[2], out.shape[2], m * a_words.shape[2], inner * b_words.shape[2],
        m * out.shape[2], _native.stream_ptr(a_words.device)), "smx_bool_mul_batched")
    return out


def bool_closure_stacked_(t_words: torch.Tensor, n: int) -> torch.Tensor:
    """Warshall closure in place on (batch, n, ld_w) packed rows, n <= 512."""
    if not t_words.is_contiguous():
        raise ValueError("stacked matrices must be contiguous")
    _native.check(_native.lib().smx_bool_warshall_batched(
        t_words.data_ptr(), t_words.shape[0], n, t_words.shape[2], n * t_words.shape[2],
        _native.stream_ptr(t_words.device)), "smx_bool_warshall_batched")
    return t_words


def fw_stacked_(t: torch.Tensor, n: int, width: int, anti: bool) -> torch.Tensor:
    """Floyd-Warshall in place on (batch, n, padded) lane storage, n <= 128."""
    if not t.is_contiguous():
        raise ValueError("stacked matrices must be contiguous")
    _native.check(_native.lib().smx_fw_batched(
        t.data_ptr(), t.shape[0], n, t.shape[2], n * t.shape[2], width // 8,
        _native.SMX_ANTI if anti else _native.SMX_DIST, _native.stream_ptr(t.device)), "smx_fw_batched")
    return t


def bool_mul_many(As, Bs) -> list[BoolMatrix]:
    """[A * B for A, B in zip(As, Bs)], same-shaped pairs in one launch."""
    As, Bs = list(As), list(Bs)
    if len(As) != len(Bs):
        raise ValueError(f"{len(As)} left operands but {len(Bs)} right operands")
    if not As:
        return []
    a0, b0 = As[0], Bs[0]
    same = all(isinstance(a, BoolMatrix) and (a.rows, a.cols) == (a0.rows, a0.cols) for a in As) and \
        all(isinstance(b, BoolMatrix) and (b.rows, b.cols) == (b0.rows, b0.cols) for b in Bs)
    if not same or a0.cols != b0.rows:
        return [a * b for a, b in zip(As, Bs)]      # per-pair validation and messages
    dev = a0.device
    a_st = torch.stack([a._words.to(dev) for a in As])
    b_st = torch.stack([b._words.to(dev) for b in Bs])
    if a0.rows % 128 == 0 and b0.cols % 128 == 0 and 128 < a0.cols <= 65536:
        out = bool_mul_stacked_tc(a_st, b_st, a0.cols, b0.cols)   # tensor cores, one launch
    else:
        out = bool_mul_stacked(a_st, b_st, a0.cols, b0.cols)
    return [BoolMatrix(a0.rows, b0.cols, out[i]) for i in range(len(As))]


def bool_mul_stacked_tc(a_words: torch.Tensor, b_words: torch.Tensor, inner: int, cols: int) -> torch.Tensor:
    """The stacked products on the tensor cores (smx_bool_mul_tc_batched: one
    unpack of every A, the fused B^T unpacks, then one split-K pair launch
    for all products).  M and ``cols`` multiples of 128, 128 < inner <= 65536."""
    from .boolmat import _stride_words
    batch, m = a_words.shape[0], a_words.shape[1]
    if b_words.shape[0] != batch or b_words.shape[1] != inner:
        raise ValueError("stacked operands disagree in batch or inner size")
    a_words, b_words = a_words.contiguous(), b_words.contiguous()
    lib = _native.lib()
    out = torch.empty((batch, m, _stride_words(cols)), dtype=torch.int32, device=a_words.device)
    nbytes = lib.smx_bool_mul_tc_batched_workspace_bytes(batch, m, cols, inner)
    ws = _native.workspace(nbytes, a_words.device)
    _native.check(lib.smx_bool_mul_tc_batched(
        a_words.data_ptr(), b_words.data_ptr(), out.data_ptr(), batch, m, cols, inner, a_words.shape[2],
        b_words.shape[2], out.shape[2], ws.data_ptr(), nbytes, _native.stream_ptr(a_words.device)),
        "smx_bool_mul_tc_batched")
    return out


def bool_closure_many(Ms) -> list[BoolMatrix]:
    """[M.transitive_closure() for M in Ms], same-sized n <= 512 in one launch."""
    Ms = list(Ms)
    if not Ms:
        return []
    m0 = Ms[0]
    if (m0.rows != m0.cols or m0.rows > WARSHALL_BATCH_MAX or
            any((m.rows, m.cols) != (m0.rows, m0.cols) for m in Ms)):
        return [m.transitive_closure() for m in Ms]
    t = torch.stack([m._words.to(m0.device) for m in Ms])
    bool_closure_stacked_(t, m0.rows)
    return [BoolMatrix(m0.rows, m0.cols, t[i]) for i in range(len(Ms))]


def closure_many(Ms) -> list[_LaneMatrix]:
    """[M.transitive_closure() for M in Ms] for AntidistMatrix / DistMatrix;
    same class, width and size n <= 128 in one launch."""
    Ms = list(Ms)
    if not Ms:
        return []
    m0 = Ms[0]
    cls = type(m0)
    if (cls not in (AntidistMatrix, DistMatrix) or m0.rows != m0.cols or m0.rows > FW_BATCH_MAX or
            any(type(m) is not cls or (m.rows, m.cols, m.width) != (m0.rows, m0.cols, m0.width) for m in Ms)):
        return [m.transitive_closure() for m in Ms]
    t = torch.stack([m._data.to(m0.device) for m in Ms])
    fw_stacked_(t, m0.rows, m0.width, anti=cls is AntidistMatrix)
    return [cls(m0.rows, m0.cols, m0.width, t[i]) for i in range(len(Ms))]
