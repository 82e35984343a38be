"""Device engines behind the matrix classes: thin calls into libsemimat_b200.so.

These replace the reference's compute engines one for one
(pkg/src/semimat/antidist.py:361-458; boolmat.py:151-189).  Each function
takes CUDA tensors in the reference's storage layout, allocates the result
and any workspace from torch's caching allocator, and launches on torch's
current stream.  Nothing here falls back to the CPU.
"""

from __future__ import annotations

import torch

from . import _native
from ._native import SMX_ANTI, SMX_DIST, check, lib, stream_ptr

_GEMM = {8: "smx_semiring_gemm_u8", 16: "smx_semiring_gemm_u16", 32: "smx_semiring_gemm_u32"}
_FW = {8: "smx_fw_u8", 16: "smx_fw_u16", 32: "smx_fw_u32"}
_TC_WS: dict = {}   # (M, N, K) -> smx_bool_mul_tc_workspace_bytes
_SCRATCH: dict = {}  # (device index, stream) -> grow-only scratch


def _stream_scratch(device: torch.device, sp: int, nbytes: int) -> torch.Tensor:
    """Per-(device, stream) grow-only scratch (<= 64 MB) for the one-call product:
    calls on one stream are ordered, so the buffer can be reused, which saves
    an allocator round trip per call.  Fresh (not kept) inside a stream
    capture, whose graph may later replay on another stream."""
    if nbytes > (64 << 20) or torch.cuda.is_current_stream_capturing():
        return _native.workspace(nbytes, device)   # large: the allocation cost is noise
    key = (device.index, sp)
    buf = _SCRATCH.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = _SCRATCH[key] = _native.workspace(nbytes, device)
    return buf


def lane_mul(a: torch.Tensor, b: torch.Tensor, inner: int, width: int, anti: bool,
             out: torch.Tensor | None = None) -> torch.Tensor:
    """C = A (x) B on padded lane storage; replaces _mul_vector (antidist.py:361-371)
    and _minplus_mul_vector (:412-422).  Computes the padded width too: B's
    padding lanes are the (+)-identity, so C's padding comes out as identity."""
    rows, cols_p = a.shape[0], b.shape[1]
    if out is None:
        out = torch.empty((rows, cols_p), dtype=a.dtype, device=a.device)
    fn = getattr(lib(), _GEMM[width])
    check(fn(a.data_ptr(), b.data_ptr(), out.data_ptr(), rows, cols_p, inner, a.shape[1],
             b.shape[1], out.shape[1], SMX_ANTI if anti else SMX_DIST, 0,
             stream_ptr(a.device)), _GEMM[width])
    return out


def lane_close_(t: torch.Tensor, n: int, width: int, anti: bool) -> torch.Tensor:
    """In-place blocked Floyd-Warshall; replaces _close_vector (antidist.py:390-398)
    and _minplus_close_vector (:440-448)."""
    ld = t.shape[1]
    nbytes = lib().smx_fw_workspace_bytes(n, ld, width // 8)
    ws = _native.workspace(nbytes, t.device)
    fn = getattr(lib(), _FW[width])
    check(fn(t.data_ptr(), n, ld, SMX_ANTI if anti else SMX_DIST, ws.data_ptr(), nbytes,
             stream_ptr(t.device)), _FW[width])
    return t


_FW_HOST = {8: "smx_fw_host_u8", 16: "smx_fw_host_u16", 32: "smx_fw_host_u32"}


def lane_close_host(host: torch.Tensor, n: int, width: int, anti: bool, out: torch.Tensor | None = None,
                    device=None) -> tuple[torch.Tensor, torch.Tensor]:
    """Closure of a matrix in host memory into host memory (smx_fw_host_*):
    the PCIe copies in and out run concurrently with the closure.  `host` and
    `out` are CPU tensors in the padded lane layout (page-locked for overlap).
    Returns (out, device copy of the closure); `out` is complete when the
    current stream reaches this point (synchronize before reading it)."""
    if host.device.type != "cpu" or not host.is_contiguous():
        raise ValueError("host matrix must be a contiguous CPU tensor")
    if out is None:
        out = torch.empty_like(host, pin_memory=True)
    if out.shape != host.shape or out.dtype != host.dtype or out.device.type != "cpu" or not out.is_contiguous():
        raise ValueError("out must be a contiguous CPU tensor shaped like the input")
    dev = _native.require_cuda(device)
    t = torch.empty(host.shape, dtype=host.dtype, device=dev)
    ld = host.shape[1]
    nbytes = lib().smx_fw_host_workspace_bytes(n, ld, width // 8)
    ws = _native.workspace(nbytes, dev)
    check(getattr(lib(), _FW_HOST[width])(host.data_ptr(), out.data_ptr(), t.data_ptr(), n, ld,
                                          SMX_ANTI if anti else SMX_DIST, ws.data_ptr(), nbytes,
                                          stream_ptr(dev)), _FW_HOST[width])
    return out, t


def bool_mul_bits(a, b):
    """Bit-packed OR/AND product (the comparison variant); boolmat.py:151-172."""
    from .boolmat import BoolMatrix, _stride_words
    out = torch.zeros((a.rows, _stride_words(b.cols)), dtype=torch.int32, device=a.device)
    check(lib().smx_bool_gemm_bits(a._words.data_ptr(), b._words.data_ptr(), out.data_ptr(),
                                   a.rows, (b.cols + 31) // 32, a.cols, a.stride_words,
                                   b.stride_words, out.shape[1], 0, stream_ptr(a.device)),
          "smx_bool_gemm_bits")
    return BoolMatrix(a.rows, b.cols, out)


def _round16(x: int) -> int:
    return -(-x // 16) * 16


def bits_to_bytes(m, transpose: bool = False) -> torch.Tensor:
    """Unpack a BoolMatrix to 0/1 bytes (rows x round16(cols)), or its transpose."""
    rows, cols = m.rows, m.cols
    if transpose:
        t8 = torch.empty((cols, _round16(rows)), dtype=torch.uint8, device=m.device)
        check(lib().smx_unpack_bits_transposed(m._words.data_ptr(), t8.data_ptr(), rows, cols,
                                               m.stride_words, t8.shape[1], stream_ptr(m.device)),
              "smx_unpack_bits_transposed")
        return t8
    b8 = torch.empty((rows, _round16(cols)), dtype=torch.uint8, device=m.device)
    check(lib().smx_unpack_bits(m._words.data_ptr(), b8.data_ptr(), rows, cols, m.stride_words,
                                b8.shape[1], stream_ptr(m.device)), "smx_unpack_bits")
    return b8


def bool_mul_tc(a, b):
    """Tensor-core product: tcgen05 kind::i8 GEMM, count > 0, packed-bit epilogue
    (one C-ABI call: unpack, fused B^T unpack, product)."""
    from .boolmat import BoolMatrix, _stride_words
    L = lib()
    out = torch.empty((a.rows, _stride_words(b.cols)), dtype=torch.int32, device=a.device)
    key = (a.rows, b.cols, a.cols)
    nbytes = _TC_WS.get(key)
    if nbytes is None:
        nbytes = _TC_WS[key] = L.smx_bool_mul_tc_workspace_bytes(a.rows, b.cols, a.cols)
    sp = stream_ptr(a.device)
    ws = _stream_scratch(a.device, sp, nbytes)
    check(L.smx_bool_mul_tc(a._words.data_ptr(), b._words.data_ptr(), out.data_ptr(), a.rows, b.cols,
                            a.cols, a.stride_words, b.stride_words, out.shape[1], ws.data_ptr(), nbytes,
                            sp), "smx_bool_mul_tc")
    return BoolMatrix(a.rows, b.cols, out)


def bool_mul(a, b):
    """BoolMatrix.__mul__ engine: the tensor-core GEMM."""
    return bool_mul_tc(a, b)


def bool_closure_tc(m):
    """Blocked Warshall on bytes with tensor-core phases 2/3."""
    from .boolmat import BoolMatrix
    t8 = bits_to_bytes(m)
    nbytes = lib().smx_bool_warshall_i8_workspace_bytes(m.rows, t8.shape[1])
    ws = _native.workspace(nbytes, m.device)
    check(lib().smx_bool_warshall_i8(t8.data_ptr(), m.rows, t8.shape[1], ws.data_ptr(), nbytes,
                                     stream_ptr(m.device)), "smx_bool_warshall_i8")
    words = torch.empty_like(m._words)
    check(lib().smx_pack_bits(t8.data_ptr(), words.data_ptr(), m.rows, m.cols, t8.shape[1],
                              m.stride_words, stream_ptr(m.device)), "smx_pack_bits")
    return BoolMatrix(m.rows, m.cols, words)


def bool_closure_bits(m):
    """Blocked Warshall on packed bits; boolmat.py:174-189."""
    from .boolmat import BoolMatrix
    words = m._words.clone()
    nbytes = lib().smx_bool_warshall_workspace_bytes(m.rows, m.stride_words)
    ws = _native.workspace(nbytes, m.device)
    check(lib().smx_bool_warshall_bits(words.data_ptr(), m.rows, m.stride_words, ws.data_ptr(),
                                       nbytes, stream_ptr(m.device)), "smx_bool_warshall_bits")
    return BoolMatrix(m.rows, m.cols, words)


def bool_closure(m):
    """BoolMatrix.transitive_closure engine."""
    return bool_closure_bits(m)


def closure_by_squaring(m, max_squarings: int = 64):
    """Closure as A (x) (I (+) A)^(2^j), squared on the GPU to a fixpoint.

    The reference's independent check (pkg/src/semimat/oracle.py:49-74,
    acceptance criterion 6) run with the device products: an algorithm with
    no shared code path with the blocked Floyd-Warshall / Warshall, used to
    cross-check them at sizes the CPU oracle cannot reach.  Works for
    BoolMatrix, AntidistMatrix and DistMatrix.
    """
    from .antidist import AntidistMatrix, DistMatrix
    from .boolmat import BoolMatrix
    if m.rows != m.cols:
        raise ValueError(f"closure needs a square matrix, got {m.rows}x{m.cols}")
    if isinstance(m, BoolMatrix):
        eye = BoolMatrix.identity(m.rows)
    elif isinstance(m, (AntidistMatrix, DistMatrix)):
        eye = type(m).identity(m.rows, m.width)
    else:
        raise TypeError(f"expected a semimat matrix, got {type(m).__name__}")
    # (+) with the identity: | is max (anti) / OR (bool); & is min (dist)
    power = (eye & m) if isinstance(m, DistMatrix) else (eye | m)
    for _ in range(max_squarings):
        nxt = power * power
        if nxt == power:
            break
        power = nxt
    return m * power
