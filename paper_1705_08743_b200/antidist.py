"""Dense saturated lane matrices on the GPU -- drop-in for semimat.antidist.

AntidistMatrix: entry a encodes distance S - a (0 = unreachable, S =
distance zero); (+) = lanewise max, (x) = max(a + b - S, 0).  DistMatrix is
the complement view: plain distances, S = unreachable, (+) = min,
(x) = min(a + b, S).  Class surface, validation order and messages follow
pkg/src/semimat/antidist.py:31-350; storage is the reference's padded layout
(rows x ceil(cols / L) * L lanes, L = 128 / width, pad = the class's
(+)-identity, antidist.py:38-55) held in HBM.  Products and closures run in
the sm_100a kernels of libsemimat_b200.so; there is no CPU path and no
scalar/vector dispatch (the reference's kernels.use_vector(), kernels.py:58-64,
is the boundary this package replaces).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .boolmat import BoolMatrix
from .scalars import sat_limit

LANES = {8: 16, 16: 8, 32: 4}
_NP = {8: np.uint8, 16: np.uint16, 32: np.uint32}
_TORCH = {8: torch.uint8, 16: torch.uint16, 32: torch.uint32}


def lane_count(width: int) -> int:
    sat_limit(width)
    return LANES[width]


def dtype_for(width: int):
    sat_limit(width)
    return _NP[width]


def _from_edges(cls, dim: int, edges, width: int):
    """Validate like the reference (first offending edge, in edge order, same
    messages: antidist.py:201-208), then fill + scatter on the GPU.  Large
    edge lists are validated on the device (smx_edges_first_invalid) after
    one staged upload; only the first offender's row is looked at on the
    host, to word its message."""
    if dim < 1:
        raise ValueError(f"matrix dimensions must be positive, got {dim}x{dim}")
    limit = sat_limit(width)
    if not isinstance(edges, np.ndarray):
        edges = list(edges)
    arr = np.asarray(edges, dtype=np.int64).reshape(-1, 3) if len(edges) else np.zeros((0, 3), np.int64)
    arr = np.ascontiguousarray(arr)
    m = arr.shape[0]

    def reject(i: int):
        u, v, w = (int(x) for x in arr[i])
        if not 0 <= u < dim:
            raise ValueError(f"source vertex {u} out of range [0, {dim})")
        if not 0 <= v < dim:
            raise ValueError(f"target vertex {v} out of range [0, {dim})")
        raise ValueError(f"weight {w} outside [0, {limit}]")

    if m < (1 << 16):   # small lists: host check, nothing launched for a bad one
        u, v, w = arr[:, 0], arr[:, 1], arr[:, 2]
        bad = (u < 0) | (u >= dim) | (v < 0) | (v >= dim) | (w < 0) | (w > limit)
        if bad.any():
            reject(int(np.argmax(bad)))
    dev = _native.require_cuda()
    lib = _native.lib()
    st = _native.stream_ptr(dev)
    dev_edges = torch.empty(arr.shape, dtype=torch.int64, device=dev)
    if m:   # (staged through the page-locked ring when large, smx_copy_h2d)
        _native.check(lib.smx_copy_h2d(dev_edges.data_ptr(), arr.ctypes.data, arr.nbytes, st), "smx_copy_h2d")
    if m >= (1 << 16):
        first = torch.empty(1, dtype=torch.int64, device=dev)
        _native.check(lib.smx_edges_first_invalid(dev_edges.data_ptr(), m, dim, limit, first.data_ptr(), st),
                      "smx_edges_first_invalid")
        i = int(first.item())
        if i < m:
            reject(i)
    data = torch.empty((dim, -(-dim // LANES[width]) * LANES[width]), dtype=_TORCH[width], device=dev)
    _native.check(lib.smx_from_edges(
        dev_edges.data_ptr(), m, data.data_ptr(), dim, data.shape[1], width // 8,
        _native.SMX_DIST if cls._PAD_IS_LIMIT else _native.SMX_ANTI, st),
        "smx_from_edges")
    return cls(dim, dim, width, data)


_COPY_STREAMS: dict = {}


def _copy_stream(dev, which: int) -> torch.cuda.Stream:
    """Side streams per device for the streamed host product's copies in (0)
    and out (1)."""
    key = (torch.device(dev).index, which)
    if key not in _COPY_STREAMS:
        _COPY_STREAMS[key] = torch.cuda.Stream(device=dev)
    return _COPY_STREAMS[key]


def _to_host(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> host array.  Large ones land in page-locked memory
    from torch's caching host allocator (55 GB/s, no first-touch page faults:
    a fresh 2 GiB pageable array costs ~0.4 s of faults on the pool's hosts,
    profiles/r02l_host_io.json)."""
    if t.numel() * t.element_size() < (8 << 20):
        return t.cpu().numpy()
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t)
    return out.numpy()


class _LaneMatrix:
    """Shared storage and entrywise algebra of the two saturated matrix types.

    Storage lives in HBM (``_dev``, a CUDA tensor).  A matrix built from a
    host array is *host-backed* until its first device operation, like the
    reference's ``_data`` (antidist.py:46-51), which is the caller's array
    itself: ``.data`` is then a read-only view of that array (no copy), and
    ``transitive_closure()`` runs the host-buffer closure (smx_fw_host_*: the
    rows stream in through page-locked staging while the closure runs, the
    finished rows stream out) into page-locked memory, returning a
    host-backed result.  Any other device use moves the array to HBM once.
    """

    __slots__ = ("rows", "cols", "width", "_dev", "_host", "_device")

    _PAD_IS_LIMIT = False

    def __init__(self, rows: int, cols: int, width: int = 8, _data=None, *, device=None):
        if rows < 1 or cols < 1:
            raise ValueError(f"matrix dimensions must be positive, got {rows}x{cols}")
        lanes = lane_count(width)
        padded = -(-cols // lanes) * lanes
        self.rows = rows
        self.cols = cols
        self.width = width
        self._dev = self._host = None
        if isinstance(_data, torch.Tensor):
            if tuple(_data.shape) != (rows, padded) or _data.dtype != _TORCH[width]:
                raise ValueError("backing array does not match the padded shape")
            if _data.device.type != "cuda":
                _data = _data.to(_native.require_cuda(device))
            self._dev = _data.contiguous()
            self._device = self._dev.device
            return
        self._device = _native.require_cuda(device)
        if _data is None:
            fill = self._pad_fill(width)
            host = np.full((rows, padded), fill, dtype=_NP[width])
        else:
            host = np.asarray(_data)
            if host.shape != (rows, padded) or host.dtype != _NP[width]:
                raise ValueError("backing array does not match the padded shape")
        self._host = host

    @property
    def _data(self) -> torch.Tensor:
        """The device storage (moves a host-backed matrix to HBM first: one
        smx_copy_h2d, which stages a large pageable array through the
        library's page-locked ring)."""
        if self._dev is None:
            src = np.ascontiguousarray(self._host)
            dev = torch.empty(src.shape, dtype=_TORCH[self.width], device=self._device)
            _native.check(_native.lib().smx_copy_h2d(dev.data_ptr(), src.ctypes.data, src.nbytes,
                                                     _native.stream_ptr(self._device)), "smx_copy_h2d")
            self._dev = dev
            self._host = None
        return self._dev

    @_data.setter
    def _data(self, value: torch.Tensor) -> None:
        self._dev = value
        self._host = None
        self._device = value.device

    @property
    def host_backed(self) -> bool:
        """True while the storage is still the host array the matrix was built on."""
        return self._dev is None

    @classmethod
    def _pad_fill(cls, width):
        return sat_limit(width) if cls._PAD_IS_LIMIT else 0

    # -- basics -------------------------------------------------------------

    @property
    def limit(self) -> int:
        return sat_limit(self.width)

    @property
    def padded_cols(self) -> int:
        return -(-self.cols // LANES[self.width]) * LANES[self.width]

    @property
    def device(self) -> torch.device:
        return self._device

    @property
    def data(self):
        """Raw lane storage including padding columns, read-only: a view of
        the backing host array (host-backed, as the reference's view,
        antidist.py:68-73), else a host copy of the device storage."""
        view = self._host.view() if self._dev is None else _to_host(self._dev)
        view.flags.writeable = False
        return view

    def to_numpy(self) -> np.ndarray:
        if self._dev is None:
            return np.array(self._host)
        return _to_host(self._dev)

    def copy(self):
        if self._dev is None:
            return type(self)(self.rows, self.cols, self.width, np.array(self._host), device=self._device)
        return type(self)(self.rows, self.cols, self.width, self._dev.clone())

    def _check_index(self, i, j):
        if not (0 <= i < self.rows and 0 <= j < self.cols):
            raise IndexError(f"index ({i}, {j}) out of range for {self.rows}x{self.cols}")

    def get(self, i: int, j: int) -> int:
        self._check_index(i, j)
        if self._dev is None:
            return int(self._host[i, j])
        return int(self._dev[i, j].cpu().numpy())

    def set(self, i: int, j: int, value: int) -> None:
        self._check_index(i, j)
        if not 0 <= value <= self.limit:
            raise ValueError(f"entry {value!r} outside [0, {self.limit}]")
        if self._dev is None:   # writes the backing array, as the reference does
            self._host[i, j] = value
            return
        self._dev[i, j] = torch.from_numpy(np.array(value, dtype=_NP[self.width])).to(self.device)

    def to_lists(self) -> list[list[int]]:
        return self.to_numpy()[:, : self.cols].tolist()

    @classmethod
    def from_lists(cls, rows: list[list[int]], width: int = 8):
        if not rows or not rows[0]:
            raise ValueError("matrix dimensions must be positive")
        ncols = len(rows[0])
        limit = sat_limit(width)
        host = np.full((len(rows), -(-ncols // LANES[width]) * LANES[width]),
                       cls._pad_fill(width), dtype=_NP[width])
        for i, row in enumerate(rows):
            if len(row) != ncols:
                raise ValueError(f"row {i} has {len(row)} entries, expected {ncols}")
            for v in row:
                if not 0 <= v <= limit:
                    raise ValueError(f"entry {v!r} outside [0, {limit}]")
            host[i, :ncols] = row
        return cls(len(rows), ncols, width, host)

    @classmethod
    def from_numpy(cls, data: np.ndarray, cols: int, width: int, device=None):
        """Wrap a padded host array (rows x padded cols, lane dtype)."""
        return cls(data.shape[0], cols, width, np.ascontiguousarray(data), device=device)

    # -- entrywise algebra (device kernel) ------------------------------------

    def _check_same(self, other):
        if type(other) is not type(self):
            raise TypeError(f"expected {type(self).__name__}, got {type(other).__name__}")
        if (self.rows, self.cols, self.width) != (other.rows, other.cols, other.width):
            raise ValueError(
                f"shape/width mismatch: {self.rows}x{self.cols}/w{self.width} vs "
                f"{other.rows}x{other.cols}/w{other.width}"
            )
        if self.device != other.device:
            raise ValueError(f"operands live on different devices: {self.device} vs {other.device}")

    def _entrywise(self, other, op: int, out_cls):
        out = torch.empty_like(self._data)
        b = other._data if other is not None else self._data
        _native.check(
            _native.lib().smx_lane_entrywise(
                self._data.data_ptr(), b.data_ptr(), out.data_ptr(), self.rows, self.cols,
                self.padded_cols, self.width // 8, op, int(out_cls._PAD_IS_LIMIT),
                _native.stream_ptr(self.device)),
            "lane entrywise")
        return out_cls(self.rows, self.cols, self.width, out)

    def __and__(self, other):
        """Lanewise minimum."""
        self._check_same(other)
        return self._entrywise(other, 0, type(self))

    def __or__(self, other):
        """Lanewise maximum."""
        self._check_same(other)
        return self._entrywise(other, 1, type(self))

    def __xor__(self, other):
        """Lanewise absolute difference."""
        self._check_same(other)
        return self._entrywise(other, 2, type(self))

    def __invert__(self):
        """Complement at width, switching between the two encodings."""
        cls = DistMatrix if isinstance(self, AntidistMatrix) else AntidistMatrix
        return self._entrywise(None, 3, cls)

    def __eq__(self, other):
        if type(other) is not type(self):
            return NotImplemented
        return (self.rows, self.cols, self.width) == (other.rows, other.cols, other.width) and bool(
            torch.equal(self._data.view(torch.uint8), other._data.to(self.device).view(torch.uint8)))

    __hash__ = None

    def __repr__(self):
        return f"<{type(self).__name__} {self.rows}x{self.cols} width={self.width}>"

    # -- shared product / closure plumbing -----------------------------------

    # Host-backed left operands of at least this many lanes take the streamed
    # host product (_mul_host); smaller ones move to HBM and stay there.
    _HOST_MUL_MIN = 1 << 24

    def _mul(self, other, anti: bool):
        """C = self (x) other: device-resident, or streamed from a large
        host-backed left operand (the reference's own call on numpy arrays)."""
        from . import engines
        if self._dev is None and self.rows * self.padded_cols >= self._HOST_MUL_MIN:
            return self._mul_host(other, anti)
        out = engines.lane_mul(self._data, other._data, self.cols, self.width, anti=anti)
        return type(self)(self.rows, other.cols, self.width, out)

    def _mul_host(self, other, anti: bool):
        """Row groups of the host-backed left operand stream in (staged,
        smx_copy_h2d) while the previous group's product runs, and each
        group's result rows stream out on a copy stream into page-locked
        memory: the PCIe copies overlap the products, and the result is
        host-backed like the closure's (transitive_closure)."""
        from . import engines
        dev = self._device
        lib = _native.lib()
        b = other._data                      # (resident for every group)
        src = np.ascontiguousarray(self._host)
        rows, ld_a, cols_p = self.rows, src.shape[1], b.shape[1]
        out = torch.empty((rows, cols_p), dtype=_TORCH[self.width], pin_memory=True)
        s = torch.cuda.current_stream(dev)
        xs, cs = _copy_stream(dev, 0), _copy_stream(dev, 1)   # copies in / out
        # 4 row groups of whole 128-row tiles: more groups shorten the first
        # copy in and the last copy out, but each group repacks B (8 groups
        # cost +18 ms of device time at n = 32768, 4 groups +3 ms)
        quarter = -(-rows // 4)
        group = max(128, -(-quarter // 128) * 128)
        xs.wait_stream(s)   # (b and earlier work first)
        for r0 in range(0, rows, group):
            r1 = min(rows, r0 + group)
            # the copy in runs on its own stream, so staging group g + 1 never
            # waits for group g's product; the allocator keeps a_g alive
            # until the product on s has read it (record_stream)
            with torch.cuda.stream(xs):
                a_g = torch.empty((r1 - r0, ld_a), dtype=_TORCH[self.width], device=dev)
                _native.check(lib.smx_copy_h2d(a_g.data_ptr(), src[r0:r1].ctypes.data,
                                               a_g.numel() * a_g.element_size(), xs.cuda_stream), "smx_copy_h2d")
            s.wait_stream(xs)
            a_g.record_stream(s)
            c_g = engines.lane_mul(a_g, b, self.cols, self.width, anti=anti)
            cs.wait_stream(s)
            with torch.cuda.stream(cs):
                out[r0:r1].copy_(c_g, non_blocking=True)
            c_g.record_stream(cs)
        s.wait_stream(cs)
        s.synchronize()
        return type(self)(rows, other.cols, self.width, out.numpy(), device=dev)

    def _mul_checks(self, other):
        if self.width != other.width:
            raise ValueError(f"width mismatch: {self.width} vs {other.width}")
        if self.cols != other.rows:
            raise ValueError(
                f"inner dimensions disagree: {self.rows}x{self.cols} times "
                f"{other.rows}x{other.cols}"
            )
        if self.device != other.device:
            raise ValueError(f"operands live on different devices: {self.device} vs {other.device}")

    def _close_host(self, in_place: bool = False) -> torch.Tensor:
        """Host-buffer closure of the backing array (smx_fw_host_*) into
        page-locked memory, or with ``in_place`` into the (contiguous) backing
        array itself, which the library stages back through its page-locked
        ring overlapped with the closure; returns the finished host result."""
        from . import engines
        host = torch.from_numpy(np.ascontiguousarray(self._host))
        res, _ = engines.lane_close_host(host, self.rows, self.width, anti=not self._PAD_IS_LIMIT,
                                         out=host if in_place else None, device=self._device)
        torch.cuda.current_stream(self._device).synchronize()
        return res

    def transitive_close(self) -> None:
        """In-place Floyd-Warshall closure (antidist.py:252-261 / :331-340).
        Host-backed: the backing array itself receives the result, as the
        reference's in-place sweep over ``_data`` does."""
        if self.rows != self.cols:
            raise ValueError(f"closure needs a square matrix, got {self.rows}x{self.cols}")
        from . import engines
        if self._dev is None and self._host.flags.writeable:
            if self._host.flags.c_contiguous:
                self._close_host(in_place=True)
            else:
                np.copyto(self._host, self._close_host().numpy())
            return
        engines.lane_close_(self._data, self.rows, self.width, anti=not self._PAD_IS_LIMIT)

    def transitive_closure(self):
        """Closure over >= 1 edge on a copy (antidist.py:263-273 / :342-350).
        Host-backed: one host-buffer closure call, whose result is a
        host-backed matrix over page-locked memory (``.data`` reads it
        without a copy)."""
        if self.rows != self.cols:
            raise ValueError(f"closure needs a square matrix, got {self.rows}x{self.cols}")
        if self._dev is None:
            res = self._close_host()
            return type(self)(self.rows, self.cols, self.width, res.numpy(), device=self._device)
        out = self.copy()
        out.transitive_close()
        return out

    @classmethod
    def closure_of_host(cls, data, width: int, out=None):
        """``cls(n, n, width, data).transitive_closure()`` for a square matrix
        in host memory, with its result also copied back to host memory, in
        one library call (smx_fw_host_*) whose PCIe copies overlap the
        closure.  ``data``: the padded lane storage (n x padded) as a CPU
        tensor (page-locked for the overlap) or array; ``out``: optional CPU
        tensor of the same shape to receive the result.  Returns
        (closure matrix on the device, host result); the host result is
        complete after ``torch.cuda.current_stream().synchronize()``."""
        host = data if isinstance(data, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(data))
        lanes = lane_count(width)
        n = host.shape[0]
        if host.dim() != 2 or host.shape[1] != -(-n // lanes) * lanes or host.dtype != _TORCH[width]:
            raise ValueError("backing array does not match the padded shape")
        from . import engines
        res, dev = engines.lane_close_host(host.contiguous(), n, width, anti=not cls._PAD_IS_LIMIT, out=out)
        return cls(n, n, width, dev), res


class AntidistMatrix(_LaneMatrix):
    """Matrix of anti-distance values (antidist.py:173-273)."""

    _PAD_IS_LIMIT = False

    @classmethod
    def zeros(cls, rows: int, cols: int, width: int = 8) -> "AntidistMatrix":
        return cls(rows, cols, width)

    @classmethod
    def identity(cls, dim: int, width: int = 8) -> "AntidistMatrix":
        if dim < 1:
            raise ValueError(f"matrix dimensions must be positive, got {dim}x{dim}")
        host = np.zeros((dim, -(-dim // LANES[width]) * LANES[width]), dtype=dtype_for(width))
        host[np.arange(dim), np.arange(dim)] = sat_limit(width)
        return cls(dim, dim, width, host)

    @classmethod
    def from_edges(cls, dim: int, edges, width: int = 8) -> "AntidistMatrix":
        """Adjacency of weighted edges (u, v, w); parallel edges keep the shortest
        (antidist.py:191-211).  Built on the device (smx_from_edges)."""
        return _from_edges(cls, dim, edges, width)

    @classmethod
    def from_boolmat(cls, mat: BoolMatrix, width: int = 8) -> "AntidistMatrix":
        """1 -> distance zero (S), 0 -> unreachable (antidist.py:213-219); one
        device pass from the packed bit rows (smx_lanes_from_bits)."""
        lanes = lane_count(width)
        padded = -(-mat.cols // lanes) * lanes
        out = torch.empty((mat.rows, padded), dtype=_TORCH[width], device=mat.device)
        _native.check(_native.lib().smx_lanes_from_bits(
            mat._words.data_ptr(), mat.stride_words, out.data_ptr(), mat.rows, mat.cols, padded,
            width // 8, _native.stream_ptr(mat.device)), "smx_lanes_from_bits")
        return cls(mat.rows, mat.cols, width, out)

    def to_boolmat(self) -> BoolMatrix:
        """Any finite distance becomes 1 (antidist.py:221-224); one device pass
        to the packed bit rows (smx_lanes_to_bits)."""
        from .boolmat import _stride_words
        words = torch.empty((self.rows, _stride_words(self.cols)), dtype=torch.int32, device=self.device)
        _native.check(_native.lib().smx_lanes_to_bits(
            self._data.data_ptr(), self.padded_cols, words.data_ptr(), words.shape[1], self.rows,
            self.cols, self.width // 8, _native.stream_ptr(self.device)), "smx_lanes_to_bits")
        return BoolMatrix(self.rows, self.cols, words)

    def __mul__(self, other) -> "AntidistMatrix":
        """max over k of the saturated sum (antidist.py:226-250)."""
        if not isinstance(other, AntidistMatrix):
            return NotImplemented
        self._mul_checks(other)
        return self._mul(other, anti=True)


class DistMatrix(_LaneMatrix):
    """Matrix of plain distances; the complement view (antidist.py:276-350)."""

    _PAD_IS_LIMIT = True

    @classmethod
    def unreachable(cls, rows: int, cols: int, width: int = 8) -> "DistMatrix":
        return cls(rows, cols, width)

    @classmethod
    def identity(cls, dim: int, width: int = 8) -> "DistMatrix":
        if dim < 1:
            raise ValueError(f"matrix dimensions must be positive, got {dim}x{dim}")
        host = np.full((dim, -(-dim // LANES[width]) * LANES[width]), sat_limit(width),
                       dtype=dtype_for(width))
        host[np.arange(dim), np.arange(dim)] = 0
        return cls(dim, dim, width, host)

    @classmethod
    def from_edges(cls, dim: int, edges, width: int = 8) -> "DistMatrix":
        """Edge weights stored directly; parallel edges keep the minimum
        (antidist.py:294-309).  Built on the device (smx_from_edges)."""
        return _from_edges(cls, dim, edges, width)

    def __mul__(self, other) -> "DistMatrix":
        """min over k of the saturating sum (antidist.py:311-329)."""
        if not isinstance(other, DistMatrix):
            return NotImplemented
        self._mul_checks(other)
        return self._mul(other, anti=False)
