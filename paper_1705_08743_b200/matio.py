"""SRMAT1 binary and text serialization for the device matrices (SURVEY.md
8(f) item 3) -- the reference's format (pkg/src/semimat/matio.py), so files
written by either implementation load in the other.

Binary: a 16-byte header (magic ``SRMAT1``, a type byte, a width byte, row and
column counts as little-endian uint32) followed by the row-major payload:
packed 64-bit little-endian blocks for Boolean matrices (padding bits zero),
bare little-endian entries without padding for lane matrices
(matio.py:96-149).  Payloads move between the file bytes and HBM with one
strided copy each way; validation messages follow the reference.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np
import torch

from .antidist import LANES, AntidistMatrix, DistMatrix
from .boolmat import BoolMatrix, _block_count, _stride_words

MAGIC = b"SRMAT1"
_HEADER = struct.Struct("<6sBBII")
_TYPE_BOOL = ord("B")
_TYPE_ANTIDIST = ord("A")
_TYPE_DIST = ord("D")
_LANE_DTYPES = {8: "<u1", 16: "<u2", 32: "<u4"}


class MatrixFormatError(ValueError):
    """Unreadable or inconsistent matrix file content (matio.py:28-29)."""


def to_binary(m) -> bytes:
    """Header + payload of ``m`` (matio.py:101-110), read straight from HBM."""
    if isinstance(m, BoolMatrix):
        header = _HEADER.pack(MAGIC, _TYPE_BOOL, 0, m.rows, m.cols)
        words = m._words[:, : 2 * m.block_columns].contiguous().cpu().numpy()
        return header + words.astype("<i4", copy=False).tobytes()
    if isinstance(m, (AntidistMatrix, DistMatrix)):
        tag = _TYPE_ANTIDIST if isinstance(m, AntidistMatrix) else _TYPE_DIST
        header = _HEADER.pack(MAGIC, tag, m.width, m.rows, m.cols)
        if m.host_backed:   # (no round trip through HBM for a matrix still on its host array)
            entries = np.ascontiguousarray(m._host[:, : m.cols])
        else:
            entries = m._data[:, : m.cols].contiguous().cpu().numpy()
        return header + entries.astype(_LANE_DTYPES[m.width], copy=False).tobytes()
    raise TypeError(f"cannot serialize {type(m).__name__}")


def from_binary(data: bytes):
    """Parse SRMAT1 bytes into a device matrix (matio.py:113-149)."""
    if len(data) < _HEADER.size:
        raise MatrixFormatError(f"truncated header: {len(data)} bytes")
    magic, tag, width, rows, cols = _HEADER.unpack_from(data)
    if magic != MAGIC:
        raise MatrixFormatError(f"bad magic {magic!r}")
    if rows < 1 or cols < 1:
        raise MatrixFormatError(f"matrix dimensions must be positive, got {rows}x{cols}")
    payload = memoryview(data)[_HEADER.size:]
    if tag == _TYPE_BOOL:
        if width != 0:
            raise MatrixFormatError(f"bool matrices carry width byte 0, got {width}")
        bpr = _block_count(cols)
        expected = rows * bpr * 8
        if len(payload) != expected:
            raise MatrixFormatError(f"payload is {len(payload)} bytes, expected {expected}")
        blocks = np.frombuffer(payload, dtype="<u8").reshape(rows, bpr)
        tail = cols & 63
        if tail and int(blocks[:, -1].max(initial=0)) >> tail:
            raise MatrixFormatError("nonzero padding bits in final block")
        words = np.zeros((rows, _stride_words(cols)), dtype="<u4")
        words[:, : 2 * bpr] = blocks.view("<u4").reshape(rows, 2 * bpr)
        return BoolMatrix(rows, cols, torch.from_numpy(words.view(np.int32)).cuda())
    if tag in (_TYPE_ANTIDIST, _TYPE_DIST):
        if width not in _LANE_DTYPES:
            raise MatrixFormatError(f"unsupported width byte {width}")
        expected = rows * cols * (width // 8)
        if len(payload) != expected:
            raise MatrixFormatError(f"payload is {len(payload)} bytes, expected {expected}")
        cls = AntidistMatrix if tag == _TYPE_ANTIDIST else DistMatrix
        entries = np.frombuffer(payload, dtype=_LANE_DTYPES[width]).reshape(rows, cols)
        padded = -(-cols // LANES[width]) * LANES[width]
        host = np.full((rows, padded), cls._pad_fill(width), dtype=entries.dtype.newbyteorder("="))
        host[:, :cols] = entries
        return cls(rows, cols, width, host)
    raise MatrixFormatError(f"unknown type byte {tag:#x}")


def format_text(m) -> str:
    """Text form: header line then one line per row (matio.py:37-47)."""
    if isinstance(m, BoolMatrix):
        bits = m.to_numpy()
        body = ["".join("1" if v else "0" for v in row) for row in bits.tolist()]
        return "\n".join([f"bool {m.rows} {m.cols}", *body]) + "\n"
    if isinstance(m, (AntidistMatrix, DistMatrix)):
        kind = "antidist" if isinstance(m, AntidistMatrix) else "dist"
        body = [" ".join(str(v) for v in row) for row in m.to_lists()]
        return "\n".join([f"{kind} {m.width} {m.rows} {m.cols}", *body]) + "\n"
    raise TypeError(f"cannot format {type(m).__name__}")


def save(m, path, binary: bool = False) -> None:
    path = Path(path)
    if binary:
        path.write_bytes(to_binary(m))
    else:
        path.write_text(format_text(m))


def _ints(fields):
    try:
        return [int(f) for f in fields]
    except ValueError:
        raise MatrixFormatError(f"non-integer header field in {fields!r}") from None


def parse_text(text: str):
    """Text grammar and messages of matio.py:50-96; rows are bulk-converted
    with numpy and uploaded once."""
    lines = text.splitlines()
    if not lines or not lines[0].split():
        raise MatrixFormatError("empty input, expected a matrix header line")
    head = lines[0].split()
    kind = head[0]
    if kind == "bool":
        if len(head) != 3:
            raise MatrixFormatError("bool header must be 'bool R C'")
        rows, cols = _ints(head[1:])
        data = lines[1:rows + 1]
        for lineno, line in enumerate(data, start=2):
            row = line.strip()
            if len(row) != cols or row.strip("01"):
                raise MatrixFormatError(f"line {lineno}: expected {cols} characters of 0/1")
        if len(data) != rows:
            raise MatrixFormatError(f"expected {rows} data rows, found {len(data)}")
        if rows < 1 or cols < 1:
            raise ValueError("matrix dimensions must be positive")
        grid = np.frombuffer("".join(l.strip() for l in data).encode(), dtype=np.uint8) - ord("0")
        return BoolMatrix.from_numpy(grid.reshape(rows, cols))
    if kind in ("antidist", "dist"):
        if len(head) != 4:
            raise MatrixFormatError(f"{kind} header must be '{kind} W R C'")
        width, rows, cols = _ints(head[1:])
        cls = AntidistMatrix if kind == "antidist" else DistMatrix
        grid = []
        for lineno, line in enumerate(lines[1:rows + 1], start=2):
            parts = line.split()
            if len(parts) != cols:
                raise MatrixFormatError(f"line {lineno}: expected {cols} values, found {len(parts)}")
            try:
                grid.append([int(p) for p in parts])
            except ValueError:
                raise MatrixFormatError(f"line {lineno}: non-integer entry") from None
        if len(grid) != rows:
            raise MatrixFormatError(f"expected {rows} data rows, found {len(grid)}")
        try:
            return cls.from_lists(grid, width)
        except ValueError as exc:
            raise MatrixFormatError(str(exc)) from None
    raise MatrixFormatError(f"unknown matrix type {kind!r}")


def load(path):
    """Read a matrix file, binary (SRMAT1 magic) or text (matio.py:162-171)."""
    data = Path(path).read_bytes()
    if data.startswith(MAGIC):
        return from_binary(data)
    try:
        text = data.decode("utf-8")
    except UnicodeDecodeError as exc:
        raise MatrixFormatError(f"{path}: neither a binary matrix nor utf-8 text") from exc
    return parse_text(text)
