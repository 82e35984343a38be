"""CPU oracle for the semimat hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
the timed CPU baseline -- never as the product path.  The product package
(`paper_1705_08743_b200`) has no import of it and no CPU fallback.

Two restatements of the reference (arxiv/paper_1705_08743, package semimat):

* ``semimat_oracle.c`` (built to ``_build/libsemimat_oracle.so``): the
  reference's numpy "vector path" engines restated in C with OpenMP row
  parallelism (see the file header for file:line citations).  Fast enough for
  the bench configs' oracle sizes (C1-C3 full size, FW at n <= 2048).
* ``naive.py``: the reference's independent pure-Python oracles
  (pkg/src/semimat/oracle.py) restated for tiny cases.

Parity of both with the reference is pinned by tests/test_oracle_golden.py
against vectors produced by the reference itself (tests/golden/).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_build" / "libsemimat_oracle.so"

_SUFFIX = {8: "u8", 16: "u16", 32: "u32"}
_DTYPE = {8: np.uint8, 16: np.uint16, 32: np.uint32}
_lib = None


def build() -> Path:
    """Compile the C oracle with the committed Makefile (idempotent)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        lib = ctypes.CDLL(str(LIB_PATH))
        i64, u32, ci, vp = ctypes.c_int64, ctypes.c_uint32, ctypes.c_int, ctypes.c_void_p
        for suf in _SUFFIX.values():
            for name in (f"orc_anti_mul_{suf}", f"orc_minplus_mul_{suf}"):
                fn = getattr(lib, name)
                fn.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i64, u32, ci]
                fn.restype = None
            for name in (f"orc_anti_close_{suf}", f"orc_minplus_close_{suf}",
                         f"orc_anti_close_blocked_{suf}", f"orc_minplus_close_blocked_{suf}"):
                fn = getattr(lib, name)
                fn.argtypes = [vp, i64, i64, i64, u32, ci]
                fn.restype = None
        lib.orc_bool_mul.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i64, ci]
        lib.orc_bool_mul.restype = None
        lib.orc_bool_close.argtypes = [vp, i64, i64, i64, ci]
        lib.orc_bool_close.restype = None
        lib.orc_max_threads.restype = ci
        _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().orc_max_threads())


def _limit(width: int) -> int:
    return (1 << width) - 1


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _lane(a: np.ndarray, width: int) -> np.ndarray:
    a = np.ascontiguousarray(a)
    if a.dtype != _DTYPE[width]:
        raise TypeError(f"expected {_DTYPE[width].__name__}, got {a.dtype}")
    return a


def semiring_mul(a: np.ndarray, b: np.ndarray, inner: int, width: int, kind: str,
                 threads: int = 0) -> np.ndarray:
    """Product of padded lane arrays a (R x Kpad) and b (inner x Cpad).

    kind "anti" restates _mul_vector (antidist.py:361-371), kind "dist"
    restates _minplus_mul_vector (antidist.py:412-422).  Returns R x Cpad.
    """
    a, b = _lane(a, width), _lane(b, width)
    rows, cols = a.shape[0], b.shape[1]
    out = np.empty((rows, cols), dtype=_DTYPE[width])
    name = ("orc_anti_mul_" if kind == "anti" else "orc_minplus_mul_") + _SUFFIX[width]
    getattr(_load(), name)(_ptr(a), _ptr(b), _ptr(out), rows, inner, cols,
                           a.shape[1], b.shape[1], cols, _limit(width), threads)
    return out


def semiring_close(t: np.ndarray, width: int, kind: str, threads: int = 0) -> np.ndarray:
    """Closure of a square padded lane array (D x Dpad); returns a new array.

    kind "anti" restates _close_vector (antidist.py:390-398), "dist" restates
    _minplus_close_vector (antidist.py:440-448).
    """
    out = np.array(_lane(t, width), copy=True)
    name = ("orc_anti_close_" if kind == "anti" else "orc_minplus_close_") + _SUFFIX[width]
    getattr(_load(), name)(_ptr(out), out.shape[0], out.shape[1], out.shape[1],
                           _limit(width), threads)
    return out


def semiring_close_blocked(t: np.ndarray, width: int, kind: str, threads: int = 0) -> np.ndarray:
    """The same closure as ``semiring_close`` in the cache-blocked three-phase
    order (semimat_oracle.c, DEFINE_CLOSE_BLOCKED): bit-identical to the
    reference's sweep (pinned by
    tests/test_oracle_golden.py), fast enough for the full-size C5 pin."""
    out = np.array(_lane(t, width), copy=True)
    name = ("orc_anti_close_blocked_" if kind == "anti" else "orc_minplus_close_blocked_") + _SUFFIX[width]
    getattr(_load(), name)(_ptr(out), out.shape[0], out.shape[1], out.shape[1],
                           _limit(width), threads)
    return out


def bool_mul(a_blocks: np.ndarray, b_blocks: np.ndarray, inner: int,
             threads: int = 0) -> np.ndarray:
    """Boolean product on uint64 block storage (boolmat.py:151-172)."""
    a = np.ascontiguousarray(a_blocks, dtype=np.uint64)
    b = np.ascontiguousarray(b_blocks, dtype=np.uint64)
    out = np.empty((a.shape[0], b.shape[1]), dtype=np.uint64)
    _load().orc_bool_mul(_ptr(a), _ptr(b), _ptr(out), a.shape[0], inner, b.shape[1],
                         a.shape[1], b.shape[1], b.shape[1], threads)
    return out


def bool_close(blocks: np.ndarray, threads: int = 0) -> np.ndarray:
    """Warshall transitive closure on uint64 block storage (boolmat.py:174-189)."""
    out = np.array(np.ascontiguousarray(blocks, dtype=np.uint64), copy=True)
    _load().orc_bool_close(_ptr(out), out.shape[0], out.shape[1], out.shape[1], threads)
    return out


def pack_bits(bits: np.ndarray) -> np.ndarray:
    """0/1 array (R x C) -> uint64 blocks (R x ceil(C/64)), LSB first (boolmat.py:3-5)."""
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    rows, cols = bits.shape
    nblk = -(-cols // 64)
    padded = np.zeros((rows, nblk * 64), dtype=np.uint8)
    padded[:, :cols] = bits
    return np.packbits(padded, axis=1, bitorder="little").view("<u8").astype(np.uint64)


def unpack_bits(blocks: np.ndarray, cols: int) -> np.ndarray:
    """uint64 blocks -> 0/1 uint8 array (R x cols)."""
    raw = np.ascontiguousarray(blocks).astype("<u8").view(np.uint8)
    raw = raw.reshape(blocks.shape[0], -1)
    return np.unpackbits(raw, axis=1, bitorder="little")[:, :cols]
