"""GPU parity of the E2M1-nibble Boolean product (tcgen05 kind::mxf4).

BoolMatrix.__mul__ (pkg/src/semimat/boolmat.py:151-172) is the count > 0
threshold of a 0/1 contraction; on nibble operands (1.0 = 0b0010, scale
factors 1.0) the f32 counts are exact and the threshold gives the same bits
as the kind::i8 product and the oracle.  Exact equality throughout.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_1705_08743_b200 import BoolMatrix, _native
from paper_1705_08743_b200 import batch as batch_mod

pytestmark = pytest.mark.gpu


def _round16(x):
    return -(-x // 16) * 16


def _words(bits: np.ndarray, extra: int = 0) -> torch.Tensor:
    """0/1 rows -> LSB-first u32 words on the device (extra pad words)."""
    rows, cols = bits.shape
    nw = (cols + 31) // 32 + extra
    padded = np.zeros((rows, nw * 32), dtype=np.uint8)
    padded[:, :cols] = bits
    w = np.packbits(padded, axis=1, bitorder="little").view(np.uint32)
    return torch.from_numpy(w.view(np.int32).copy()).cuda()


def _nibbles(bits: np.ndarray, ld: int) -> np.ndarray:
    """0/1 rows -> E2M1 nibble rows (bit k -> nibble k, low nibble first)."""
    rows, cols = bits.shape
    v = np.zeros((rows, 2 * ld), dtype=np.uint8)
    v[:, :cols] = bits * 2
    return (v[:, 0::2] | (v[:, 1::2] << 4)).astype(np.uint8)


def _unpack_out(c: torch.Tensor, n: int) -> np.ndarray:
    got = c.cpu().numpy().view(np.uint32)
    return np.unpackbits(got.view(np.uint8), axis=1, bitorder="little")[:, :n].astype(bool)


@pytest.mark.parametrize("shape", [(100, 77, 33), (256, 1000, 129), (64, 40, 1)])
def test_unpack_nibbles_layout(shape):
    """smx_unpack_nibbles: A rows and the transposed B operand, ragged sizes
    (bits past cols in the input words are ignored; bytes past ceil(cols/2)
    are left alone)."""
    m, k, n = shape
    lib = _native.lib()
    rng = np.random.default_rng(m * k + n)
    a = (rng.random((m, k)) < 0.4).astype(np.uint8)
    b = (rng.random((k, n)) < 0.4).astype(np.uint8)
    aw = _words(a, extra=1)
    bw = _words(b, extra=1)
    aw_np = aw.cpu().numpy()
    aw_np[:, -1] = -1                                  # garbage past the columns
    aw = torch.from_numpy(aw_np).cuda()
    ld = _round16((k + 1) // 2) + 16
    an = torch.full((m, ld), 0xAB, dtype=torch.uint8, device="cuda")
    bt = torch.full((n, ld), 0xAB, dtype=torch.uint8, device="cuda")
    _native.check(lib.smx_unpack_nibbles(aw.data_ptr(), an.data_ptr(), m, k, aw.shape[1], ld, bw.data_ptr(),
                                         bt.data_ptr(), k, n, bw.shape[1], ld, _native.stream_ptr()), "nib")
    kb = (k + 1) // 2
    np.testing.assert_array_equal(an.cpu().numpy()[:, :kb], _nibbles(a, ld)[:, :kb])
    np.testing.assert_array_equal(bt.cpu().numpy()[:, :kb], _nibbles(np.ascontiguousarray(b.T), ld)[:, :kb])
    assert (an.cpu().numpy()[:, kb + 16:] == 0xAB).all()


# (smx_set_tc_pair, smx_set_tc_tile_n): automatic, the plain kernel at each
# tile width, the forced pair and the quad
_CONFIGS = [(1, 0), (0, 0), (0, 64), (0, 128), (0, 256), (2, 0), (3, 0)]


@pytest.mark.parametrize("shape", [(1024, 1024, 1024), (1000, 777, 1001), (130, 100, 129), (256, 256, 3000),
                                   (64, 2000, 384), (128, 128, 1), (300, 64, 513), (520, 333, 1537),
                                   (2048, 2048, 2048), (1300, 2100, 777), (128, 256, 40000),
                                   (1024, 1024, 65536 + 512)])
def test_gemm_f4_matches_i8_and_numpy(shape, oracle_lib):
    """smx_bool_gemm_f4 on nibble operands, on every kernel configuration:
    plain and OR-accumulating into a random output, ragged M / N / K (odd K:
    the last byte's high nibble is zero), K past the 6-stage ring, long thin
    products (split K with atomic OR), K past the i8 path's 65536 limit;
    padding words past N untouched."""
    m, n, k = shape
    lib = _native.lib()
    rng = np.random.default_rng(11 * m + n + k)
    dens = 0.03 if k < 10000 else 0.0005
    a = (rng.random((m, k)) < dens).astype(np.uint8)
    b = (rng.random((k, n)) < dens).astype(np.uint8)
    want = (a.astype(np.float32) @ b.astype(np.float32)) > 0
    ld = _round16((k + 1) // 2)
    A = torch.from_numpy(_nibbles(a, ld)).cuda()
    Bt = torch.from_numpy(_nibbles(np.ascontiguousarray(b.T), ld)).cuda()
    ldc = (n + 31) // 32 + 2
    init = rng.integers(0, 2 ** 32, (m, ldc), dtype=np.uint64).astype(np.uint32)
    nw = (n + 31) // 32
    prev = np.unpackbits(init.view(np.uint8), axis=1, bitorder="little")[:, :n].astype(bool)
    old_pair, old_tile = lib.smx_set_tc_pair(1), lib.smx_set_tc_tile_n(0)
    try:
        for pair, tile in _CONFIGS:
            lib.smx_set_tc_pair(pair)
            lib.smx_set_tc_tile_n(tile)
            for acc in (0, 1):
                C = torch.from_numpy(init.view(np.int32).copy()).cuda()
                _native.check(lib.smx_bool_gemm_f4(A.data_ptr(), Bt.data_ptr(), C.data_ptr(), m, n, k, ld, ld, ldc,
                                                   acc, _native.stream_ptr()), "f4")
                np.testing.assert_array_equal(_unpack_out(C, n), want | prev if acc else want,
                                              err_msg=f"acc={acc} pair={pair} tile={tile} {shape}")
                np.testing.assert_array_equal(C.cpu().numpy().view(np.uint32)[:, nw:], init[:, nw:])
    finally:
        lib.smx_set_tc_pair(old_pair)
        lib.smx_set_tc_tile_n(old_tile)
    if k <= 4096:
        want_bits = oracle_lib.bool_mul(oracle_lib.pack_bits(a), oracle_lib.pack_bits(b), k)
        ma, mb = BoolMatrix.from_numpy(a), BoolMatrix.from_numpy(b)
        old = lib.smx_set_tc_f4(1)
        try:
            for f4 in (1, 0):
                lib.smx_set_tc_f4(f4)
                np.testing.assert_array_equal((ma * mb).blocks, want_bits, err_msg=f"public f4={f4} {shape}")
        finally:
            lib.smx_set_tc_f4(old)
    assert lib.smx_set_tc_f4(2) < 0


def test_gemm_f4_all_ones_counts():
    """Dense operands (every count = K, up to 4096): the f32 accumulator and
    the upper-half threshold see large counts; a single nonzero product per
    output (count 1) still sets the bit."""
    lib = _native.lib()
    m = n = 256
    for k in (4096, 257):
        a = np.ones((m, k), dtype=np.uint8)
        b = np.ones((k, n), dtype=np.uint8)
        ld = _round16((k + 1) // 2)
        A = torch.from_numpy(_nibbles(a, ld)).cuda()
        Bt = torch.from_numpy(_nibbles(b.T.copy(), ld)).cuda()
        C = torch.zeros((m, n // 32), dtype=torch.int32, device="cuda")
        _native.check(lib.smx_bool_gemm_f4(A.data_ptr(), Bt.data_ptr(), C.data_ptr(), m, n, k, ld, ld, n // 32, 0,
                                           _native.stream_ptr()), "f4 ones")
        assert _unpack_out(C, n).all()
    # permutation: row i of A has one bit at k = (7 i) % K, B = identity: C = A
    k = 256
    a = np.zeros((m, k), dtype=np.uint8)
    a[np.arange(m), (7 * np.arange(m)) % k] = 1
    b = np.eye(k, n, dtype=np.uint8)
    ld = _round16(k // 2)
    A = torch.from_numpy(_nibbles(a, ld)).cuda()
    Bt = torch.from_numpy(_nibbles(b.T.copy(), ld)).cuda()
    C = torch.zeros((m, n // 32), dtype=torch.int32, device="cuda")
    _native.check(lib.smx_bool_gemm_f4(A.data_ptr(), Bt.data_ptr(), C.data_ptr(), m, n, k, ld, ld, n // 32, 0,
                                       _native.stream_ptr()), "f4 perm")
    np.testing.assert_array_equal(_unpack_out(C, n), a.astype(bool))


@pytest.mark.parametrize("batch,m,k,n", [(5, 256, 300, 384), (16, 1024, 1024, 1024), (3, 128, 129, 128)])
def test_batched_f4_matches_i8(batch, m, k, n):
    """smx_bool_mul_tc_batched on nibbles (default) and on bytes: identical."""
    rng = np.random.default_rng(batch + 3 * k)
    ma = [BoolMatrix.from_numpy(rng.random((m, k)) < 0.03) for _ in range(batch)]
    mb = [BoolMatrix.from_numpy(rng.random((k, n)) < 0.03) for _ in range(batch)]
    lib = _native.lib()
    old = lib.smx_set_tc_f4(1)
    old_ks = lib.smx_set_tc_batch_ks(2)
    old_st = lib.smx_set_tc_f4_batch_stages(2)
    try:
        lib.smx_set_tc_f4(0)
        want = [x.blocks for x in batch_mod.bool_mul_many(ma, mb)]
        for f4, ks, st in ((0, 1, 2), (1, 2, 2), (1, 1, 2), (1, 1, 3), (1, 2, 3), (1, 4, 2)):
            lib.smx_set_tc_f4(f4)
            lib.smx_set_tc_batch_ks(ks)
            lib.smx_set_tc_f4_batch_stages(st)
            got = [x.blocks for x in batch_mod.bool_mul_many(ma, mb)]
            for i in range(batch):
                np.testing.assert_array_equal(got[i], want[i], err_msg=f"product {i} f4={f4} ks={ks} st={st}")
    finally:
        lib.smx_set_tc_f4(old)
        lib.smx_set_tc_batch_ks(old_ks)
        lib.smx_set_tc_f4_batch_stages(old_st)
    assert lib.smx_set_tc_f4_batch_stages(4) < 0
