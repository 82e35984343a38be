"""The reference's acceptance criteria 1, 2, 3 and 5, run against the GPU path.

Ports of pkg/tests/test_acceptance.py (criterion 1 :28-57, 2 :60-85,
3 :88-116, 5 :153-201): same generators, seeds, sizes and trial counts, with
the reference's BoolMatrix / AntidistMatrix / kernels swapped for this
package's device classes.  The oracles are the pinned restatements in
oracle/naive.py (tests/test_oracle_golden.py ties them to the reference).
Every comparison is exact: all arithmetic on this path is integer.

Each criterion runs both through the batched kernels (csrc/lanes.cu, one
launch for the whole suite) and through the public per-matrix calls, so the
drop-in path itself is covered, not only the batch entry points.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import naive
from paper_1705_08743_b200 import AntidistMatrix, BoolMatrix, batch, kernels
from paper_1705_08743_b200.scalars import sat_limit

pytestmark = pytest.mark.gpu

WIDTHS = (8, 16, 32)


def _pack_rows(rows):
    return tuple(sum(v << j for j, v in enumerate(row)) for row in rows)


# -- criterion 1: exhaustive 3x3 Boolean products and closures ----------------

def test_criterion_1_exhaustive_3x3():
    dense = [[[(bits >> (3 * r + c)) & 1 for c in range(3)] for r in range(3)] for bits in range(512)]
    mats = [BoolMatrix.from_lists(g) for g in dense]
    words = torch.stack([m._words for m in mats])                      # (512, 3, 4)
    ia = torch.arange(512, device=words.device).repeat_interleave(512)
    ib = torch.arange(512, device=words.device).repeat(512)
    out = batch.bool_mul_stacked(words[ia], words[ib], 3, 3)           # 262,144 products, one launch
    sig = out[:, :, 0].cpu().numpy().astype(np.int64) & 0xFFFFFFFF
    expected = {}
    mismatch = 0
    for x in range(512):
        for y in range(512):
            key = _pack_rows(naive.bool_product(dense[x], dense[y]))
            expected[(x, y)] = key
            if tuple(int(v) for v in sig[x * 512 + y]) != key:
                mismatch += 1
    assert mismatch == 0
    # the public BoolMatrix.__mul__ on a seeded sample of the same pairs
    rng = np.random.default_rng(1)
    for x, y in rng.integers(0, 512, size=(1024, 2)).tolist():
        got = mats[x] * mats[y]
        assert tuple(int(w) for w in got.blocks[:, 0]) == expected[(x, y)]
    # 512 closures vs repeated squaring and walk enumeration, batched and public
    closed = batch.bool_closure_many(mats)
    for g, m, c in zip(dense, mats, closed):
        want = _pack_rows(naive.closure_by_squaring(g))
        assert want == _pack_rows(naive.walk_closure(g))
        assert tuple(int(w) for w in c.blocks[:, 0]) == want
        assert tuple(int(w) for w in m.transitive_closure().blocks[:, 0]) == want


# -- criterion 2: random digraphs vs Dijkstra -----------------------------------

@pytest.mark.parametrize("width", WIDTHS)
def test_criterion_2_random_closure_vs_dijkstra(width):
    limit = sat_limit(width)
    rng = np.random.default_rng(1000 + width)
    graphs = []
    for _ in range(500):
        dim = int(rng.integers(2, 65))
        p = float(rng.uniform(0.1, 0.5))
        mask = rng.random((dim, dim)) < p
        np.fill_diagonal(mask, False)
        us, vs = np.nonzero(mask)
        ws = rng.integers(1, 11, size=us.size)
        graphs.append((dim, list(zip(us.tolist(), vs.tolist(), ws.tolist()))))
    mismatch = 0
    by_dim: dict[int, list] = {}
    for dim, edges in graphs:
        m = AntidistMatrix.from_edges(dim, edges, width)
        want = naive.apsp_antidist(dim, edges, limit)
        if m.transitive_closure().to_lists() != want:       # the public call
            mismatch += 1
        by_dim.setdefault(dim, []).append((m, want))
    for dim, items in by_dim.items():                        # batched, one launch per size
        for (m, want), c in zip(items, batch.closure_many([m for m, _ in items])):
            if c.to_lists() != want:
                mismatch += 1
    assert mismatch == 0


# -- criterion 3: De Morgan dualities --------------------------------------------

@pytest.mark.parametrize("width", WIDTHS)
def test_criterion_3_de_morgan(width):
    limit = sat_limit(width)
    rng = np.random.default_rng(3000 + width)

    def rand(rows, cols):
        grid = rng.integers(0, limit + 1, size=(rows, cols))
        grid[rng.random((rows, cols)) < 0.25] = 0
        return AntidistMatrix.from_lists(grid.tolist(), width)

    mismatch = 0
    for _ in range(1000):
        rows, inner, cols = (int(x) for x in rng.integers(1, 13, size=3))
        a, a2 = rand(rows, inner), rand(rows, inner)
        b = rand(inner, cols)
        if ~(a | a2) != ((~a) & (~a2)):
            mismatch += 1
        if ~(a * b) != ((~a) * (~b)):
            mismatch += 1
        square = rand(inner, inner)
        if (~square).transitive_closure() != ~(square.transitive_closure()):
            mismatch += 1
    assert mismatch == 0


# -- criterion 5: lane kernels bit-exact, random and boundary blocks -----------

def _definitions(fn, a, b, limit):
    """The scalar path's definitions (kernels.py:147-189), on int64 numpy."""
    a, b = np.asarray(a, dtype=np.int64), np.asarray(b, dtype=np.int64)
    return {
        "subsat": np.maximum(a - b, 0),
        "addsat": np.minimum(a + b, limit),
        "maxlanes": np.maximum(a, b),
        "minlanes": np.minimum(a, b),
        "absdiff": np.abs(a - b),
    }[fn].tolist()


@pytest.mark.parametrize("width", WIDTHS)
def test_criterion_5_kernel_bit_exactness(width):
    limit = sat_limit(width)
    lanes = kernels.lane_count(width)
    rng = np.random.default_rng(5000 + width)
    blocks = 100_000
    a = rng.integers(0, limit + 1, size=blocks * lanes, dtype=np.uint64).tolist()
    b = rng.integers(0, limit + 1, size=blocks * lanes, dtype=np.uint64).tolist()
    boundary = (0, 1, limit - 1, limit)
    pat_a, pat_b = [], []
    for pos in range(lanes):
        for x in boundary:
            for y in boundary:
                for fill_a in (0, limit):
                    for fill_b in (0, limit):
                        row_a, row_b = [fill_a] * lanes, [fill_b] * lanes
                        row_a[pos], row_b[pos] = x, y
                        pat_a.extend(row_a)
                        pat_b.extend(row_b)
    for name in ("subsat", "addsat", "maxlanes", "minlanes", "absdiff"):
        fn = getattr(kernels, name)
        for x, y in ((a, b), (pat_a, pat_b)):
            with kernels.forced_vector():
                vec = fn(x, y, width)
            with kernels.forced_scalar():
                sca = fn(x, y, width)
            assert vec == sca == _definitions(name, x, y, limit), name
        # the boundary patterns once more against pure-Python per-lane definitions
        py = {"subsat": lambda p, q: p - q if p > q else 0,
              "addsat": lambda p, q: min(p + q, limit),
              "maxlanes": max, "minlanes": min, "absdiff": lambda p, q: abs(p - q)}[name]
        assert fn(pat_a, pat_b, width) == [py(p, q) for p, q in zip(pat_a, pat_b)], name
    clone_values = sorted({*boundary, *rng.integers(0, limit + 1, size=500).tolist()})
    for value in clone_values:
        assert kernels.clonenot(value, width) == [limit - value] * lanes
    assert kernels.clonenot(3, width, count=4 * lanes) == [limit - 3] * (4 * lanes)


def test_array_level_lane_forms_on_device():
    """np_subsat / np_addsat / np_absdiff with broadcasting (kernels.py:195-204):
    numpy in -> numpy out, CUDA tensors in -> CUDA tensor out."""
    rng = np.random.default_rng(7)
    for dt, limit in ((np.uint8, 255), (np.uint16, 65535), (np.uint32, 2**32 - 1)):
        a = rng.integers(0, limit + 1, size=(37, 19), dtype=np.uint64).astype(dt)
        g = rng.integers(0, limit + 1, size=(37, 1), dtype=np.uint64).astype(dt)
        np.testing.assert_array_equal(kernels.np_subsat(a, g), np.maximum(a, g) - g)
        np.testing.assert_array_equal(kernels.np_addsat(a, g, limit), np.minimum(a, limit - g) + g)
        np.testing.assert_array_equal(kernels.np_absdiff(a, g),
                                      np.bitwise_or(np.maximum(a, g) - g, np.maximum(g, a) - a))
        ta, tg = torch.from_numpy(a).cuda(), torch.from_numpy(g).cuda()
        got = kernels.np_subsat(ta, tg)
        assert got.is_cuda and got.shape == (37, 19)
        np.testing.assert_array_equal(got.cpu().numpy(), np.maximum(a, g) - g)


def test_bool_bridge_round_trip_on_device():
    """from_boolmat / to_boolmat run on the device (smx_lanes_*), every width,
    ragged widths straddling the word and lane-block boundaries."""
    rng = np.random.default_rng(11)
    for rows, cols in ((1, 1), (3, 33), (70, 65), (129, 200)):
        bits = (rng.random((rows, cols)) < 0.4).astype(np.uint8)
        bm = BoolMatrix.from_numpy(bits)
        for w in WIDTHS:
            am = AntidistMatrix.from_boolmat(bm, w)
            assert am.data.shape[1] % kernels.lane_count(w) == 0
            np.testing.assert_array_equal(am.data[:, :cols], bits.astype(am.data.dtype) * sat_limit(w))
            assert not am.data[:, cols:].any()                 # padding = 0
            assert am.to_boolmat() == bm
            assert am.to_boolmat().blocks.tobytes() == bm.blocks.tobytes()
