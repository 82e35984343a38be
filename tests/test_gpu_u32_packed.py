"""GPU parity of the u32 lanes on the packed phase-3 / product kernel
(semiring_packed.cuh with Lane<uint32_t>: one cell per word; kernels.py:35).

* closures at sizes that take the packed look-ahead schedule (n > one pivot
  block), with small weights (bounded tiles, certified first rounds) and with
  weights near 2^31 (the general two-instruction update, saturation at S);
* public products above the packed threshold (M*N >= 2^22, K >= 256) with
  certifiable and non-certifiable operands, both kinds;
* the sharded closure's certified update (smx_semiring_gemm_skip_certified,
  elem_bytes = 4) on the packed path;
* n = 8192 (the C4 size, 256-vertex blocks): the u32 closure equals the u16
  closure of the same graph, widened (no distance reaches 2^16 - 1 there).
Every comparison is exact equality against the C oracle or the u16 path.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_1705_08743_b200 import AntidistMatrix, DistMatrix, _native, workloads

pytestmark = pytest.mark.gpu

S32 = (1 << 32) - 1


def _graph(rng, n, p, wmax, kind):
    mask = rng.random((n, n)) < p
    w = rng.integers(1, wmax, size=(n, n), dtype=np.uint64)
    if kind == "anti":
        t = np.where(mask, S32 - w, 0)
    else:
        t = np.where(mask, w, S32)
    return t.astype(np.uint32)


@pytest.mark.parametrize("kind", ["anti", "dist"])
@pytest.mark.parametrize("wmax", [1000, 1 << 31])
@pytest.mark.parametrize("n", [640, 1100])
def test_u32_closure_packed_matches_oracle(kind, wmax, n, oracle_lib):
    rng = np.random.default_rng(n + (wmax & 0xFFFF))
    t = _graph(rng, n, 4.0 / n, wmax, kind)
    cls = AntidistMatrix if kind == "anti" else DistMatrix
    got = cls(n, n, 32, t).transitive_closure().data
    np.testing.assert_array_equal(got, oracle_lib.semiring_close_blocked(t, 32, kind))


@pytest.mark.parametrize("kind", ["anti", "dist"])
@pytest.mark.parametrize("wmax", [1000, 1 << 31])
def test_u32_product_packed_matches_oracle(kind, wmax, oracle_lib):
    rng = np.random.default_rng(wmax & 0xFFFF)
    m, k, n = 2048, 520, 2100     # ragged k and n: partial k-tile and column tile
    a = _graph(rng, max(m, k), 0.2, wmax, kind)[:m, :k].copy()
    b = _graph(rng, max(k, n), 0.2, wmax, kind)[:k, :n].copy()
    # lanes: u32 rows are padded to a multiple of 4
    ap = np.full((m, 520), 0 if kind == "anti" else S32, dtype=np.uint32)
    ap[:, :k] = a
    bp = np.full((k, 2100), 0 if kind == "anti" else S32, dtype=np.uint32)
    bp[:, :n] = b
    cls = AntidistMatrix if kind == "anti" else DistMatrix
    got = (cls(m, k, 32, ap) * cls(k, n, 32, bp)).data
    want = oracle_lib.semiring_mul(ap, bp, k, 32, kind)
    np.testing.assert_array_equal(got, want)


def test_u32_certified_skip_gemm_on_packed_path(oracle_lib):
    """M*N = 2^24 takes the packed path; rows [1024, 1280) are left alone."""
    lib = _native.lib()
    rng = np.random.default_rng(5)
    m = n = 4096
    k = 256
    a = _graph(rng, m, 0.05, 1000, "anti")[:, :k].copy()
    b = _graph(rng, m, 0.05, 1000, "anti")[:k, :].copy()
    c0 = _graph(rng, m, 0.01, 1000, "anti")
    want = np.maximum(c0, oracle_lib.semiring_mul(a, b, k, 32, "anti"))
    want[1024:1280] = c0[1024:1280]
    for fn in (lib.smx_semiring_gemm_skip_certified, lib.smx_semiring_gemm_skip):
        A, B, C = (torch.from_numpy(x.view(np.int32)).cuda() for x in (a, b, c0.copy()))
        rc = fn(A.data_ptr(), B.data_ptr(), C.data_ptr(), m, n, k, k, n, n, 4, _native.SMX_ANTI, 1024, 256,
                _native.stream_ptr())
        assert rc == 0
        np.testing.assert_array_equal(C.cpu().numpy().view(np.uint32), want)


def test_u32_c4_closure_equals_u16_closure():
    """n = 8192 on the C4 generator: 32 rounds of 256-vertex blocks with the
    packed u32 phase 3; distances stay far below 2^16 - 1, so the u32 closure
    is the u16 closure widened."""
    n = 8192
    (t16,) = workloads.make_inputs(workloads.CONFIGS["c4_fw_u16"], n)
    want16 = DistMatrix(n, n, 16, (65535 - t16).astype(np.uint16)).transitive_closure().data
    assert int(want16[want16 != 65535].max()) < 60000
    d32 = np.where(t16 == 0, S32, 65535 - t16.astype(np.uint64)).astype(np.uint32)
    got = DistMatrix(n, n, 32, d32).transitive_closure().data
    want = np.where(want16 == 65535, S32, want16.astype(np.uint64)).astype(np.uint32)
    np.testing.assert_array_equal(got, want)
