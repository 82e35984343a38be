"""GPU parity of the host-buffer closure (smx_fw_host_*, fw.cu fw_host_run).

The call copies rows in group by group and closes them as they arrive
(ingest: one catch-up product of K = rows already closed), closes the last
four pivot blocks alone and finishes every other row with one product of
K = |L| (egress) whose chunks are copied out while the rest runs.  Its result
must be bit-identical to the reference: the oracle at small n, the
reference's own output digests at the BASELINE config sizes, and the
device-resident closure at full size.  Exact equality throughout.
"""

from __future__ import annotations

import contextlib
import hashlib

import numpy as np
import pytest
import torch

from paper_1705_08743_b200 import AntidistMatrix, DistMatrix, _native, workloads

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@contextlib.contextmanager
def stream_mode(mode: int):
    """smx_set_fw_host_stream: 2 streams from 8 pivot blocks on, so that small
    n exercise the streamed schedule; 1 is the automatic default."""
    lib = _native.lib()
    old = lib.smx_set_fw_host_stream(mode)
    try:
        yield
    finally:
        lib.smx_set_fw_host_stream(old)


@pytest.fixture(params=[2, 0], ids=["streamed", "serial"])
def mode(request):
    with stream_mode(request.param):
        yield request.param


def host_closure(cls, t: np.ndarray, width: int, pinned: bool = True):
    src = torch.from_numpy(np.ascontiguousarray(t))
    if pinned:
        src = src.pin_memory()
    m, res = cls.closure_of_host(src, width)
    torch.cuda.synchronize()
    return m, res.numpy()


def random_graph(n, width, density, rng):
    lim = (1 << width) - 1
    lanes = 128 // width
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32}[width]
    host = np.zeros((n, -(-n // lanes) * lanes), dtype=dt)
    w = rng.integers(1, min(lim, 1000) + 1, size=(n, n))
    host[:, :n] = np.where(rng.random((n, n)) < density, lim - w, 0).astype(dt)
    return host


@pytest.mark.parametrize("n", [300, 897, 1000, 2048, 3000, 5000])
@pytest.mark.parametrize("kind", ["anti", "dist"])
def test_host_closure_matches_oracle_u16(n, kind, mode, oracle_lib):
    """Below 8 pivot blocks the call runs copy-in / closure / copy-out; from 8
    blocks on (n > 896 at the 128 block) mode 2 streams.  Ragged n included."""
    rng = np.random.default_rng(n)
    t = random_graph(n, 16, 0.02, rng)
    cls = AntidistMatrix
    if kind == "dist":
        t = (65535 - t.astype(np.uint32)).astype(np.uint16)   # complement: the DistMatrix view
        cls = DistMatrix
    want = oracle_lib.semiring_close(t, 16, kind)
    m, got = host_closure(cls, t, 16)
    np.testing.assert_array_equal(got, want, err_msg=f"n={n} {kind}")
    np.testing.assert_array_equal(m.data, want)          # the device copy holds the closure too


@pytest.mark.parametrize("width,n", [(8, 1500), (8, 2048), (32, 1000)])
def test_host_closure_other_widths(width, n, mode, oracle_lib):
    rng = np.random.default_rng(width * n)
    t = random_graph(n, width, 0.03, rng)
    _, got = host_closure(AntidistMatrix, t, width)
    np.testing.assert_array_equal(got, oracle_lib.semiring_close(t, width, "anti"))


@pytest.mark.parametrize("block,n", [(256, 2100), (512, 4100), (128, 1200)])
def test_host_closure_block_sizes(block, n, mode, oracle_lib):
    lib = _native.lib()
    old = lib.smx_set_fw_block(block)
    try:
        rng = np.random.default_rng(block + n)
        t = random_graph(n, 16, 0.01, rng)
        _, got = host_closure(AntidistMatrix, t, 16)
    finally:
        lib.smx_set_fw_block(old)
    np.testing.assert_array_equal(got, oracle_lib.semiring_close(t, 16, "anti"))


def test_host_closure_in_place_and_pageable(mode, oracle_lib):
    """host_out may be host_in; pageable input still gives the same bytes."""
    rng = np.random.default_rng(3)
    t = random_graph(2500, 16, 0.02, rng)
    want = oracle_lib.semiring_close(t, 16, "anti")
    _, got = host_closure(AntidistMatrix, t, 16, pinned=False)
    np.testing.assert_array_equal(got, want)
    buf = torch.from_numpy(t.copy()).pin_memory()
    AntidistMatrix.closure_of_host(buf, 16, out=buf)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(buf.numpy(), want)


@pytest.mark.parametrize("layout", ["pageable_in_place", "pageable_out", "pinned_in_pageable_out"])
def test_host_closure_pageable_out_staged(layout):
    """A pageable host_out is staged back through the page-locked ring
    (HostEgress, host_stage.cu): n = 8192 u16 streamed (128 MB: the egress
    runs through every 64 MB slot, after the ingest has used them), in place
    on the caller's own array, into a separate pageable array, and from a
    page-locked input; equal to the device-resident closure."""
    cfg = workloads.CONFIGS["c4_fw_u16"]
    (t,) = workloads.make_inputs(cfg, 8192)
    want = sha(AntidistMatrix(8192, 8192, 16, torch.from_numpy(t).cuda()).transitive_closure()._data.cpu().numpy())
    src = torch.from_numpy(t.copy())
    if layout == "pinned_in_pageable_out":
        src = src.pin_memory()
    out = src if layout == "pageable_in_place" else torch.from_numpy(np.full_like(t, 7))
    with stream_mode(2):
        for _ in range(2):
            if layout == "pageable_in_place":
                out.copy_(torch.from_numpy(t))
            AntidistMatrix.closure_of_host(src, 16, out=out)
            torch.cuda.synchronize()
            assert sha(out.numpy()) == want, layout
    if layout != "pageable_in_place":
        assert sha(src.numpy()) == sha(t)                 # the input is untouched


def test_host_closure_rejects_bad_shapes():
    with pytest.raises(ValueError):
        AntidistMatrix.closure_of_host(torch.zeros((10, 10), dtype=torch.uint16), 16)   # not padded
    with pytest.raises(ValueError):
        AntidistMatrix.closure_of_host(torch.zeros((16, 16), dtype=torch.uint8), 16)    # wrong dtype


@pytest.mark.parametrize("name", ["c4_fw_u16", "c5_fw_u16"])
def test_host_closure_matches_reference_digest(config_digests, name, mode):
    """C4 at n = 1024 and 8192, C5 at n = 2048: the reference's own output sha256."""
    cfg = workloads.CONFIGS[name]
    seen = 0
    for d in config_digests:
        if d["config"] != name:
            continue
        (t,) = workloads.make_inputs(cfg, d["n"])
        _, got = host_closure(AntidistMatrix, t, cfg.width)
        assert sha(got) == d["output_sha256"], (name, d["n"])
        seen += 1
    assert seen >= 1


def test_host_closure_full_size_matches_device_closure():
    """C5 generator at n = 16384 (512 blocks: groups 1024 / 4096 / 14336 + the
    last 2048 rows; streamed by the automatic mode): identical to the
    device-resident closure."""
    cfg = workloads.CONFIGS["c5_fw_u16"]
    n = 16384
    (t,) = workloads.make_inputs(cfg, n)
    dev = AntidistMatrix(n, n, 16, torch.from_numpy(t).cuda()).transitive_closure()
    _, got = host_closure(AntidistMatrix, t, 16)
    assert np.array_equal(got, dev.data)


@pytest.mark.parametrize("n", [700, 2048])
@pytest.mark.parametrize("kind", ["anti", "dist"])
def test_dropin_host_backed_closure(n, kind, mode, oracle_lib):
    """The reference's literal call on an ordinary (pageable) numpy array:
    ``AntidistMatrix(n, n, 16, arr).transitive_closure().data``.  The matrix
    is host-backed (its ``.data`` is a read-only view of ``arr``, as the
    reference's is, antidist.py:68-73), the closure runs as one host-buffer
    call whose input is staged through page-locked slots (host_stage.cuh),
    and the result is host-backed page-locked memory.  In-place
    ``transitive_close()`` writes the caller's array, as the reference's
    in-place sweep over ``_data`` does."""
    rng = np.random.default_rng(n + 17)
    t = random_graph(n, 16, 0.03, rng)
    cls = AntidistMatrix
    if kind == "dist":
        t = (65535 - t.astype(np.uint32)).astype(np.uint16)
        cls = DistMatrix
    keep = t.copy()
    want = oracle_lib.semiring_close(t, 16, kind)
    m = cls(n, n, 16, t)
    assert m.host_backed and np.shares_memory(m.data, t) and not m.data.flags.writeable
    r = m.transitive_closure()
    assert r.host_backed
    np.testing.assert_array_equal(r.data, want, err_msg=f"n={n} {kind}")
    np.testing.assert_array_equal(t, keep)                      # closure() leaves the input alone
    assert m.host_backed
    np.testing.assert_array_equal((m * m).data, oracle_lib.semiring_mul(keep, keep, n, 16, kind))
    assert not m.host_backed                                    # the product moved it to HBM
    m2 = cls(n, n, 16, t)
    m2.transitive_close()                                       # in place: the caller's array
    np.testing.assert_array_equal(t, want)
    assert m2.host_backed and m2.get(3, 5) == int(want[3, 5])


def test_dropin_staged_ring_reuse_matches_device_closure():
    """n = 8192 u16 (128 MB, several 64 MB staging slots), twice in a row
    (the ring's slots reused across calls), streamed; equal to the
    device-resident closure of the same input and to the C4 reference digest
    path's generator output shape."""
    cfg = workloads.CONFIGS["c4_fw_u16"]
    (t,) = workloads.make_inputs(cfg, 8192)
    dev = AntidistMatrix(8192, 8192, 16, torch.from_numpy(t).cuda()).transitive_closure()
    want = dev._data.cpu().numpy()
    with stream_mode(2):
        for _ in range(2):
            got = AntidistMatrix(8192, 8192, 16, t).transitive_closure()
            assert got.host_backed
            assert sha(got.data) == sha(want)


@pytest.mark.parametrize("width,kind,shape", [(16, "anti", (6000, 3000, 2050)), (8, "dist", (4096, 4096, 4096)),
                                              (32, "anti", (9000, 2000, 1300))])
def test_streamed_host_product_matches_device(width, kind, shape):
    """A large host-backed left operand takes the streamed host product (row
    groups staged in while the previous group's product runs, results copied
    out into page-locked memory): the result is host-backed and equals the
    device-resident product of the same operands, ragged shapes included."""
    m, k, n = shape
    rng = np.random.default_rng(m + n)
    lim = (1 << width) - 1
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32}[width]
    cls = AntidistMatrix if kind == "anti" else DistMatrix
    pad = 128 // width

    def rnd(r, c):
        a = np.full((r, -(-c // pad) * pad), 0 if kind == "anti" else lim, dtype=dt)
        v = rng.integers(1, min(lim, 1000), (r, c))
        keep = rng.random((r, c)) < 0.3
        a[:, :c] = np.where(keep, (lim - v) if kind == "anti" else v, a[:, :c]).astype(dt)
        return a

    a, b = rnd(m, k), rnd(k, n)
    ha, hb = cls(m, k, width, a), cls(k, n, width, b)
    assert ha.rows * ha.padded_cols >= cls._HOST_MUL_MIN
    got = ha * hb
    assert got.host_backed
    want = cls(m, k, width, torch.from_numpy(a).cuda()) * cls(k, n, width, torch.from_numpy(b).cuda())
    assert not want.host_backed
    np.testing.assert_array_equal(got.data, want.data)
    np.testing.assert_array_equal(ha.data, a)    # the inputs are untouched
