"""GPU parity: the sm_100a path through the reference-facing class API must be
bit-identical to the reference (golden vectors made by the reference itself)
and to the pinned CPU oracle.  All arithmetic is integer, so every comparison
is exact equality -- there is no tolerance anywhere in this file.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest
import torch

from paper_1705_08743_b200 import AntidistMatrix, BoolMatrix, DistMatrix, engines, workloads

pytestmark = pytest.mark.gpu

CLS = {"anti": AntidistMatrix, "dist": DistMatrix}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def lane(kind, data, cols, width):
    return CLS[kind](data.shape[0], cols, width, np.array(data))   # (a copy: the fixtures are shared)


# -- golden small cases: products, closures, Boolean ---------------------------

def test_small_products(small_cases):
    n = 0
    for meta, arr in small_cases:
        if meta["op"] != "mul":
            continue
        a = lane(meta["kind"], arr["a"], meta["inner"], meta["width"])
        b = lane(meta["kind"], arr["b"], meta["cols"], meta["width"])
        got = (a * b).data
        np.testing.assert_array_equal(got, arr["out"], err_msg=meta["name"])
        n += 1
    assert n >= 90


def test_small_closures(small_cases):
    for meta, arr in small_cases:
        if meta["op"] != "closure":
            continue
        m = lane(meta["kind"], arr["t"], meta["dim"], meta["width"])
        got = m.transitive_closure()
        np.testing.assert_array_equal(got.data, arr["out"], err_msg=meta["name"])
        assert m.data.tobytes() == arr["t"].tobytes()          # closure() leaves the input alone
        m.transitive_close()                                   # in-place variant agrees
        np.testing.assert_array_equal(m.data, arr["out"], err_msg=meta["name"])


def test_small_bool(small_cases):
    for meta, arr in small_cases:
        if meta["op"] == "bool_mul":
            got = BoolMatrix.from_numpy(arr["a"]) * BoolMatrix.from_numpy(arr["b"])
            np.testing.assert_array_equal(got.blocks, arr["out_blocks"], err_msg=meta["name"])
            assert got.to_lists() == arr["out"].tolist()
            bits = engines.bool_mul_bits(BoolMatrix.from_numpy(arr["a"]), BoolMatrix.from_numpy(arr["b"]))
            np.testing.assert_array_equal(bits.blocks, arr["out_blocks"], err_msg=meta["name"])
        elif meta["op"] == "bool_closure":
            m = BoolMatrix.from_numpy(arr["t"])
            np.testing.assert_array_equal(m.transitive_closure().blocks, arr["out_blocks"],
                                          err_msg=meta["name"])
            assert m.reflexive_transitive_closure().to_lists() == arr["refl"].tolist()


def test_samples(samples):
    a = AntidistMatrix.from_lists(samples["a4"]["rows"], 8)
    b = AntidistMatrix.from_lists(samples["b4"]["rows"], 8)
    assert (a * b).to_lists() == samples["a4_times_b4"]
    for name in ("chain3", "cycle3"):
        s = samples[name]
        assert BoolMatrix.from_lists(s["bool_adjacency"]).transitive_closure().to_lists() == s["bool_closure"]
        assert BoolMatrix.from_lists(s["bool_adjacency"]).reflexive_transitive_closure().to_lists() == \
            s["bool_reflexive"]
        assert AntidistMatrix.from_lists(s["antidist_adjacency"], 8).transitive_closure().to_lists() == \
            s["antidist_closure"]
        assert DistMatrix.from_lists(s["dist_adjacency"], 8).transitive_closure().to_lists() == \
            s["dist_closure"]


def test_reference_golden_values():
    """tests/test_antidist.py:130-206 golden values, through the GPU classes."""
    a = AntidistMatrix.zeros(3, 3, 8)
    a.set(0, 1, 252)
    b = AntidistMatrix.zeros(3, 3, 8)
    b.set(1, 2, 251)
    assert (a * b).get(0, 2) == 248
    m = AntidistMatrix.from_edges(3, [(0, 1, 3), (1, 2, 4)], 8)
    assert m.transitive_closure().get(0, 2) == 248
    for width, want in ((8, 0), (16, 65535 - 300)):
        chain = AntidistMatrix.from_edges(31, [(i, i + 1, 10) for i in range(30)], width)
        assert chain.transitive_closure().get(0, 30) == want
    d = DistMatrix.from_edges(2, [(0, 1, 3), (1, 0, 4)], 8).transitive_closure()
    assert d.get(0, 0) == 7 and d.get(1, 1) == 7


# -- BASELINE.json configurations: sha256 of the reference output ---------------

def _gpu_output(cfg, n):
    inputs = workloads.make_inputs(cfg, n)
    if cfg.op == "bool_mul":
        out = (BoolMatrix.from_numpy(inputs[0]) * BoolMatrix.from_numpy(inputs[1])).blocks
    elif cfg.op == "bool_closure":
        out = BoolMatrix.from_numpy(inputs[0]).transitive_closure().blocks
    elif cfg.op == "mul":
        out = (lane("anti", inputs[0], n, cfg.width) * lane("anti", inputs[1], n, cfg.width)).data
    else:
        out = lane("anti", inputs[0], n, cfg.width).transitive_closure().data
    return out


@pytest.mark.parametrize("name", list(workloads.CONFIGS))
def test_config_matches_reference_digest(config_digests, name):
    cfg = workloads.CONFIGS[name]
    for d in config_digests:
        # full-size oracle pins (band digests) have their own test
        if d["config"] == name and "band_sha256" not in d:
            assert sha(_gpu_output(cfg, d["n"])) == d["output_sha256"], (name, d["n"])


# -- full-size, size-independent properties -------------------------------------

def test_fw_full_size_bellman_fixpoint():
    """C4 at n = 8192: T+ = T (+) T+ (x) T, and closing T+ again changes nothing."""
    cfg = workloads.CONFIGS["c4_fw_u16"]
    (t,) = workloads.make_inputs(cfg)
    a = lane("anti", t, cfg.n, 16)
    c = a.transitive_closure()
    assert (a | (c * a)) == c
    assert c.transitive_closure() == c


def test_widths_agree_on_small_weights():
    """Same graph at u8 / u16 / u32 gives the same distances while they fit (test_antidist.py:235-246)."""
    rng = np.random.default_rng(7)
    n = 300
    edges = [(int(u), int(v), int(w)) for u, v, w in
             zip(rng.integers(0, n, 3000), rng.integers(0, n, 3000), rng.integers(1, 4, 3000))]
    d = {w: DistMatrix.from_edges(n, edges, w).transitive_closure().to_numpy()[:, :n].astype(np.int64)
         for w in (8, 16, 32)}
    assert (d[16] < 255).all()
    np.testing.assert_array_equal(d[8], d[16])
    np.testing.assert_array_equal(d[16], d[32])


def test_anti_and_dist_are_complement_duals():
    """~(A * B) == (~A) * (~B) and ~closure(A) == closure(~A) (test_antidist.py:277-311)."""
    cfg = workloads.CONFIGS["c3_mul_u16"]
    a_np, b_np = workloads.make_inputs(cfg, 1000)
    a, b = lane("anti", a_np, 1000, 16), lane("anti", b_np, 1000, 16)
    assert ~(a * b) == (~a) * (~b)
    assert ~a.transitive_closure() == (~a).transitive_closure()


def test_ragged_and_edge_shapes(oracle_lib):
    rng = np.random.default_rng(11)
    for width in (8, 16, 32):
        for rows, inner, cols in [(1, 1, 1), (1000, 777, 1001), (129, 3, 257), (5, 300, 2)]:
            for kind in ("anti", "dist"):
                lim = (1 << width) - 1
                a_np = rng.integers(0, lim + 1, size=(rows, inner), dtype=np.uint64)
                b_np = rng.integers(0, lim + 1, size=(inner, cols), dtype=np.uint64)
                a = CLS[kind].from_lists(a_np.tolist(), width) if rows * inner < 5000 else \
                    _fast_lane(kind, a_np, width)
                b = CLS[kind].from_lists(b_np.tolist(), width) if inner * cols < 5000 else \
                    _fast_lane(kind, b_np, width)
                got = (a * b).data
                want = oracle_lib.semiring_mul(a.data, b.data, inner, width, kind)
                np.testing.assert_array_equal(got, want, err_msg=f"{width} {rows}x{inner}x{cols} {kind}")


def _fast_lane(kind, vals, width):
    rows, cols = vals.shape
    lanes = {8: 16, 16: 8, 32: 4}[width]
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32}[width]
    pad = 0 if kind == "anti" else (1 << width) - 1
    host = np.full((rows, -(-cols // lanes) * lanes), pad, dtype=dt)
    host[:, :cols] = vals.astype(dt)
    return CLS[kind](rows, cols, width, host)


def test_fw_odd_sizes(oracle_lib):
    """Closures whose size is not a multiple of the 128-vertex pivot block."""
    rng = np.random.default_rng(5)
    for n in (129, 200, 383, 640):
        for width in (8, 16, 32):
            lim = (1 << width) - 1
            vals = np.where(rng.random((n, n)) < 0.03, lim - rng.integers(1, 30, (n, n)), 0)
            m = _fast_lane("anti", vals, width)
            np.testing.assert_array_equal(m.transitive_closure().data,
                                          oracle_lib.semiring_close(m.data, width, "anti"),
                                          err_msg=f"n={n} w={width}")
            d = ~m
            np.testing.assert_array_equal(d.transitive_closure().data,
                                          oracle_lib.semiring_close(d.data, width, "dist"))


def test_bool_odd_sizes(oracle_lib):
    rng = np.random.default_rng(6)
    for n in (257, 300, 700, 1500):
        bits = (rng.random((n, n)) < 1.5 / n).astype(np.uint8)
        m = BoolMatrix.from_numpy(bits)
        want = oracle_lib.bool_close(oracle_lib.pack_bits(bits))
        np.testing.assert_array_equal(m.transitive_closure().blocks, want, err_msg=f"n={n}")
        b2 = (rng.random((n, 333)) < 0.01).astype(np.uint8)
        want = oracle_lib.bool_mul(oracle_lib.pack_bits(bits), oracle_lib.pack_bits(b2), n)
        np.testing.assert_array_equal((m * BoolMatrix.from_numpy(b2)).blocks, want)


def test_errors_match_reference():
    a = AntidistMatrix.zeros(2, 3, 8)
    with pytest.raises(ValueError, match="inner dimensions disagree"):
        a * AntidistMatrix.zeros(2, 3, 8)
    with pytest.raises(ValueError, match="width mismatch"):
        a * AntidistMatrix.zeros(3, 2, 16)
    with pytest.raises(TypeError):
        a * DistMatrix.unreachable(3, 2, 8)
    with pytest.raises(ValueError, match="closure needs a square matrix"):
        a.transitive_closure()
    with pytest.raises(ValueError, match="closure needs a square matrix"):
        BoolMatrix.zeros(2, 3).transitive_closure()
    with pytest.raises(ValueError, match="inner dimensions disagree"):
        BoolMatrix.zeros(2, 3) * BoolMatrix.zeros(2, 3)
    with pytest.raises(TypeError):
        BoolMatrix.zeros(2, 2) * a
    with pytest.raises(ValueError):
        AntidistMatrix.zeros(0, 2, 8)


def test_c_abi_rejects_misaligned():
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    t = torch.zeros(64, 64, dtype=torch.uint16, device="cuda")
    rc = lib.smx_semiring_gemm_u16(t.data_ptr() + 2, t.data_ptr(), t.data_ptr(), 8, 8, 8, 64, 64,
                                   64, 0, 0, None)
    assert rc == -2
    rc = lib.smx_semiring_gemm_u16(t.data_ptr(), t.data_ptr(), t.data_ptr(), 8, 8, 8, 63, 64, 64, 0,
                                   0, None)
    assert rc == -2
    assert lib.smx_fw_u16(t.data_ptr(), 300, 64, 0, None, 0, None) == -1


# -- tensor-core Boolean engine, both output layouts -----------------------------

def test_bool_tc_engines_match_reference(small_cases, config_digests):
    for meta, arr in small_cases:
        if meta["op"] == "bool_closure":
            got = engines.bool_closure_tc(BoolMatrix.from_numpy(arr["t"]))
            np.testing.assert_array_equal(got.blocks, arr["out_blocks"], err_msg=meta["name"])
            got = engines.bool_closure_bits(BoolMatrix.from_numpy(arr["t"]))
            np.testing.assert_array_equal(got.blocks, arr["out_blocks"], err_msg=meta["name"])
    for name, fn in (("c2_bool_warshall", engines.bool_closure_tc),
                     ("c2_bool_warshall", engines.bool_closure_bits)):
        cfg = workloads.CONFIGS[name]
        d = next(x for x in config_digests if x["config"] == name)
        (t,) = workloads.make_inputs(cfg, d["n"])
        assert sha(fn(BoolMatrix.from_numpy(t)).blocks) == d["output_sha256"]
    cfg = workloads.CONFIGS["c1_bool_mul"]
    d = next(x for x in config_digests if x["config"] == "c1_bool_mul")
    a, b = workloads.make_inputs(cfg)
    for fn in (engines.bool_mul_tc, engines.bool_mul_bits):
        assert sha(fn(BoolMatrix.from_numpy(a), BoolMatrix.from_numpy(b)).blocks) == d["output_sha256"]


def test_bool_tc_bytes_output_and_accumulate(oracle_lib):
    """smx_bool_gemm_i8 byte epilogue, OR-accumulate, ragged M/N/K, all tile widths."""
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    rng = np.random.default_rng(3)
    for m, n, k in [(1, 1, 1), (128, 64, 128), (300, 1000, 77), (1024, 520, 2000), (4096, 4096, 256)]:
        a = (rng.random((m, k)) < 0.02).astype(np.uint8)
        b = (rng.random((k, n)) < 0.02).astype(np.uint8)
        c0 = (rng.random((m, n)) < 0.1).astype(np.uint8)
        want = ((a.astype(np.int64) @ b.astype(np.int64)) > 0).astype(np.uint8)
        r16 = lambda x: -(-x // 16) * 16  # noqa: E731
        ta = torch.zeros((m, r16(k)), dtype=torch.uint8, device="cuda")
        ta[:, :k] = torch.from_numpy(a)
        tbt = torch.zeros((n, r16(k)), dtype=torch.uint8, device="cuda")
        tbt[:, :k] = torch.from_numpy(np.ascontiguousarray(b.T))
        for acc in (0, 1):
            tc = torch.zeros((m, r16(n)), dtype=torch.uint8, device="cuda")
            tc[:, :n] = torch.from_numpy(c0)
            rc = lib.smx_bool_gemm_i8(ta.data_ptr(), tbt.data_ptr(), tc.data_ptr(), None, m, n, k,
                                      ta.shape[1], tbt.shape[1], tc.shape[1], acc,
                                      _native.stream_ptr())
            assert rc == 0
            exp = (want | c0) if acc else want
            np.testing.assert_array_equal(tc[:, :n].cpu().numpy(), exp, err_msg=f"{m}x{n}x{k} acc={acc}")
            assert (tc[:, n:].cpu().numpy() == 0).all()


# -- row-panel-sharded closure: the GPU ops, ranks emulated in lockstep ----------

@pytest.mark.parametrize("world,n,block", [(1, 1000, None), (2, 1000, None), (3, 1280, None), (8, 2048, None),
                                           (2, 2100, 512), (3, 1536, 512)])
def test_sharded_fw_gpu_ops_lockstep(world, n, block, oracle_lib):
    """ShardedFW with CudaFwOps for `world` ranks on one GPU, run round by round
    in one process (the broadcast becomes a device copy; no rank ever waits on
    another, so this is safe on a single GPU) -- bit-identical to the oracle."""
    from paper_1705_08743_b200 import sharded
    cfg = workloads.CONFIGS["c5_fw_u16"]
    (full,) = workloads.make_inputs(cfg, n)
    ranks = []
    for r in range(world):
        ops = sharded.CudaFwOps(16, anti=True, block=block)
        fw = sharded.ShardedFW(n=n, rank=r, world=world, ops=ops)
        ranks.append((fw, torch.from_numpy(full[fw.row0:fw.row1].copy()).cuda()))
    block = ranks[0][0].block
    for k0 in range(0, n, block):
        owner = ranks[0][0].owner(k0)
        begun = [fw.begin_round(local, k0) for fw, local in ranks]
        src = begun[owner][0]
        for r, (panel, _) in enumerate(begun):
            if r != owner:
                panel.copy_(src)
        for (fw, local), (panel, skip) in zip(ranks, begun):
            fw.end_round(local, panel, k0, skip)
    got = torch.cat([local for _, local in ranks]).cpu().numpy()
    np.testing.assert_array_equal(got, oracle_lib.semiring_close(full, 16, "anti"))


# -- the verified 1-instruction k-tiles ------------------------------------------

@pytest.mark.parametrize("width", [16, 32])
def test_bounded_fastpath_is_exact(width, oracle_lib):
    """Tiles whose lanes are all < 2^(w-1) take the 1-instruction update; tiles
    with larger values or unreachable entries take the general one.  Both must
    equal the oracle, and forcing the general form must not change a bit."""
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    rng = np.random.default_rng(21)
    half = 1 << (width - 1)
    n = 700
    cases = {
        "all_bounded": rng.integers(0, half, size=(n, n), dtype=np.uint64),
        "edge_of_bound": rng.integers(half - 3, half, size=(n, n), dtype=np.uint64),
        "mixed": np.where(rng.random((n, n)) < 0.5, rng.integers(0, half, size=(n, n)),
                          rng.integers(half, 1 << width, size=(n, n))).astype(np.uint64),
        "sparse_unreachable": np.where(rng.random((n, n)) < 0.999, rng.integers(0, 50, size=(n, n)),
                                       (1 << width) - 1).astype(np.uint64),
    }
    for name, vals in cases.items():
        a = _fast_lane("dist", vals, width)
        b = _fast_lane("dist", vals[::-1].copy(), width)
        want = oracle_lib.semiring_mul(a.data, b.data, n, width, "dist")
        np.testing.assert_array_equal((a * b).data, want, err_msg=name)
        old = lib.smx_set_bounded_fastpath(0)
        try:
            np.testing.assert_array_equal((a * b).data, want, err_msg=name + " (general)")
        finally:
            lib.smx_set_bounded_fastpath(old)
        anti = ~a
        np.testing.assert_array_equal((anti * ~b).data,
                                      oracle_lib.semiring_mul(anti.data, (~b).data, n, width, "anti"))


def test_fw_fastpath_on_off_identical():
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    cfg = workloads.CONFIGS["c4_fw_u16"]
    (t,) = workloads.make_inputs(cfg, 2048)
    fast = lane("anti", t, 2048, 16).transitive_closure().data
    old = lib.smx_set_bounded_fastpath(0)
    try:
        slow = lane("anti", t, 2048, 16).transitive_closure().data
    finally:
        lib.smx_set_bounded_fastpath(old)
    np.testing.assert_array_equal(fast, slow)


@pytest.mark.parametrize("n", [129, 300, 1000, 1100, 2048])
def test_fw_lookahead_and_serial_schedules_agree(n, oracle_lib):
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    cfg = workloads.CONFIGS["c5_fw_u16"]
    (t,) = workloads.make_inputs(cfg, n)
    want = oracle_lib.semiring_close(t, 16, "anti")
    for la, lite, blk, split in ((1, 0, 0, 1), (0, 0, 0, 1), (1, 1, 0, 1), (1, 0, 256, 1), (1, 1, 256, 1),
                                 (0, 0, 256, 1), (1, 0, 128, 1), (1, 0, 512, 1), (0, 0, 512, 1), (1, 1, 512, 1),
                                 (1, 0, 0, 0), (1, 0, 256, 0), (1, 0, 512, 0), (1, 0, 0, 2), (1, 0, 256, 2),
                                 (1, 1, 512, 2), (1, 0, 0, 10), (1, 0, 512, 12), (1, 0, 0, 101), (1, 0, 512, 101)):
        # split >= 10: the row panel on the register-staged tiles (smx_set_fw_packed_panel(0)); else
        # always on the packed kernel (2); split >= 100: one packed row-panel buffer
        olds = (lib.smx_set_fw_lookahead(la), lib.smx_set_fw_side_lite(lite), lib.smx_set_fw_block(blk),
                lib.smx_set_fw_split_3a(split % 10), lib.smx_set_fw_packed_panel(2 if split % 100 < 10 else 0),
                lib.smx_set_fw_panel_buffers(1 if split >= 100 else 2))
        try:
            for width_kind in ("anti", "dist"):
                m = lane("anti", t, n, 16)
                if width_kind == "dist":
                    m = ~m
                    np.testing.assert_array_equal((~m.transitive_closure()).data, want,
                                                  err_msg=f"la={la} lite={lite} blk={blk} split={split}")
                else:
                    np.testing.assert_array_equal(m.transitive_closure().data, want,
                                                  err_msg=f"la={la} lite={lite} blk={blk} split={split}")
        finally:
            lib.smx_set_fw_lookahead(olds[0])
            lib.smx_set_fw_side_lite(olds[1])
            lib.smx_set_fw_block(olds[2])
            lib.smx_set_fw_split_3a(olds[3])
            lib.smx_set_fw_packed_panel(olds[4])
            lib.smx_set_fw_panel_buffers(olds[5])


@pytest.mark.parametrize("n", [640, 2048])
def test_sharded_fw_gpu_lookahead_single_rank(n, oracle_lib):
    """The pipelined ShardedFW schedule (side stream, double-buffered panel) on
    the GPU ops at world = 1 -- bit-identical to the oracle."""
    from paper_1705_08743_b200 import sharded
    (full,) = workloads.make_inputs(workloads.CONFIGS["c5_fw_u16"], n)
    local = torch.from_numpy(full.copy()).cuda()
    sharded.ShardedFW(n=n, rank=0, world=1, ops=sharded.CudaFwOps(16, anti=True)).run(local)
    np.testing.assert_array_equal(local.cpu().numpy(), oracle_lib.semiring_close(full, 16, "anti"))


# -- entrywise algebra and the Boolean bridge ---------------

def test_entrywise_match_reference():
    import json
    from conftest import GOLDEN
    manifest = json.loads((GOLDEN / "entrywise.json").read_text())
    arrs = np.load(GOLDEN / "entrywise.npz")
    for meta in manifest:
        g = lambda k: arrs[f"{meta['name']}__{k}"]  # noqa: E731
        if meta["kind"] == "bool":
            a, b = BoolMatrix.from_numpy(g("a")), BoolMatrix.from_numpy(g("b"))
            for op, got in (("or", a | b), ("and", a & b), ("xor", a ^ b), ("inv", ~a)):
                np.testing.assert_array_equal(got.blocks, g(op), err_msg=f"{meta['name']} {op}")
            for w in (8, 16):
                np.testing.assert_array_equal(AntidistMatrix.from_boolmat(a, w).data, g(f"fromboolmat{w}"))
        else:
            a = lane(meta["kind"], g("a"), meta["cols"], meta["width"])
            b = lane(meta["kind"], g("b"), meta["cols"], meta["width"])
            for op, got in (("or", a | b), ("and", a & b), ("xor", a ^ b), ("inv", ~a)):
                np.testing.assert_array_equal(got.data, g(op), err_msg=f"{meta['name']} {op}")
            assert isinstance(~a, DistMatrix if meta["kind"] == "anti" else AntidistMatrix)
            if meta["kind"] == "anti":
                assert a.to_boolmat().to_lists() == g("toboolmat").tolist()


# -- device construction from edge lists --------------------

@pytest.mark.parametrize("width", [8, 16, 32])
def test_from_edges_device(width):
    rng = np.random.default_rng(width)
    n, m = 300, 20000
    lim = (1 << width) - 1
    edges = np.stack([rng.integers(0, n, m), rng.integers(0, n, m),
                      rng.integers(0, min(lim, 5000) + 1, m)], axis=1)
    edges[:50, :2] = edges[50:100, :2]                       # force parallel edges
    lanes = {8: 16, 16: 8, 32: 4}[width]
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32}[width]
    want_a = np.zeros((n, -(-n // lanes) * lanes), dtype=np.int64)
    np.maximum.at(want_a, (edges[:, 0], edges[:, 1]), lim - edges[:, 2])
    want_d = np.full((n, -(-n // lanes) * lanes), lim, dtype=np.int64)
    np.minimum.at(want_d, (edges[:, 0], edges[:, 1]), edges[:, 2])
    got_a = AntidistMatrix.from_edges(n, edges, width)
    got_d = DistMatrix.from_edges(n, [tuple(e) for e in edges.tolist()], width)
    np.testing.assert_array_equal(got_a.data, want_a.astype(dt))
    np.testing.assert_array_equal(got_d.data, want_d.astype(dt))
    assert AntidistMatrix.from_edges(4, [], width) == AntidistMatrix.zeros(4, 4, width)


def test_from_edges_errors_match_reference():
    with pytest.raises(ValueError, match="source vertex 5 out of range"):
        AntidistMatrix.from_edges(2, [(0, 1, 1), (5, 0, 1), (0, 9, 1)], 8)
    with pytest.raises(ValueError, match="target vertex 9 out of range"):
        AntidistMatrix.from_edges(2, [(0, 1, 1), (0, 9, 1), (5, 0, 1)], 8)
    with pytest.raises(ValueError, match="weight 300 outside"):
        DistMatrix.from_edges(2, [(0, 1, 300)], 8)
    m = AntidistMatrix.from_edges(2, [(0, 1, 3), (0, 1, 5)], 8)
    assert m.get(0, 1) == 252
    assert AntidistMatrix.from_edges(1, [(0, 0, 0)], 8).get(0, 0) == 255


# -- an independent closure algorithm on the device ---------

def test_closure_by_squaring_matches_fw_and_warshall():
    """A (x) (I (+) A)^(2^j) by repeated GPU squaring (oracle.py:49-74) equals the
    blocked FW / Warshall closure at sizes beyond the CPU oracle's reach."""
    cfg = workloads.CONFIGS["c4_fw_u16"]
    (t,) = workloads.make_inputs(cfg, 4096)
    a = lane("anti", t, 4096, 16)
    assert engines.closure_by_squaring(a) == a.transitive_closure()
    d = ~a
    assert engines.closure_by_squaring(d) == d.transitive_closure()
    (b,) = workloads.make_inputs(workloads.CONFIGS["c2_bool_warshall"], 2048)
    bm = BoolMatrix.from_numpy(b)
    assert engines.closure_by_squaring(bm) == bm.transitive_closure()


@pytest.mark.parametrize("block", [512, 256])
def test_fw_n16384_matches_squaring(block):
    """n >= 16384 takes the 512-vertex pivot block by default (256 forced here
    too); cross-check the closure with the independent repeated-squaring
    algorithm and the Bellman fixpoint."""
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    cfg = workloads.CONFIGS["c5_fw_u16"]
    (t,) = workloads.make_inputs(cfg, 16384)
    a = lane("anti", t, 16384, 16)
    old = lib.smx_set_fw_block(block)
    try:
        assert lib.smx_fw_block_for(16384, 2) == block
        c = a.transitive_closure()
    finally:
        lib.smx_set_fw_block(old)
    assert (a | (c * a)) == c
    assert engines.closure_by_squaring(a) == c


@pytest.mark.parametrize("width", [16, 32])
def test_sparse_bounded_certificates_are_exact(width, oracle_lib):
    """Large products take the certified shifted 1-instruction form when every
    A row / B column / C tile lane is S or < 2^(w-2); values at the edge of the
    certificate (2^(w-2) - 1) and just past it (2^(w-2)) must both be exact."""
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    rng = np.random.default_rng(33)
    q = 1 << (width - 2)
    S = (1 << width) - 1
    n = 1100                                             # M*N >= 2^20: certified path
    edge = np.where(rng.random((n, n)) < 0.5, S, rng.integers(q - 4, q, size=(n, n))).astype(np.uint64)
    over = edge.copy()
    over[rng.integers(0, n, 50), rng.integers(0, n, 50)] = q   # breaks the certificate
    sparse = np.where(rng.random((n, n)) < 0.9, S, rng.integers(0, 1000, size=(n, n))).astype(np.uint64)
    for name, vals in (("edge", edge), ("over", over), ("sparse", sparse)):
        a = _fast_lane("dist", vals, width)
        b = _fast_lane("dist", vals.T.copy(), width)
        want = oracle_lib.semiring_mul(a.data, b.data, n, width, "dist")
        np.testing.assert_array_equal((a * b).data, want, err_msg=name)
        old = lib.smx_set_bounded_fastpath(0)
        try:
            np.testing.assert_array_equal((a * b).data, want, err_msg=name + " (general)")
        finally:
            lib.smx_set_bounded_fastpath(old)
        aa, ba = ~a, ~b
        np.testing.assert_array_equal((aa * ba).data,
                                      oracle_lib.semiring_mul(aa.data, ba.data, n, width, "anti"),
                                      err_msg=name + " anti")


# -- SRMAT1 / text I/O to and from HBM ----------------------

def test_matio_matches_reference_bytes(tmp_path):
    import json
    from conftest import GOLDEN
    from paper_1705_08743_b200 import matio
    for case in json.loads((GOLDEN / "matio.json").read_text()):
        if case["kind"] == "bool":
            m = BoolMatrix.from_lists(case["bits"])
        else:
            m = CLS[case["kind"]].from_lists(case["rows"], case["width"])
        assert matio.to_binary(m).hex() == case["binary"]
        assert matio.format_text(m) == case["text"]
        back = matio.from_binary(bytes.fromhex(case["binary"]))
        assert type(back) is type(m) and back == m
        assert matio.parse_text(case["text"]) == m
        p = tmp_path / "m.bin"
        matio.save(m, p, binary=True)
        assert matio.load(p) == m
        matio.save(m, p)
        assert matio.load(p) == m


def test_matio_errors_match_reference():
    from paper_1705_08743_b200 import matio
    with pytest.raises(matio.MatrixFormatError, match="truncated header"):
        matio.from_binary(b"SRMAT1")
    with pytest.raises(matio.MatrixFormatError, match="bad magic"):
        matio.from_binary(b"XXXXXX" + bytes(10))
    bad = bytearray(matio.to_binary(BoolMatrix.from_lists([[1] * 65])))
    bad[-1] |= 0x80                                   # a padding bit of the final block
    with pytest.raises(matio.MatrixFormatError, match="nonzero padding bits"):
        matio.from_binary(bytes(bad))
    with pytest.raises(matio.MatrixFormatError, match="expected 3 values"):
        matio.parse_text("antidist 8 1 3\n1 2\n")


# -- graph replay (smx_set_graphs) ---------------------------------------------

def test_graph_replay_tracks_buffer_contents(oracle_lib):
    """Replayed graphs read the buffers' current contents: closing the same
    buffer with new data each call (graph hit after the first) matches the
    oracle, for FW u16, bit Warshall and the tensor-core product; the same
    calls inside a user's torch.cuda.graph capture run into that capture."""
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    n = 700
    ins = [workloads.make_inputs(workloads.CONFIGS[c], n)[0] for c in ("c5_fw_u16", "c4_fw_u16")]
    m = lane("anti", ins[0], n, 16)
    buf = m._data
    before = lib.smx_launch_count()
    for t in (ins[0], ins[1], ins[0], ins[1]):
        buf.copy_(lane("anti", t, n, 16)._data)
        engines.lane_close_(buf, n, 16, True)
        got = lane("anti", t, n, 16)
        got._data.copy_(buf)
        np.testing.assert_array_equal(got.data, oracle_lib.semiring_close(t, 16, "anti"))
    assert lib.smx_launch_count() - before >= 4 * 10   # replays still count their kernels

    # a user capture around the call: the library launches into it eagerly
    g = torch.cuda.CUDAGraph()
    buf.copy_(lane("anti", ins[0], n, 16)._data)
    with torch.cuda.graph(g):
        engines.lane_close_(buf, n, 16, True)
    buf.copy_(lane("anti", ins[1], n, 16)._data)
    g.replay()
    torch.cuda.synchronize()
    got = lane("anti", ins[1], n, 16)
    got._data.copy_(buf)
    np.testing.assert_array_equal(got.data, oracle_lib.semiring_close(ins[1], 16, "anti"))

    # bit Warshall on one buffer, two graphs-hit calls with different contents
    rng = np.random.default_rng(5)
    nb = 1100
    mats = [rng.random((nb, nb)) < p for p in (2 / nb, 1 / nb)]
    bm = BoolMatrix.from_numpy(mats[0])
    words = bm._words.clone()
    nbytes = lib.smx_bool_warshall_workspace_bytes(nb, bm.stride_words)
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    for mat in (mats[0], mats[1], mats[0]):
        words.copy_(BoolMatrix.from_numpy(mat)._words)
        _native.check(lib.smx_bool_warshall_bits(words.data_ptr(), nb, bm.stride_words, ws.data_ptr(), nbytes,
                                                 _native.stream_ptr()), "warshall")
        from oracle import pack_bits
        got = BoolMatrix(nb, nb, words.clone()).blocks
        np.testing.assert_array_equal(got, oracle_lib.bool_close(pack_bits(mat)))

    # tensor-core product: same operand buffers, new contents
    a = BoolMatrix.from_numpy(mats[0][:, :900])
    b = BoolMatrix.from_numpy(mats[1][:900, :])
    first = engines.bool_mul_tc(a, b).to_numpy()
    a._words.copy_(BoolMatrix.from_numpy(mats[1][:, :900])._words)
    second = engines.bool_mul_tc(a, b).to_numpy()
    ref2 = (mats[1][:, :900].astype(np.int32) @ mats[1][:900, :].astype(np.int32)) > 0
    ref1 = (mats[0][:, :900].astype(np.int32) @ mats[1][:900, :].astype(np.int32)) > 0
    np.testing.assert_array_equal(first, ref1)
    np.testing.assert_array_equal(second, ref2)


def test_graphs_off_matches_graphs_on():
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    (t,) = workloads.make_inputs(workloads.CONFIGS["c4_fw_u16"], 1500)
    outs = []
    for on in (1, 0):
        old = lib.smx_set_graphs(on)
        try:
            outs.append(lane("dist", t, 1500, 16).transitive_closure().data)
        finally:
            lib.smx_set_graphs(old)
    np.testing.assert_array_equal(outs[0], outs[1])


@pytest.mark.parametrize("kind", ["anti", "dist"])
def test_packed_skip_gemm_matches_register_kernel_and_oracle(kind, oracle_lib):
    """smx_semiring_gemm_skip u16 at a size that takes the packed phase-3
    kernel (ragged M/N, a skipped row range): equal to the register-staged
    kernel (smx_set_fw_packed(0)) everywhere and to the oracle on 300 rows."""
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    rng = np.random.default_rng(11)
    M, N, K = 4200, 4100, 256
    S = 0xFFFF
    def mat(r, c, dens):
        v = rng.integers(0, 30000, (r, c), dtype=np.uint32)
        v[rng.random((r, c)) > dens] = S if kind == "dist" else 0
        if kind == "anti":
            v[rng.random((r, c)) < dens / 4] = S - rng.integers(0, 1000)  # near-zero distances
        return v.astype(np.uint16)
    a, b, c = mat(M, K, 0.5), mat(K, N, 0.5), mat(M, N, 0.3)
    ldc = 4104
    cpad = np.zeros((M, ldc), dtype=np.uint16); cpad[:, :N] = c
    bpad = np.zeros((K, ldc), dtype=np.uint16); bpad[:, :N] = b
    kid = 0 if kind == "anti" else 1
    outs = []
    for packed in (1, 0):
        old = lib.smx_set_fw_packed(packed)
        try:
            ta = torch.from_numpy(a.view(np.int16)).cuda()
            tb = torch.from_numpy(bpad.view(np.int16)).cuda()
            tc = torch.from_numpy(cpad.view(np.int16)).cuda()
            _native.check(lib.smx_semiring_gemm_skip(ta.data_ptr(), tb.data_ptr(), tc.data_ptr(), M, N, K, K,
                                                     ldc, ldc, 2, kid, 1024, 256, _native.stream_ptr()), "skip")
            torch.cuda.synchronize()
            outs.append(tc.cpu().numpy().view(np.uint16)[:, :N].copy())
        finally:
            lib.smx_set_fw_packed(old)
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[0][1024:1280], c[1024:1280])   # skipped rows untouched
    prod = oracle_lib.semiring_mul(a[:300], b, K, 16, kind)
    want = np.maximum(c[:300], prod) if kind == "anti" else np.minimum(c[:300], prod)
    np.testing.assert_array_equal(outs[0][:300], want)


@pytest.mark.parametrize("case", ["certified", "one_large", "full_range", "u8"])
@pytest.mark.parametrize("kind", ["anti", "dist"])
def test_public_u16_product_packed_path(case, kind, oracle_lib):
    """smx_semiring_gemm_u16 at sizes that take the packed kernel: the
    product-wide shifted encoding (certified), a single large lane that voids
    the certificate, and full-range lanes (per-tile flags) -- each equal to
    the register-staged kernel and to the oracle on 256 rows.  K = 700 spans
    a ragged last k-tile."""
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    rng = np.random.default_rng({"certified": 1, "one_large": 2, "full_range": 3, "u8": 4}[case])
    M, N, K = 2100, 2056, 700
    w = 8 if case == "u8" else 16
    S = (1 << w) - 1
    hi = {"full_range": 60000, "u8": 250}.get(case, 1000)
    def mat(r, c):
        v = rng.integers(0, hi, (r, c), dtype=np.uint32)
        v[rng.random((r, c)) > 0.2] = S
        return v
    a, b = mat(M, K), mat(K, N)
    if case == "one_large":
        a[1234, 77] = 40000
    if kind == "anti":
        a, b = S - a, S - b
    dt, st = (np.uint8, np.int8) if w == 8 else (np.uint16, np.int16)
    a, b = a.astype(dt), b.astype(dt)
    lda, ldn = 704, 2064
    apad = np.zeros((M, lda), dt); apad[:, :K] = a
    bpad = np.zeros((K, ldn), dt); bpad[:, :N] = b
    kid = 0 if kind == "anti" else 1
    outs = []
    for packed in (1, 0):
        old = lib.smx_set_fw_packed(packed)
        try:
            ta = torch.from_numpy(apad.view(st)).cuda()
            tb = torch.from_numpy(bpad.view(st)).cuda()
            tc = torch.empty((M, ldn), dtype=ta.dtype, device="cuda")
            fn = getattr(lib, f"smx_semiring_gemm_u{w}")
            _native.check(fn(ta.data_ptr(), tb.data_ptr(), tc.data_ptr(), M, N, K, lda, ldn, ldn, kid, 0,
                             _native.stream_ptr()), "product")
            torch.cuda.synchronize()
            outs.append(tc.cpu().numpy().view(dt)[:, :N].copy())
        finally:
            lib.smx_set_fw_packed(old)
    np.testing.assert_array_equal(outs[0], outs[1])
    rows = np.r_[0:128, 1200:1328]
    want = oracle_lib.semiring_mul(apad[rows], b, K, w, kind)
    np.testing.assert_array_equal(outs[0][rows], want)

    # accumulate = 1 into a random C: C (+)= A (x) B, folded after the K loop
    c0 = mat(M, N).astype(dt) if kind == "dist" else (S - mat(M, N)).astype(dt)
    cpad = np.zeros((M, ldn), dt); cpad[:, :N] = c0
    tc = torch.from_numpy(cpad.view(st)).cuda()
    ta = torch.from_numpy(apad.view(st)).cuda()   # kept alive across the async call
    tb = torch.from_numpy(bpad.view(st)).cuda()
    _native.check(getattr(lib, f"smx_semiring_gemm_u{w}")(
        ta.data_ptr(), tb.data_ptr(), tc.data_ptr(), M, N, K, lda, ldn, ldn, kid, 1, _native.stream_ptr()),
        "accumulate")
    torch.cuda.synchronize()
    got = tc.cpu().numpy().view(dt)[:, :N]
    comb = np.maximum if kind == "anti" else np.minimum
    np.testing.assert_array_equal(got, comb(c0, outs[0]))


@pytest.mark.parametrize("n", [1100, 2304])
def test_fw_u8_packed_and_register_paths_agree(n, oracle_lib):
    """u8 closures through the packed phase 3 (default) and the register-staged
    one (smx_set_fw_packed(0)), both schedules: equal to the oracle."""
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    rng = np.random.default_rng(n)
    cpad = -(-n // 16) * 16
    t = np.zeros((n, cpad), np.uint8)
    t[:, :n] = np.where(rng.random((n, n)) < 0.05, 255 - rng.integers(1, 60, (n, n)), 0)
    np.fill_diagonal(t, 255)
    want = oracle_lib.semiring_close(t, 8, "anti")
    for packed, la in ((1, 1), (1, 0), (0, 1)):
        olds = (lib.smx_set_fw_packed(packed), lib.smx_set_fw_lookahead(la))
        try:
            np.testing.assert_array_equal(lane("anti", t, n, 8).transitive_closure().data, want,
                                          err_msg=f"packed={packed} la={la}")
        finally:
            lib.smx_set_fw_packed(olds[0])
            lib.smx_set_fw_lookahead(olds[1])


def test_bool_warshall_512_blocks_ragged(oracle_lib):
    """n >= 8192 takes 512-vertex Warshall blocks (16-word pivot tiles, 512
    threads); a ragged n and a denser graph exercise partial tiles and the
    table pivot's dense path.  Bit-exact against the C oracle."""
    from oracle import pack_bits
    rng = np.random.default_rng(77)
    n = 8300
    a = rng.random((n, n), dtype=np.float32) < 3.0 / n
    got = BoolMatrix.from_numpy(a).transitive_closure().blocks
    np.testing.assert_array_equal(got, oracle_lib.bool_close(pack_bits(a)))


@pytest.mark.parametrize("w", [8, 16])
def test_pivot_kernels_blocked_and_register_agree(w, oracle_lib):
    """smx_fw_pivot on tiles of 1..512 vertices: the blocked 128 kernel and the
    one-barrier-per-vertex register kernel (as leaves of the in-place 2 x 2
    recursion above 128) both equal the oracle closure, anti and dist, dense
    and sparse, inside a larger padded matrix (only the b x b tile changes)."""
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    S = (1 << w) - 1
    dt = np.uint8 if w == 8 else np.uint16
    rng = np.random.default_rng(70 + w)
    sizes = (1, 5, 31, 32, 33, 64, 100, 127, 128, 129, 200, 256) + ((300, 512) if w == 16 else ())
    for b in sizes:
        for density in (0.05, 0.6):
            for kind in ("anti", "dist"):
                ld = ((b + 32 + 15) // 16) * 16
                full = rng.integers(0, S + 1, (b + 12, ld)).astype(dt)
                v = rng.integers(1, min(S, 300), (b, b))
                tile = np.where(rng.random((b, b)) < density, v, S)
                if kind == "anti":
                    tile = S - tile
                full[:b, :b] = tile.astype(dt)
                pad = ((b + 15) // 16) * 16 if w == 8 else ((b + 7) // 8) * 8
                t_or = np.full((b, pad), 0 if kind == "anti" else S, dt)
                t_or[:, :b] = full[:b, :b]
                want = oracle_lib.semiring_close(t_or, w, kind)[:, :b]
                for blocked in (1, 0):
                    old = lib.smx_set_fw_pivot_blocked(blocked)
                    try:
                        dev = torch.from_numpy(full.copy()).cuda()
                        _native.check(lib.smx_fw_pivot(dev.data_ptr(), b, ld, w // 8, 0 if kind == "anti" else 1,
                                                       _native.stream_ptr()), "pivot")
                        got = dev.cpu().numpy()
                    finally:
                        lib.smx_set_fw_pivot_blocked(old)
                    np.testing.assert_array_equal(got[:b, :b], want, err_msg=f"b={b} {kind} blocked={blocked}")
                    outside = full.copy()
                    outside[:b, :b] = got[:b, :b]
                    np.testing.assert_array_equal(got, outside)          # nothing outside the tile moves


@pytest.mark.parametrize("m4r", [1, 0])
def test_bits_gemm_four_russians_and_predicate_kernels(m4r, oracle_lib):
    """The bit-packed product (engines.bool_mul_bits) on the four-Russians
    kernel and on the per-k predicate kernel: ragged shapes, densities from
    sparse to dense, small and large tile configurations, split-K -- equal to
    the oracle; and the bit Warshall closure with either kernel equal to the
    reference digest at C2's size."""
    from paper_1705_08743_b200 import _native
    lib = _native.lib()
    old = lib.smx_set_bits_m4r(m4r)
    try:
        rng = np.random.default_rng(80 + m4r)
        for (m, k, n), p in [((1, 1, 1), 0.5), ((300, 700, 1000), 0.01), ((300, 700, 1000), 0.3),
                             ((1024, 1024, 1024), 0.05), ((2049, 100, 33), 0.2), ((64, 5000, 70), 0.002),
                             ((4096, 256, 4096), 0.01)]:
            a = (rng.random((m, k)) < p).astype(np.uint8)
            b = (rng.random((k, n)) < p).astype(np.uint8)
            got = engines.bool_mul_bits(BoolMatrix.from_numpy(a), BoolMatrix.from_numpy(b)).blocks
            want = oracle_lib.bool_mul(oracle_lib.pack_bits(a), oracle_lib.pack_bits(b), k)
            np.testing.assert_array_equal(got, want, err_msg=f"{m}x{k}x{n} p={p} m4r={m4r}")
        cfg = workloads.CONFIGS["c2_bool_warshall"]
        (t,) = workloads.make_inputs(cfg)
        out = BoolMatrix.from_numpy(t).transitive_closure().blocks
        (d,) = [x for x in json_digests() if x["config"] == "c2_bool_warshall"]
        assert sha(out) == d["output_sha256"]
    finally:
        lib.smx_set_bits_m4r(old)


def json_digests():
    import json
    from pathlib import Path
    return json.loads((Path(__file__).parent / "golden" / "config_digests.json").read_text())
