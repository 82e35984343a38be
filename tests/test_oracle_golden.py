"""Pin the CPU oracle to the reference (CPU only).

The golden fixtures in tests/golden/ were produced by running the reference
package itself (tests/golden/make_golden.py).  Here the C restatement
(oracle/semimat_oracle.c) and the pure-Python restatement (oracle/naive.py)
must reproduce them exactly, so every later GPU-vs-oracle comparison is
anchored to the reference.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from oracle import naive
from paper_1705_08743_b200 import workloads

LIMIT = {8: 0xFF, 16: 0xFFFF, 32: 0xFFFFFFFF}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_small_products_match_reference(oracle_lib, small_cases):
    n = 0
    for meta, arr in small_cases:
        if meta["op"] != "mul":
            continue
        got = oracle_lib.semiring_mul(arr["a"], arr["b"], meta["inner"], meta["width"], meta["kind"])
        np.testing.assert_array_equal(got, arr["out"], err_msg=meta["name"])
        n += 1
    assert n >= 90


def test_small_closures_match_reference(oracle_lib, small_cases):
    n = 0
    for meta, arr in small_cases:
        if meta["op"] != "closure":
            continue
        got = oracle_lib.semiring_close(arr["t"], meta["width"], meta["kind"])
        np.testing.assert_array_equal(got, arr["out"], err_msg=meta["name"])
        n += 1
    assert n >= 70


def test_small_bool_match_reference(oracle_lib, small_cases):
    for meta, arr in small_cases:
        if meta["op"] == "bool_mul":
            a = oracle_lib.pack_bits(arr["a"])
            b = oracle_lib.pack_bits(arr["b"])
            got = oracle_lib.bool_mul(a, b, meta["inner"])
            np.testing.assert_array_equal(got, arr["out_blocks"], err_msg=meta["name"])
            np.testing.assert_array_equal(oracle_lib.unpack_bits(got, meta["cols"]), arr["out"])
        elif meta["op"] == "bool_closure":
            got = oracle_lib.bool_close(oracle_lib.pack_bits(arr["t"]))
            np.testing.assert_array_equal(got, arr["out_blocks"], err_msg=meta["name"])


def test_naive_oracles_match_reference(small_cases):
    """The definition-level restatements agree with the reference on small cases."""
    checked = 0
    for meta, arr in small_cases:
        if meta["op"] == "mul" and meta["rows"] * meta["inner"] * meta["cols"] <= 20000:
            w, inner, cols = meta["width"], meta["inner"], meta["cols"]
            a = arr["a"][:, :inner].astype(np.int64).tolist()
            b = arr["b"][:, :cols].astype(np.int64).tolist()
            fn = naive.antidist_product if meta["kind"] == "anti" else naive.dist_product
            assert fn(a, b, LIMIT[w]) == arr["out"][:, :cols].astype(np.int64).tolist(), meta["name"]
            checked += 1
        elif meta["op"] == "bool_mul" and meta["rows"] * meta["inner"] * meta["cols"] <= 20000:
            assert naive.bool_product(arr["a"].tolist(), arr["b"].tolist()) == arr["out"].tolist()
            checked += 1
        elif meta["op"] == "bool_closure" and meta["dim"] <= 6:
            t = arr["t"].tolist()
            assert naive.walk_closure(t) == arr["out"].tolist()
            assert naive.closure_by_squaring(t) == arr["out"].tolist()
            checked += 1
    assert checked >= 20


def test_samples_match_reference(oracle_lib, samples):
    """pkg/samples a4 x b4 and the chain3 / cycle3 closures (tests/test_cli.py:186-197)."""
    a = np.array(samples["a4"]["rows"], dtype=np.uint8)
    b = np.array(samples["b4"]["rows"], dtype=np.uint8)
    pad = lambda m: np.pad(m, ((0, 0), (0, 16 - m.shape[1])))  # noqa: E731
    got = oracle_lib.semiring_mul(pad(a), pad(b), 4, 8, "anti")[:, :4]
    assert got.tolist() == samples["a4_times_b4"]
    assert naive.antidist_product(a.astype(int).tolist(), b.astype(int).tolist(), 255) == \
        samples["a4_times_b4"]
    chain = samples["chain3"]
    t = pad(np.array(chain["antidist_adjacency"], dtype=np.uint8))
    assert oracle_lib.semiring_close(t, 8, "anti")[:, :3].tolist() == chain["antidist_closure"]
    assert chain["antidist_closure"][0][2] == 248          # README.md:84-93 golden value
    assert chain["dist_closure"][0][2] == 7
    cyc = samples["cycle3"]
    bits = oracle_lib.pack_bits(np.array(cyc["bool_adjacency"], dtype=np.uint8))
    assert oracle_lib.unpack_bits(oracle_lib.bool_close(bits), 3).tolist() == cyc["bool_closure"]
    assert cyc["bool_closure"] == [[1, 1, 1]] * 3


def test_scalar_golden_values():
    """Golden scalars of the reference tests (tests/test_scalars.py:31 etc.)."""
    from paper_1705_08743_b200 import scalars
    assert scalars.sat_mul(250, 252) == 247
    assert scalars.sat_mul(252, 251) == 248
    assert scalars.dist_mul(3, 4) == 7
    assert scalars.dist_mul(200, 100) == 255
    assert scalars.sat_neg(3) == 252
    with pytest.raises(ValueError):
        scalars.sat_limit(12)


def test_generators_are_pinned(config_digests):
    """The seeded generators reproduce the inputs the reference digests were made from."""
    for d in config_digests:
        if d["n"] > 4096:
            continue
        cfg = workloads.CONFIGS[d["config"]]
        inputs = workloads.make_inputs(cfg, d["n"])
        assert [sha(x) for x in inputs] == d["input_sha256"], d["config"]


@pytest.mark.parametrize("name", ["c1_bool_mul", "c2_bool_warshall", "c4_fw_u16", "c5_fw_u16",
                                  "c5_mul_u16", "c3_mul_u8", "c3_mul_u16"])
def test_oracle_reproduces_reference_digest(oracle_lib, config_digests, name):
    """C oracle == reference at every config's oracle size (full size for C1-C3)."""
    d = next(x for x in config_digests if x["config"] == name and x["n"] ==
             workloads.CONFIGS[name].oracle_n)
    cfg = workloads.CONFIGS[name]
    inputs = workloads.make_inputs(cfg, d["n"])
    if cfg.op == "bool_mul":
        out = oracle_lib.bool_mul(oracle_lib.pack_bits(inputs[0]), oracle_lib.pack_bits(inputs[1]), d["n"])
    elif cfg.op == "bool_closure":
        out = oracle_lib.bool_close(oracle_lib.pack_bits(inputs[0]))
    elif cfg.op == "mul":
        out = oracle_lib.semiring_mul(inputs[0], inputs[1], d["n"], cfg.width, "anti")
    else:
        out = oracle_lib.semiring_close(inputs[0], cfg.width, "anti")
    assert sha(out) == d["output_sha256"]


def test_matio_fixture_is_self_consistent():
    """The reference bytes decode to the reference rows (host-only check of the
    fixture itself, so a corrupt fixture fails on the CPU too)."""
    import json
    import struct
    from conftest import GOLDEN
    for case in json.loads((GOLDEN / "matio.json").read_text()):
        raw = bytes.fromhex(case["binary"])
        magic, tag, width, rows, cols = struct.unpack_from("<6sBBII", raw)
        assert magic == b"SRMAT1"
        if case["kind"] == "bool":
            assert tag == ord("B") and width == 0
            blocks = np.frombuffer(raw[16:], dtype="<u8").reshape(rows, -1)
            bits = np.unpackbits(blocks.view(np.uint8).reshape(rows, -1), axis=1, bitorder="little")
            assert bits[:, :cols].tolist() == case["bits"]
        else:
            dt = {8: "<u1", 16: "<u2", 32: "<u4"}[width]
            assert np.frombuffer(raw[16:], dtype=dt).reshape(rows, cols).tolist() == case["rows"]


def test_blocked_oracle_matches_reference_cases(oracle_lib, small_cases):
    """The cache-blocked closure (used for the full-size C5 pin) reproduces
    every reference closure fixture, anti and dist, all widths."""
    n = 0
    for meta, arr in small_cases:
        if meta["op"] != "closure":
            continue
        got = oracle_lib.semiring_close_blocked(arr["t"], meta["width"], meta["kind"])
        np.testing.assert_array_equal(got, arr["out"], err_msg=meta["name"])
        n += 1
    assert n >= 70


@pytest.mark.parametrize("width,kind", [(8, "anti"), (16, "dist"), (32, "anti"), (16, "anti")])
def test_blocked_oracle_matches_plain_sweep(oracle_lib, width, kind):
    """Blocked order == the reference's vertex-at-a-time sweep on sizes that
    straddle the 128 block and the 2048 column tile (ragged, padded)."""
    rng = np.random.default_rng(width * 7 + len(kind))
    S = LIMIT[width]
    dt = {8: np.uint8, 16: np.uint16, 32: np.uint32}[width]
    lanes = {8: 16, 16: 8, 32: 4}[width]
    for n in (1, 127, 129, 300, 2100):
        cp = -(-n // lanes) * lanes
        mask = rng.random((n, n)) < min(1.0, 3.0 / n)
        vals = S - rng.integers(1, 1000 if width > 8 else 254, size=(n, n))
        t = np.full((n, cp), 0 if kind == "anti" else S, dtype=dt)
        t[:, :n] = np.where(mask, vals if kind == "anti" else S - vals, t[:, :n])
        np.testing.assert_array_equal(oracle_lib.semiring_close_blocked(t, width, kind),
                                      oracle_lib.semiring_close(t, width, kind), err_msg=str(n))


def test_blocked_oracle_reproduces_reference_c4_8192(oracle_lib, config_digests):
    """The blocked oracle at the full C4 size equals the reference's own
    sha256 (a 26-minute run of the reference's numpy engine), so the
    full-size C5 digest it produced (tools/oracle_full_digest.py) is anchored
    to the reference at scale, not only to the plain restatement."""
    d = next(x for x in config_digests if x["config"] == "c4_fw_u16" and x["n"] == 8192)
    (t,) = workloads.make_inputs(workloads.CONFIGS["c4_fw_u16"], 8192)
    assert sha(t) == d["input_sha256"][0]
    assert sha(oracle_lib.semiring_close_blocked(t, 16, "anti")) == d["output_sha256"]
