"""Randomised differential run against the CPU oracle (development aid; the
oracle is the checker here, as in tests/): products and closures of the lane
types at random shapes, widths, kinds and value regimes (sparse small weights,
lanes at the edges of the 2^(w-2) certificate and of the 2^(w-1) bound, full
range, near S), Boolean products and closures at random densities, all through
the public classes.  Every result must equal the oracle's bit for bit.

    python tools/fuzz_parity.py [seconds] [seed] [big|mid|sharded|hoststream]

`big`: closures near n = 8192 / 16384 (the packed phase 3, look-ahead, ragged
last blocks; against the oracle's blocked closure), products of a few
thousand squared, Boolean closures and products up to 17000 / 9000, from
host arrays and device tensors.  `mid`: closures at n = 1300-6700 and
Boolean closures at 1800-7000 (the sizes between the other two modes).
`hoststream`: mid-size closures of host arrays with the streamed host-buffer
schedule forced (smx_set_fw_host_stream(2)).

Prints one JSON line per failure and a summary line."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle  # noqa: E402
from paper_1705_08743_b200 import AntidistMatrix, BoolMatrix, DistMatrix  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(seed)
DT = {8: np.uint8, 16: np.uint16, 32: np.uint32}


def lanes_per_chunk(w):
    return 16 // (w // 8)


def dist_values(r, c, w, regime):
    """Distance-form cells (S = unreachable)."""
    S = (1 << w) - 1
    p = float(rng.choice([0.02, 0.1, 0.5, 1.0]))
    if regime == "small":
        v = rng.integers(0, min(S, 1001), (r, c), dtype=np.uint64)
    elif regime == "cert_edge":      # around 2^(w-2), the product-wide certificate
        q = 1 << (w - 2)
        v = q - 3 + rng.integers(0, 6, (r, c), dtype=np.uint64)
        v[rng.random((r, c)) < 0.7] = rng.integers(0, 50)
    elif regime == "bound_edge":     # around 2^(w-1), the per-tile bounded test
        h = 1 << (w - 1)
        v = h - 3 + rng.integers(0, 6, (r, c), dtype=np.uint64)
        v[rng.random((r, c)) < 0.7] = rng.integers(0, 50)
    elif regime == "near_s":
        v = S - rng.integers(0, 4, (r, c), dtype=np.uint64)
        v[rng.random((r, c)) < 0.5] = rng.integers(0, 5)
    else:                            # full range
        v = rng.integers(0, S + 1, (r, c), dtype=np.uint64)
    v[rng.random((r, c)) > p] = S
    return v


def padded(v, w, kind):
    S = (1 << w) - 1
    r, c = v.shape
    L = lanes_per_chunk(w)
    cp = -(-c // L) * L
    out = np.full((r, cp), S, dtype=np.uint64)     # distance-form pad = S
    out[:, :c] = v
    if kind == "anti":
        out = S - out
    return out.astype(DT[w])


def rand_dim(lo, hi):
    return int(np.exp(rng.uniform(np.log(lo), np.log(hi))))


def case_lane_mul():
    w = int(rng.choice([8, 16, 16, 32]))
    kind = str(rng.choice(["anti", "dist"]))
    if rng.random() < 0.35:          # shapes that take the packed kernel
        M, N, K = rand_dim(1500, 2600), rand_dim(1500, 2600), rand_dim(256, 700)
    else:
        M, N, K = rand_dim(1, 1500), rand_dim(1, 1500), rand_dim(1, 900)
    regime = str(rng.choice(["small", "cert_edge", "bound_edge", "near_s", "full"]))
    a = padded(dist_values(M, K, w, regime), w, kind)
    b = padded(dist_values(K, N, w, regime), w, kind)
    cls = AntidistMatrix if kind == "anti" else DistMatrix
    got = (cls(M, K, w, a) * cls(K, N, w, b)).data
    want = oracle.semiring_mul(a, b, K, w, kind)
    return {"op": "lane_mul", "w": w, "kind": kind, "M": M, "N": N, "K": K, "regime": regime}, np.array_equal(got, want)


def case_lane_close():
    w = int(rng.choice([8, 16, 16, 32]))
    kind = str(rng.choice(["anti", "dist"]))
    n = rand_dim(1, 1300)
    regime = str(rng.choice(["small", "small", "cert_edge", "bound_edge", "near_s", "full"]))
    v = dist_values(n, n, w, regime)
    if rng.random() < 0.7:
        v[np.arange(n), np.arange(n)] = 0
    t = padded(v, w, kind)
    cls = AntidistMatrix if kind == "anti" else DistMatrix
    got = cls(n, n, w, t).transitive_closure().data
    want = oracle.semiring_close(t, w, kind)
    return {"op": "lane_close", "w": w, "kind": kind, "n": n, "regime": regime}, np.array_equal(got, want)


def case_bool_mul():
    M, N, K = rand_dim(1, 2000), rand_dim(1, 2000), rand_dim(1, 2000)
    p = float(rng.choice([0.001, 0.01, 0.05, 0.3, 0.9]))
    a = (rng.random((M, K)) < p).astype(np.uint8)
    b = (rng.random((K, N)) < p).astype(np.uint8)
    got = (BoolMatrix.from_numpy(a) * BoolMatrix.from_numpy(b)).blocks
    want = oracle.bool_mul(oracle.pack_bits(a), oracle.pack_bits(b), K)
    return {"op": "bool_mul", "M": M, "N": N, "K": K, "p": p}, np.array_equal(got, want)


def case_bool_close():
    n = rand_dim(1, 1800)
    p = float(rng.choice([0.5, 1.0, 2.0, 4.0])) / max(n, 1)
    t = (rng.random((n, n)) < p).astype(np.uint8)
    m = BoolMatrix.from_numpy(t)
    got = (m.transitive_closure() if rng.random() < 0.7 else m.reflexive_transitive_closure())
    want = oracle.bool_close(oracle.pack_bits(t))
    gb = got.blocks
    if not np.array_equal(gb, want):        # (reflexive: join the identity on the oracle side)
        eye = oracle.pack_bits(np.eye(n, dtype=np.uint8))
        want = want | eye
    return {"op": "bool_close", "n": n, "p": p}, np.array_equal(gb, want)


def _operand(cls, r, c, w, arr):
    """Half the time a device tensor (device-resident paths), else the numpy
    array itself (host-backed paths: staged closure, streamed product)."""
    if HOSTSTREAM or rng.random() < 0.5:
        return cls(r, c, w, arr), "host"
    st = {8: np.int8, 16: np.int16, 32: np.int32}[w]
    tt = {8: torch.uint8, 16: torch.uint16, 32: torch.uint32}[w]
    return cls(r, c, w, torch.from_numpy(arr.view(st)).cuda().view(tt)), "device"


def case_big_close():
    """Closures near n = 8192 (and sometimes 16384): the packed phase 3 with
    per-tile flags, certified rounds, look-ahead and ragged last blocks, at
    value regimes the configs' generators do not produce."""
    w = int(rng.choice([8, 16, 16, 16, 32]))
    kind = str(rng.choice(["anti", "dist"]))
    if MID:
        n = int(rng.integers(1300, 6700))
    elif rng.random() < 0.12 and w == 16:
        n = 16384 - 8 * int(rng.integers(0, 120))
    else:
        n = 8600 - 8 * int(rng.integers(0, 250))
    regime = str(rng.choice(["cert_edge", "bound_edge", "near_s", "full", "small"]))
    v = dist_values(n, n, w, regime)
    v[np.arange(n), np.arange(n)] = 0
    t = padded(v, w, kind)
    cls = AntidistMatrix if kind == "anti" else DistMatrix
    m, where = _operand(cls, n, n, w, t)
    got = m.transitive_closure().data
    want = oracle.semiring_close_blocked(t, w, kind)
    return ({"op": "big_close", "w": w, "kind": kind, "n": n, "regime": regime, "operand": where},
            np.array_equal(got, want))


def case_big_mul():
    """Products of a few thousand squared with ragged dimensions: the packed
    kernel with K chunks, the certificate, the streamed host product."""
    w = int(rng.choice([8, 16, 16, 32]))
    kind = str(rng.choice(["anti", "dist"]))
    M, N, K = (int(rng.integers(2500, 6000)) for _ in range(3))
    regime = str(rng.choice(["small", "cert_edge", "bound_edge", "near_s", "full"]))
    a = padded(dist_values(M, K, w, regime), w, kind)
    b = padded(dist_values(K, N, w, regime), w, kind)
    cls = AntidistMatrix if kind == "anti" else DistMatrix
    ma, wa = _operand(cls, M, K, w, a)
    mb, wb = _operand(cls, K, N, w, b)
    got = (ma * mb).data
    want = oracle.semiring_mul(a, b, K, w, kind)
    return ({"op": "big_mul", "w": w, "kind": kind, "M": M, "N": N, "K": K, "regime": regime,
             "operands": wa + "/" + wb}, np.array_equal(got, want))


def case_big_sharded():
    """The row-panel-sharded closure's GPU ops at sizes that reach the packed
    (and certified) skip-GEMM: one rank's pipelined schedule (Python and C++
    orchestration, world = 1), or 2-4 ranks in lockstep on this one GPU (the
    broadcast becomes a device copy; no rank waits on another)."""
    from paper_1705_08743_b200 import sharded
    kind = str(rng.choice(["anti", "dist"]))
    n = int(rng.integers(500, 1100)) * 8
    regime = str(rng.choice(["cert_edge", "bound_edge", "full", "small", "small"]))
    v = dist_values(n, n, 16, regime)
    v[np.arange(n), np.arange(n)] = 0
    full = padded(v, 16, kind)
    mode = str(rng.choice(["python1", "native1", "lockstep"]))
    anti = kind == "anti"
    if mode == "python1":
        fw = sharded.ShardedFW(n=n, rank=0, world=1, ops=sharded.CudaFwOps(16, anti=anti))
        got = fw.run(torch.from_numpy(full.view(np.int16)).cuda().view(torch.uint16)).cpu().numpy()
        world = 1
    elif mode == "native1":
        fw = sharded.NativeShardedFW(n, 0, 1, 16, anti=anti)
        got = fw.run(torch.from_numpy(full.view(np.int16)).cuda().view(torch.uint16)).cpu().numpy()
        world = 1
    else:
        world = int(rng.integers(2, 5))
        ranks = []
        for r in range(world):
            fw = sharded.ShardedFW(n=n, rank=r, world=world, ops=sharded.CudaFwOps(16, anti=anti))
            loc = torch.from_numpy(full[fw.row0:fw.row1].copy().view(np.int16)).cuda().view(torch.uint16)
            ranks.append((fw, loc))
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
    want = oracle.semiring_close_blocked(full, 16, kind)
    return ({"op": "big_sharded", "mode": mode, "world": world, "kind": kind, "n": n, "regime": regime},
            np.array_equal(got.view(np.uint16), want))


def case_big_bool():
    if rng.random() < 0.5:
        n = int(rng.integers(1800, 7000)) if MID else int(rng.integers(7000, 17000))
        p = float(rng.choice([0.5, 1.0, 2.0, 4.0])) / n
        t = (rng.random((n, n)) < p).astype(np.uint8)
        got = BoolMatrix.from_numpy(t).transitive_closure().blocks
        want = oracle.bool_close(oracle.pack_bits(t))
        return {"op": "big_bool_close", "n": n, "p": p}, np.array_equal(got, want)
    M, N, K = (int(rng.integers(3000, 9000)) for _ in range(3))
    p = float(rng.choice([0.0005, 0.005, 0.05]))
    a = (rng.random((M, K)) < p).astype(np.uint8)
    b = (rng.random((K, N)) < p).astype(np.uint8)
    got = (BoolMatrix.from_numpy(a) * BoolMatrix.from_numpy(b)).blocks
    want = oracle.bool_mul(oracle.pack_bits(a), oracle.pack_bits(b), K)
    return {"op": "big_bool_mul", "M": M, "N": N, "K": K, "p": p}, np.array_equal(got, want)


def case_entrywise():
    """lanewise min / max / absolute difference / complement
    and the Boolean bridge, against numpy on the valid columns; padding lanes
    must hold the result type's (+)-identity (antidist.py:128-156, :213-224)."""
    w = int(rng.choice([8, 16, 32]))
    kind = str(rng.choice(["anti", "dist"]))
    S = (1 << w) - 1
    r, c = rand_dim(1, 3000), rand_dim(1, 3000)
    a = padded(dist_values(r, c, w, "full"), w, kind)
    b = padded(dist_values(r, c, w, str(rng.choice(["full", "small", "near_s"]))), w, kind)
    cls = AntidistMatrix if kind == "anti" else DistMatrix
    ma, mb = cls(r, c, w, a), cls(r, c, w, b)
    av, bv = a[:, :c].astype(np.uint64), b[:, :c].astype(np.uint64)
    pad = 0 if kind == "anti" else S
    ok = True
    for name, got, want in (("and", (ma & mb).data, np.minimum(av, bv)), ("or", (ma | mb).data, np.maximum(av, bv)),
                            ("xor", (ma ^ mb).data, np.maximum(av, bv) - np.minimum(av, bv))):
        ok = ok and np.array_equal(got[:, :c].astype(np.uint64), want) and bool((got[:, c:] == pad).all())
    inv = ~ma
    ok = ok and type(inv) is (DistMatrix if kind == "anti" else AntidistMatrix)
    ok = ok and np.array_equal(inv.data[:, :c].astype(np.uint64), S - av)
    ok = ok and bool((inv.data[:, c:] == (S if kind == "anti" else 0)).all())
    if kind == "anti":
        bits = (rng.random((r, c)) < 0.3).astype(np.uint8)
        lanes = AntidistMatrix.from_boolmat(BoolMatrix.from_numpy(bits), w)
        ok = ok and np.array_equal(lanes.data[:, :c].astype(np.uint64), bits.astype(np.uint64) * S)
        ok = ok and bool((lanes.data[:, c:] == 0).all())
        ok = ok and np.array_equal(ma.to_boolmat().to_numpy(), (av != 0).astype(np.uint8))
    return {"op": "entrywise", "w": w, "kind": kind, "r": r, "c": c}, bool(ok)


def case_batch():
    """Many small problems per launch (batch.py): stacked Boolean products
    (tensor cores on 128-multiple shapes, bits otherwise), stacked Boolean
    closures (n <= 512) and stacked lane closures (n <= 128)."""
    from paper_1705_08743_b200 import batch
    which = str(rng.choice(["bool_mul_tc", "bool_mul_bits", "bool_close", "lane_close"]))
    nb = int(rng.integers(1, 24))
    ok = True
    if which.startswith("bool_mul"):
        if which == "bool_mul_tc":
            M, N, K = (128 * int(rng.integers(1, 6)) for _ in range(3))
            K += 128
        else:
            M, N, K = rand_dim(1, 500), rand_dim(1, 500), rand_dim(1, 500)
        p = float(rng.choice([0.01, 0.05, 0.3]))
        As = [(rng.random((M, K)) < p).astype(np.uint8) for _ in range(nb)]
        Bs = [(rng.random((K, N)) < p).astype(np.uint8) for _ in range(nb)]
        got = batch.bool_mul_many([BoolMatrix.from_numpy(a) for a in As], [BoolMatrix.from_numpy(b) for b in Bs])
        for g, a, b in zip(got, As, Bs):
            ok = ok and np.array_equal(g.blocks, oracle.bool_mul(oracle.pack_bits(a), oracle.pack_bits(b), K))
        desc = {"M": M, "N": N, "K": K}
    elif which == "bool_close":
        n = rand_dim(1, 512)
        Ts = [(rng.random((n, n)) < 2.0 / n).astype(np.uint8) for _ in range(nb)]
        got = batch.bool_closure_many([BoolMatrix.from_numpy(t) for t in Ts])
        for g, t in zip(got, Ts):
            ok = ok and np.array_equal(g.blocks, oracle.bool_close(oracle.pack_bits(t)))
        desc = {"n": n}
    else:
        w = int(rng.choice([8, 16, 32]))
        kind = str(rng.choice(["anti", "dist"]))
        n = rand_dim(1, 128)
        regime = str(rng.choice(["small", "cert_edge", "bound_edge", "near_s", "full"]))
        Ts = [padded(dist_values(n, n, w, regime), w, kind) for _ in range(nb)]
        cls = AntidistMatrix if kind == "anti" else DistMatrix
        got = batch.closure_many([cls(n, n, w, t) for t in Ts])
        for g, t in zip(got, Ts):
            ok = ok and np.array_equal(g.data, oracle.semiring_close(t, w, kind))
        desc = {"n": n, "w": w, "kind": kind, "regime": regime}
    return dict({"op": "batch_" + which, "batch": nb}, **desc), bool(ok)


cases = [case_lane_mul, case_lane_mul, case_lane_close, case_bool_mul, case_bool_close, case_entrywise, case_batch]
MID = len(sys.argv) > 3 and sys.argv[3] in ("mid", "hoststream")
if MID:
    cases = [case_big_close, case_big_close, case_big_bool]
HOSTSTREAM = len(sys.argv) > 3 and sys.argv[3] == "hoststream"
if HOSTSTREAM:
    # every host-backed closure takes the streamed schedule (ingest groups,
    # staged copies in and out, egress products), whatever its size
    from paper_1705_08743_b200 import _native
    _native.lib().smx_set_fw_host_stream(2)
    cases = [case_big_close]
if len(sys.argv) > 3 and sys.argv[3] == "big":
    cases = [case_big_close, case_big_close, case_big_mul, case_big_bool, case_big_sharded]
if len(sys.argv) > 3 and sys.argv[3] == "sharded":
    cases = [case_big_sharded]
counts, fails = {}, 0
t0 = time.time()
i = 0
while time.time() - t0 < budget:
    fn = cases[i % len(cases)]
    i += 1
    try:
        desc, ok = fn()
    except Exception as ex:   # noqa: BLE001
        desc, ok = {"op": fn.__name__, "error": repr(ex)[:300]}, False
    counts[desc["op"]] = counts.get(desc["op"], 0) + 1
    if not ok:
        fails += 1
        print(json.dumps({"FAIL": desc, "case_index": i, "seed": seed}), flush=True)
torch.cuda.synchronize()
try:   # resident and device memory at the end: a leak in a host or staging path would show here
    import psutil
    rss = round(psutil.Process().memory_info().rss / 2 ** 30, 2)
except Exception:   # noqa: BLE001
    rss = None
print(json.dumps({"seed": seed, "seconds": round(time.time() - t0, 1), "cases": counts, "failures": fails,
                  "rss_gib": rss, "cuda_reserved_gib": round(torch.cuda.memory_reserved() / 2 ** 30, 2)}))
