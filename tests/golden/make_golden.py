"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py            # small cases + samples + digests
    python tests/golden/make_golden.py --big      # also the n=8192 FW digest (~30 min)

The reference package (pure Python + numpy) is imported from
/root/reference/pkg/src; its numpy vector engines produce every output
stored here.  Outputs:

* small_cases.npz  -- inputs and reference outputs of many small products and
  closures (widths 8/16/32, anti-distance, distance, Boolean), incl. ragged
  and padded shapes, empty graphs, saturating chains, all-identity matrices.
* samples.json     -- the reference's sample files (pkg/samples) as matrices,
  with the reference's product / closure results.
* config_digests.json -- sha256 of the reference output for every
  BASELINE.json config at its oracle size, inputs from
  paper_1705_08743_b200.workloads (same generator, same seed).

Nothing here is read by the product; tests/ compare the C oracle and the GPU
path against these files.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import random
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
REF_SRC = Path("/root/reference/pkg/src")
REF_SAMPLES = Path("/root/reference/pkg/samples")
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REF_SRC))

from semimat import kernels  # noqa: E402  (the reference)
from semimat.antidist import AntidistMatrix, DistMatrix  # noqa: E402
from semimat.boolmat import BoolMatrix  # noqa: E402

from paper_1705_08743_b200 import workloads  # noqa: E402

LANE_CLS = {"anti": AntidistMatrix, "dist": DistMatrix}


def digest(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def ref_bool(bits: np.ndarray) -> BoolMatrix:
    rows, cols = bits.shape
    m = BoolMatrix(rows, cols)
    nblk = m.block_columns
    padded = np.zeros((rows, nblk * 64), dtype=np.uint8)
    padded[:, :cols] = bits
    m._blocks[...] = np.packbits(padded, axis=1, bitorder="little").view("<u8")
    assert m.to_lists() == bits.tolist()
    return m


def ref_lane(kind: str, data: np.ndarray, cols: int, width: int):
    cls = LANE_CLS[kind]
    return cls(data.shape[0], cols, width, np.ascontiguousarray(data))


def rand_lane(rng: random.Random, rows: int, cols: int, width: int, kind: str,
              ident_chance: float) -> np.ndarray:
    limit = (1 << width) - 1
    ident = 0 if kind == "anti" else limit
    cls = LANE_CLS[kind]
    m = cls(rows, cols, width)
    vals = [[ident if rng.random() < ident_chance else rng.randrange(limit + 1)
             for _ in range(cols)] for _ in range(rows)]
    m._data[:, :cols] = np.array(vals, dtype=m._data.dtype)
    return np.array(m._data)


def rand_graph_lane(rng: random.Random, dim: int, p: float, wmax: int, width: int,
                    kind: str) -> np.ndarray:
    cls = LANE_CLS[kind]
    edges = [(u, v, rng.randint(0, wmax)) for u in range(dim) for v in range(dim)
             if rng.random() < p]
    return np.array(cls.from_edges(dim, edges, width)._data)


def small_cases():
    cases = {}
    manifest = []
    rng = random.Random(20260101)

    def add(name, meta, **arrays):
        for k, v in arrays.items():
            cases[f"{name}__{k}"] = v
        manifest.append(dict(name=name, **meta))

    with kernels.forced_vector():
        # -- lane products: random ragged shapes, all widths, both encodings
        idx = 0
        for width in (8, 16, 32):
            for kind in ("anti", "dist"):
                shapes = [(1, 1, 1), (1, 7, 3), (5, 1, 9), (17, 33, 65), (64, 64, 64),
                          (3, 130, 5)]
                shapes += [(rng.randint(1, 48), rng.randint(1, 48), rng.randint(1, 48))
                           for _ in range(10)]
                for rows, inner, cols in shapes:
                    ic = rng.choice([0.0, 0.3, 0.7, 0.95])
                    a = rand_lane(rng, rows, inner, width, kind, ic)
                    b = rand_lane(rng, inner, cols, width, kind, ic)
                    out = (ref_lane(kind, a, inner, width) * ref_lane(kind, b, cols, width))._data
                    add(f"mul{idx}", dict(op="mul", kind=kind, width=width, rows=rows,
                                          inner=inner, cols=cols), a=a, b=b, out=np.array(out))
                    idx += 1
        # -- lane closures: random digraphs, saturating chains, empty, full
        idx = 0
        for width in (8, 16, 32):
            for kind in ("anti", "dist"):
                specs = [(rng.randint(1, 80), rng.uniform(0.02, 0.4),
                          rng.choice([10, 200, (1 << width) - 1])) for _ in range(8)]
                specs += [(1, 1.0, 5), (37, 0.0, 1), (70, 0.08, 1000), (130, 0.03, 5000)]
                for dim, p, wmax in specs:
                    wmax = min(wmax, (1 << width) - 1)
                    t = rand_graph_lane(rng, dim, p, wmax, width, kind)
                    out = ref_lane(kind, t, dim, width).transitive_closure()._data
                    add(f"close{idx}", dict(op="closure", kind=kind, width=width, dim=dim),
                        t=t, out=np.array(out))
                    idx += 1
                # chain of 30 edges of weight 10 (saturates at u8)
                cls = LANE_CLS[kind]
                chain = cls.from_edges(31, [(i, i + 1, 10) for i in range(30)], width)
                out = chain.transitive_closure()._data
                add(f"close{idx}", dict(op="closure", kind=kind, width=width, dim=31),
                    t=np.array(chain._data), out=np.array(out))
                idx += 1
        # -- Boolean products and closures
        idx = 0
        shapes = [(1, 1, 1), (3, 64, 65), (65, 63, 129), (128, 128, 128), (100, 257, 31)]
        shapes += [(rng.randint(1, 140), rng.randint(1, 140), rng.randint(1, 140))
                   for _ in range(10)]
        for rows, inner, cols in shapes:
            p = rng.choice([0.01, 0.05, 0.3])
            a = (np.array([[rng.random() < p for _ in range(inner)] for _ in range(rows)])
                 .astype(np.uint8))
            b = (np.array([[rng.random() < p for _ in range(cols)] for _ in range(inner)])
                 .astype(np.uint8))
            out = ref_bool(a) * ref_bool(b)
            add(f"bmul{idx}", dict(op="bool_mul", rows=rows, inner=inner, cols=cols),
                a=a, b=b, out=np.array(out.to_lists(), dtype=np.uint8),
                out_blocks=np.array(out._blocks))
            idx += 1
        idx = 0
        for dim in [1, 2, 6, 63, 64, 65, 130, 200, 257] + [rng.randint(3, 300) for _ in range(6)]:
            p = rng.choice([1.5 / dim, 2.0 / dim, 0.05])
            t = np.array([[rng.random() < p for _ in range(dim)] for _ in range(dim)]).astype(np.uint8)
            m = ref_bool(t)
            c = m.transitive_closure()
            r = m.reflexive_transitive_closure()
            add(f"bclose{idx}", dict(op="bool_closure", dim=dim), t=t,
                out=np.array(c.to_lists(), dtype=np.uint8),
                refl=np.array(r.to_lists(), dtype=np.uint8),
                out_blocks=np.array(c._blocks))
            idx += 1
    return cases, manifest


def entrywise_cases():
    """Entrywise |, &, ^, ~ of the reference (antidist.py:128-156,
    boolmat.py:120-137), incl. padding restoration and the Boolean bridge."""
    cases, manifest = {}, []
    rng = random.Random(777)
    with kernels.forced_vector():
        idx = 0
        for width in (8, 16, 32):
            for kind in ("anti", "dist"):
                for rows, cols in [(1, 1), (3, 17), (5, 64), (9, 33), (2, 130)]:
                    a = rand_lane(rng, rows, cols, width, kind, 0.3)
                    b = rand_lane(rng, rows, cols, width, kind, 0.3)
                    ma, mb = ref_lane(kind, a, cols, width), ref_lane(kind, b, cols, width)
                    name = f"ew{idx}"
                    manifest.append(dict(name=name, kind=kind, width=width, rows=rows, cols=cols))
                    cases[f"{name}__a"], cases[f"{name}__b"] = a, b
                    cases[f"{name}__or"] = np.array((ma | mb)._data)
                    cases[f"{name}__and"] = np.array((ma & mb)._data)
                    cases[f"{name}__xor"] = np.array((ma ^ mb)._data)
                    cases[f"{name}__inv"] = np.array((~ma)._data)
                    if kind == "anti":
                        cases[f"{name}__toboolmat"] = np.array(ma.to_boolmat().to_lists(), dtype=np.uint8)
                    idx += 1
        for rows, cols in [(1, 1), (4, 63), (7, 64), (5, 65), (3, 200)]:
            a = np.array([[rng.random() < 0.4 for _ in range(cols)] for _ in range(rows)], dtype=np.uint8)
            b = np.array([[rng.random() < 0.4 for _ in range(cols)] for _ in range(rows)], dtype=np.uint8)
            ma, mb = ref_bool(a), ref_bool(b)
            name = f"bew{idx}"
            manifest.append(dict(name=name, kind="bool", rows=rows, cols=cols))
            cases[f"{name}__a"], cases[f"{name}__b"] = a, b
            for op, m in (("or", ma | mb), ("and", ma & mb), ("xor", ma ^ mb), ("inv", ~ma)):
                cases[f"{name}__{op}"] = np.array(m._blocks)
            for w in (8, 16):
                cases[f"{name}__fromboolmat{w}"] = np.array(AntidistMatrix.from_boolmat(ma, w)._data)
            idx += 1
    return cases, manifest


def matio_cases():
    """The reference's SRMAT1 bytes and text for assorted matrices
    (matio.py:37-149), incl. the 65-column Boolean padding case."""
    from semimat import matio
    rng = random.Random(4242)
    out = []
    for rows, cols in [(1, 1), (3, 65), (5, 64), (2, 130)]:
        bits = np.array([[rng.random() < 0.4 for _ in range(cols)] for _ in range(rows)], dtype=np.uint8)
        m = ref_bool(bits)
        out.append(dict(kind="bool", bits=bits.tolist(), binary=matio.to_binary(m).hex(),
                        text=matio.format_text(m)))
    for width in (8, 16, 32):
        for kind in ("anti", "dist"):
            for rows, cols in [(1, 1), (3, 17), (4, 9)]:
                data = rand_lane(rng, rows, cols, width, kind, 0.3)
                m = ref_lane(kind, data, cols, width)
                out.append(dict(kind=kind, width=width, rows=m.to_lists(), binary=matio.to_binary(m).hex(),
                                text=matio.format_text(m)))
    return out


def samples():
    """The reference's sample files, parsed with the reference's own loaders."""
    from semimat import graphio, matio
    out = {}
    a4 = matio.load(REF_SAMPLES / "a4.antidist")
    b4 = matio.load(REF_SAMPLES / "b4.antidist")
    out["a4"] = dict(width=a4.width, rows=a4.to_lists())
    out["b4"] = dict(width=b4.width, rows=b4.to_lists())
    out["a4_times_b4"] = (a4 * b4).to_lists()
    for name in ("chain3", "cycle3"):
        spec = graphio.parse_edge_list((REF_SAMPLES / f"{name}.graph").read_text())
        out[name] = dict(
            vertices=spec.vertex_count if hasattr(spec, "vertex_count") else None,
            bool_adjacency=graphio.bool_adjacency(spec).to_lists(),
            bool_closure=graphio.bool_adjacency(spec).transitive_closure().to_lists(),
            bool_reflexive=graphio.bool_adjacency(spec).reflexive_transitive_closure().to_lists(),
            antidist_adjacency=graphio.antidist_adjacency(spec, 8).to_lists(),
            antidist_closure=graphio.antidist_adjacency(spec, 8).transitive_closure().to_lists(),
            dist_adjacency=graphio.dist_adjacency(spec, 8).to_lists(),
            dist_closure=graphio.dist_adjacency(spec, 8).transitive_closure().to_lists(),
        )
    return out


def config_digest(name: str, n: int) -> dict:
    cfg = workloads.CONFIGS[name]
    inputs = workloads.make_inputs(cfg, n)
    t0 = time.perf_counter()
    with kernels.forced_vector():
        if cfg.op == "bool_mul":
            out = (ref_bool(inputs[0]) * ref_bool(inputs[1]))._blocks
        elif cfg.op == "bool_closure":
            out = ref_bool(inputs[0]).transitive_closure()._blocks
        elif cfg.op == "mul":
            a = ref_lane("anti", inputs[0], n, cfg.width)
            b = ref_lane("anti", inputs[1], n, cfg.width)
            out = (a * b)._data
        else:
            out = ref_lane("anti", inputs[0], n, cfg.width).transitive_closure()._data
    secs = time.perf_counter() - t0
    return dict(config=name, n=n, seed=cfg.seed, op=cfg.op, width=cfg.width,
                input_sha256=[digest(x) for x in inputs], output_sha256=digest(out),
                output_nonzero=int(np.count_nonzero(out)), ref_seconds=round(secs, 3),
                layout="uint64 blocks" if cfg.op.startswith("bool") else "padded lanes")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also digest C4 at n=8192")
    ap.add_argument("--only-digests", action="store_true")
    ap.add_argument("--only-entrywise", action="store_true")
    args = ap.parse_args()

    if not args.only_digests:
        cases, manifest = entrywise_cases()
        np.savez_compressed(HERE / "entrywise.npz", **cases)
        (HERE / "entrywise.json").write_text(json.dumps(manifest, indent=0))
        print(f"entrywise cases: {len(manifest)}")
        (HERE / "matio.json").write_text(json.dumps(matio_cases(), indent=0))
        if args.only_entrywise:
            return

    if not args.only_digests:
        cases, manifest = small_cases()
        np.savez_compressed(HERE / "small_cases.npz", **cases)
        (HERE / "small_cases.json").write_text(json.dumps(manifest, indent=0))
        (HERE / "samples.json").write_text(json.dumps(samples(), indent=1))
        print(f"small cases: {len(manifest)}")

    path = HERE / "config_digests.json"
    existing = json.loads(path.read_text()) if path.exists() else []
    done = {(d["config"], d["n"]) for d in existing}
    todo = [(name, cfg.oracle_n) for name, cfg in workloads.CONFIGS.items()]
    if args.big:
        todo.append(("c4_fw_u16", 8192))
    for name, n in todo:
        if (name, n) in done:
            continue
        d = config_digest(name, n)
        print(json.dumps(d))
        existing.append(d)
        path.write_text(json.dumps(existing, indent=1))


if __name__ == "__main__":
    main()
