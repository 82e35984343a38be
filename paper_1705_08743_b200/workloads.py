"""Seeded synthetic inputs for the BASELINE.json configurations.

There is no public dataset for this path: BASELINE.json defines the inputs
as seeded random graphs.  One ``np.random.default_rng(seed)`` stream per
config is filled in row chunks (so n = 32768 never materialises an n x n
float64 array), and the same function at a smaller n gives the oracle-size
cross-check instance (never a slice of the large one).

Encodings follow the reference:
* Boolean: 0/1 per entry (pkg/src/semimat/boolmat.py); one byte per entry.
* anti-distance: value S - w for an edge of weight w, 0 = no edge
  (pkg/src/semimat/antidist.py:191-211, scalars.py:3-13); "diagonal 0"
  (distance zero) is S on the diagonal.
* distance (DistMatrix): the complement S - a (antidist.py:151-156).
Rows are padded to whole 128-bit blocks with the class's additive identity
(antidist.py:38-55): 0 for anti-distance.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

LANES = {8: 16, 16: 8, 32: 4}
DTYPES = {8: np.uint8, 16: np.uint16, 32: np.uint32}
_CHUNK_CELLS = 1 << 24


def padded_cols(cols: int, width: int) -> int:
    lanes = LANES[width]
    return -(-cols // lanes) * lanes


def _chunk_rows(n: int) -> int:
    return max(1, _CHUNK_CELLS // max(n, 1))


def bernoulli_bits(rng: np.random.Generator, rows: int, cols: int, p: float,
                   no_self_loops: bool = False) -> np.ndarray:
    """0/1 uint8 matrix with iid Bernoulli(p) entries (row-chunked)."""
    out = np.empty((rows, cols), dtype=np.uint8)
    step = _chunk_rows(cols)
    for r0 in range(0, rows, step):
        r1 = min(rows, r0 + step)
        out[r0:r1] = rng.random((r1 - r0, cols)) < p
    if no_self_loops:
        d = np.arange(min(rows, cols))
        out[d, d] = 0
    return out


def antidist_graph(rng: np.random.Generator, rows: int, cols: int, p: float,
                   wmin: int, wmax: int, width: int, diag_zero: bool = False,
                   keep: tuple[int, int] | None = None) -> np.ndarray:
    """Padded anti-distance adjacency: edge (prob p) -> S - w, w ~ U[wmin, wmax].

    ``keep=(r0, r1)`` returns only rows [r0, r1) (the whole stream is still
    drawn, so the rows equal those of the full matrix) -- a rank's row panel.
    """
    limit = (1 << width) - 1
    dtype = DTYPES[width]
    k0, k1 = keep if keep is not None else (0, rows)
    out = np.zeros((k1 - k0, padded_cols(cols, width)), dtype=dtype)
    step = _chunk_rows(cols)
    for r0 in range(0, rows, step):
        r1 = min(rows, r0 + step)
        mask = rng.random((r1 - r0, cols)) < p
        w = rng.integers(wmin, wmax + 1, size=int(mask.sum()), dtype=np.int64)
        lo, hi = max(r0, k0), min(r1, k1)
        if lo >= hi:
            continue
        block = np.zeros((r1 - r0, cols), dtype=dtype)
        block[mask] = (limit - w).astype(dtype)
        out[lo - k0:hi - k0, :cols] = block[lo - r0:hi - r0]
    if diag_zero:
        d = np.arange(max(k0, 0), min(k1, cols))
        out[d - k0, d] = limit
    return out


@dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration."""
    name: str
    op: str            # "bool_mul" | "bool_closure" | "mul" | "closure"
    n: int             # full size
    oracle_n: int      # size the CPU oracle cross-checks at
    p: float
    width: int = 16
    wmax: int = 1000
    seed: int = 0
    index: int = 0     # position in BASELINE.json configs

    def p_at(self, n: int) -> float:
        # C2's density is "mean out-degree 2": p = 2/n at every size.
        return 2.0 / n if self.name.startswith("c2") else self.p


CONFIGS = {
    "c1_bool_mul": Config("c1_bool_mul", "bool_mul", 1024, 1024, 0.05, seed=101, index=0),
    "c2_bool_warshall": Config("c2_bool_warshall", "bool_closure", 4096, 4096, 2 / 4096,
                               seed=102, index=1),
    "c3_mul_u8": Config("c3_mul_u8", "mul", 4096, 4096, 0.1, width=8, wmax=254,
                        seed=103, index=2),
    "c3_mul_u16": Config("c3_mul_u16", "mul", 4096, 4096, 0.1, width=16, wmax=1000,
                         seed=104, index=2),
    "c4_fw_u16": Config("c4_fw_u16", "closure", 8192, 1024, 0.05, seed=105, index=3),
    "c5_fw_u16": Config("c5_fw_u16", "closure", 32768, 2048, 0.02, seed=106, index=4),
    "c5_mul_u16": Config("c5_mul_u16", "mul", 32768, 2048, 0.02, seed=107, index=4),
}


def make_inputs(cfg: Config, n: int | None = None, rows: tuple[int, int] | None = None):
    """Seeded inputs of ``cfg`` at size n (default: full size).

    Returns a tuple of numpy arrays: (A, B) for products, (T,) for closures.
    Boolean inputs are 0/1 uint8 n x n; lane inputs are n x padded(n) arrays
    in the anti-distance encoding.  ``rows=(r0, r1)`` keeps only that row
    panel of A / T (B stays whole) -- what one rank of a row-panel-sharded
    run owns; the values are identical to the same rows of the full input.
    """
    n = cfg.n if n is None else n
    rng = np.random.default_rng(cfg.seed)
    p = cfg.p_at(n)
    if cfg.op == "bool_mul":
        return bernoulli_bits(rng, n, n, p), bernoulli_bits(rng, n, n, p)
    if cfg.op == "bool_closure":
        return (bernoulli_bits(rng, n, n, p, no_self_loops=True),)
    if cfg.op == "mul":
        a = antidist_graph(rng, n, n, p, 1, cfg.wmax, cfg.width, keep=rows)
        b = antidist_graph(rng, n, n, p, 1, cfg.wmax, cfg.width)
        return a, b
    if cfg.op == "closure":
        return (antidist_graph(rng, n, n, p, 1, cfg.wmax, cfg.width, diag_zero=True, keep=rows),)
    raise ValueError(cfg.op)
