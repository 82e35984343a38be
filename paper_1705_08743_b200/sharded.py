"""Row-panel-sharded Floyd-Warshall and semiring product across GPUs.

One process per GPU (torch.distributed, NCCL over NVLink / NVSwitch).  Rank p
owns a contiguous panel of rows, a whole number of pivot blocks, so every
pivot block has exactly one owner.  Per pivot block K:

  owner : 1. close the pivot tile T[K,K]            (smx_fw_pivot)
          2. T[K,:] (+)= T[K,K]* (x) T[K,:]         (semiring GEMM, snapshot)
  all   : 3. broadcast the pivot row panel T[K,:]   (ncclBroadcast, b x n lanes)
          4. T[own,:] (+)= T[own,K] (x) T[K,:]       (semiring GEMM over the own
             rows, skipping the pivot rows on the owner; the j in K part is
             the column-panel update, so phases 2b and 3 are one GEMM)

This is the only data exchange of the closure; the product needs none (A is
row-sharded, B replicated) and runs as independent local GEMMs.  Both are
bit-identical to the single-GPU closure because every closure order agrees
(fw.cu header).

The per-rank compute steps are an injectable ``ops`` object: ``CudaFwOps``
calls libsemimat_b200.so; the CPU tests inject an oracle-backed version to
exercise this orchestration (owners, broadcasts, skip ranges) with gloo.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _native


def rows_per_rank(n: int, world: int, block: int) -> int:
    per = -(-n // world)
    return -(-per // block) * block


def row_range(n: int, world: int, rank: int, block: int) -> tuple[int, int]:
    per = rows_per_rank(n, world, block)
    return min(n, rank * per), min(n, (rank + 1) * per)


class CudaFwOps:
    """Per-rank FW steps on the GPU through the C ABI."""

    def __init__(self, width: int, anti: bool):
        self.width = width
        self.eb = width // 8
        self.kind = _native.SMX_ANTI if anti else _native.SMX_DIST
        self.block = _native.lib().smx_fw_block(self.eb)
        self._cp = None

    def _at(self, t: torch.Tensor, r: int, c: int) -> int:
        return t.data_ptr() + (r * t.shape[1] + c) * self.eb

    def pivot(self, t: torch.Tensor, r0: int, c0: int, b: int) -> None:
        _native.check(_native.lib().smx_fw_pivot(self._at(t, r0, c0), b, t.shape[1], self.eb,
                                                 self.kind, _native.stream_ptr(t.device)),
                      "smx_fw_pivot")

    def panel_update(self, t: torch.Tensor, r0: int, k0: int, b: int, n: int) -> None:
        rp = t[r0:r0 + b].clone()
        ld = t.shape[1]
        _native.check(_native.lib().smx_semiring_gemm_skip(
            self._at(rp, 0, k0), rp.data_ptr(), self._at(t, r0, 0), b, n, b, ld, ld, ld, self.eb,
            self.kind, 0, 0, _native.stream_ptr(t.device)), "pivot row panel")

    def rest_update(self, t: torch.Tensor, panel: torch.Tensor, k0: int, b: int, n: int,
                    skip: tuple[int, int] | None) -> None:
        rows = t.shape[0]
        if rows == 0:
            return
        if self._cp is None or self._cp.shape[0] < rows or self._cp.device != t.device:
            self._cp = torch.empty((rows, self.block), dtype=t.dtype, device=t.device)
        cp = self._cp[:rows]
        cp[:, :b].copy_(t[:, k0:k0 + b])
        s0, sn = skip if skip is not None else (0, 0)
        _native.check(_native.lib().smx_semiring_gemm_skip(
            cp.data_ptr(), panel.data_ptr(), t.data_ptr(), rows, n, b, cp.shape[1], panel.shape[1],
            t.shape[1], self.eb, self.kind, s0, sn, _native.stream_ptr(t.device)),
            "row-panel update")


@dataclass
class ShardedFW:
    """Blocked Floyd-Warshall over ``world`` ranks, rank ``rank`` holding rows
    [row0, row1) of the n x ld matrix in ``local``."""

    n: int
    rank: int
    world: int
    ops: object
    group: object = None

    def __post_init__(self):
        self.block = self.ops.block
        self.per = rows_per_rank(self.n, self.world, self.block)
        self.row0, self.row1 = row_range(self.n, self.world, self.rank, self.block)

    def owner(self, k0: int) -> int:
        return k0 // self.per

    def begin_round(self, local: torch.Tensor, k0: int):
        """Owner: close the pivot tile and update the pivot row panel.  Returns
        (panel, skip): the owner's panel rows, or this rank's receive buffer."""
        bb = min(self.block, self.n - k0)
        if self.owner(k0) == self.rank:
            lk = k0 - self.row0
            self.ops.pivot(local, lk, k0, bb)
            self.ops.panel_update(local, lk, k0, bb, self.n)
            return local[lk:lk + bb], (lk, bb)
        if getattr(self, "_recv", None) is None or self._recv.device != local.device:
            self._recv = torch.empty((self.block, local.shape[1]), dtype=local.dtype,
                                     device=local.device)
        return self._recv[:bb], None

    def end_round(self, local: torch.Tensor, panel: torch.Tensor, k0: int, skip) -> None:
        """Every rank: fold the pivot row panel into its own rows."""
        bb = min(self.block, self.n - k0)
        self.ops.rest_update(local, panel, k0, bb, self.n, skip)

    def run(self, local: torch.Tensor) -> torch.Tensor:
        for k0 in range(0, self.n, self.block):
            panel, skip = self.begin_round(local, k0)
            if self.world > 1:
                dist.broadcast(panel.view(torch.uint8), src=self.owner(k0), group=self.group)
            self.end_round(local, panel, k0, skip)
        return local


def sharded_mul(a_rows: torch.Tensor, b: torch.Tensor, inner: int, width: int, anti: bool,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """Row-panel-sharded product: this rank's rows of A (x) the replicated B.
    No collective: each rank's output rows depend only on its own A rows."""
    from . import engines
    return engines.lane_mul(a_rows, b, inner, width, anti, out)


def gather_rows(local: torch.Tensor, n: int, world: int, block: int, group=None) -> torch.Tensor:
    """All-gather the row panels into the full matrix (for verification)."""
    per = rows_per_rank(n, world, block)
    padded = torch.zeros((per, local.shape[1]), dtype=local.dtype, device=local.device)
    padded[: local.shape[0]] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather([p.view(torch.uint8) for p in parts], padded.view(torch.uint8), group=group)
    return torch.cat(parts)[:n]
