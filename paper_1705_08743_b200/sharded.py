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

On GPUs the rounds are pipelined (``run`` -> ``_run_lookahead``): on a
high-priority side stream the owner of block r+1 updates its rows K_{r+1}
with round r's panel, closes pivot r+1, updates its row panel and broadcasts
it, while every rank's main stream applies round r to the rest of its rows.
The serial owner work and the NVLink transfer hide behind the bulk GEMM
instead of stalling all ranks once per block.

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
    """Per-rank FW steps on the GPU through the C ABI (launched on torch's
    current stream, so callers control overlap with torch.cuda.stream)."""

    def __init__(self, width: int, anti: bool, block: int | None = None):
        self.width = width
        self.eb = width // 8
        self.kind = _native.SMX_ANTI if anti else _native.SMX_DIST
        mx = _native.lib().smx_fw_block(self.eb)
        # default 256: row panels stay fine-grained across ranks, and the
        # owner's pivot chain stays short against 1/P of a round's phase 3;
        # callers with >= 4096 rows per rank pass 512 (see block_for)
        self.block = min(block or 256, mx)
        self._cp = None
        # set by ShardedFW for its first two rounds: their operands are the
        # mostly unreachable input graph, so the updates certify them for the
        # 1-instruction shifted encoding (fw.cu, fw_rounds_packed)
        self.certify = False

    @staticmethod
    def block_for(n: int, world: int, width: int) -> int:
        """Pivot block of the sharded closure: 512 (u16) once every rank holds
        >= 4096 rows -- the owner's 512 chain then still hides behind its
        rank's phase 3 -- else 256."""
        return 512 if width == 16 and n // max(world, 1) >= 4096 else 256

    def _at(self, t: torch.Tensor, r: int, c: int) -> int:
        return t.data_ptr() + (r * t.shape[1] + c) * self.eb

    def pivot(self, t: torch.Tensor, r0: int, c0: int, b: int) -> None:
        _native.check(_native.lib().smx_fw_pivot(self._at(t, r0, c0), b, t.shape[1], self.eb,
                                                 self.kind, _native.stream_ptr(t.device)),
                      "smx_fw_pivot")

    def panel_update(self, t: torch.Tensor, r0: int, k0: int, b: int, n: int) -> None:
        """T[K,:] (+)= T[K,K]* (x) T[K,:] in place (no snapshot needed: the
        pivot tile is closed, so every interleaving gives the same result;
        see fw_pivot_and_row_panel in fw.cu)."""
        ld = t.shape[1]
        _native.check(_native.lib().smx_semiring_gemm_skip(
            self._at(t, r0, k0), self._at(t, r0, 0), self._at(t, r0, 0), b, n, b, ld, ld, ld, self.eb,
            self.kind, 0, 0, _native.stream_ptr(t.device)), "pivot row panel")

    def snapshot(self, t: torch.Tensor, k0: int, b: int) -> torch.Tensor:
        """Column panel T[own rows, K] into a (rows x block) buffer."""
        rows = t.shape[0]
        if self._cp is None or self._cp.shape[0] < rows or self._cp.device != t.device:
            self._cp = torch.empty((max(rows, 1), self.block), dtype=t.dtype, device=t.device)
        cp = self._cp[:rows]
        cp[:, :b].copy_(t[:, k0:k0 + b])
        return cp

    def update_rows(self, t: torch.Tensor, cp: torch.Tensor, panel: torch.Tensor, b: int, n: int,
                    lo: int, hi: int, skip: tuple[int, int] | None) -> None:
        """T[lo:hi, :] (+)= CP[lo:hi] (x) panel, skipping local rows `skip`."""
        if hi <= lo:
            return
        s0, sn = (skip[0] - lo, skip[1]) if skip is not None else (0, 0)
        fn = (_native.lib().smx_semiring_gemm_skip_certified if self.certify
              else _native.lib().smx_semiring_gemm_skip)
        _native.check(fn(
            self._at(cp, lo, 0), panel.data_ptr(), self._at(t, lo, 0), hi - lo, n, b, cp.shape[1],
            panel.shape[1], t.shape[1], self.eb, self.kind, s0, sn, _native.stream_ptr(t.device)),
            "row-panel update")

    def rest_update(self, t, panel, k0, b, n, skip) -> None:
        cp = self.snapshot(t, k0, b)
        self.update_rows(t, cp, panel, b, n, 0, t.shape[0], skip)


@dataclass
class ShardedFW:
    """Blocked Floyd-Warshall over ``world`` ranks, rank ``rank`` holding rows
    [row0, row1) of the n x ld matrix in ``local``."""

    n: int
    rank: int
    world: int
    ops: object
    group: object = None
    lookahead: bool = True
    # measurement hook (bench.py's per-rank roofline): when a list, every bulk
    # row update (phase 3b) of the pipelined schedule appends (start event,
    # end event, cell-updates), the events recorded on the main stream
    trace: list | None = None

    def __post_init__(self):
        self.block = self.ops.block
        self.per = rows_per_rank(self.n, self.world, self.block)
        self.row0, self.row1 = row_range(self.n, self.world, self.rank, self.block)
        self._recv = None
        self._side = None

    def owner(self, k0: int) -> int:
        return k0 // self.per

    def _bb(self, k0: int) -> int:
        return min(self.block, self.n - k0)

    def _recv_buf(self, local: torch.Tensor, slot: int) -> torch.Tensor:
        if self._recv is None or self._recv[0].device != local.device:
            self._recv = [torch.empty((self.block, local.shape[1]), dtype=local.dtype,
                                      device=local.device) for _ in range(2)]
        return self._recv[slot]

    # -- simple schedule (also the step API of the single-GPU lockstep test) --

    def begin_round(self, local: torch.Tensor, k0: int):
        """Owner: close the pivot tile and update the pivot row panel.  Returns
        (panel, skip): the owner's panel rows, or this rank's receive buffer."""
        bb = self._bb(k0)
        if self.owner(k0) == self.rank:
            lk = k0 - self.row0
            self.ops.pivot(local, lk, k0, bb)
            self.ops.panel_update(local, lk, k0, bb, self.n)
            return local[lk:lk + bb], (lk, bb)
        return self._recv_buf(local, 0)[:bb], None

    def end_round(self, local: torch.Tensor, panel: torch.Tensor, k0: int, skip) -> None:
        """Every rank: fold the pivot row panel into its own rows."""
        self.ops.rest_update(local, panel, k0, self._bb(k0), self.n, skip)

    def _bcast(self, panel: torch.Tensor, k0: int) -> None:
        # NCCL runs this on its own internal stream, ordered after the current
        # (side) stream; create the process group with
        # ProcessGroupNCCL.Options(is_high_priority_stream=True) (bench.py
        # does) so the panel is not queued behind the bulk GEMM's CTAs
        if self.world > 1:
            dist.broadcast(panel.view(torch.uint8), src=self.owner(k0), group=self.group)

    def run(self, local: torch.Tensor) -> torch.Tensor:
        if self.lookahead and hasattr(self.ops, "update_rows"):
            return self._run_lookahead(local)
        for k0 in range(0, self.n, self.block):
            panel, skip = self.begin_round(local, k0)
            self._bcast(panel, k0)
            self.end_round(local, panel, k0, skip)
        return local

    # -- pipelined schedule ----------------------------------------------------

    def _panel(self, local: torch.Tensor, r: int) -> torch.Tensor:
        k0 = r * self.block
        bb = self._bb(k0)
        if self.owner(k0) == self.rank:
            lk = k0 - self.row0
            return local[lk:lk + bb]
        return self._recv_buf(local, r % 2)[:bb]

    def _owner_work(self, local: torch.Tensor, r: int) -> None:
        k0 = r * self.block
        if self.owner(k0) == self.rank:
            lk, bb = k0 - self.row0, self._bb(k0)
            self.ops.pivot(local, lk, k0, bb)
            self.ops.panel_update(local, lk, k0, bb, self.n)

    def _run_lookahead(self, local: torch.Tensor) -> torch.Tensor:
        import contextlib
        n, B, ops = self.n, self.block, self.ops
        R = -(-n // B)
        rows = local.shape[0]
        if local.is_cuda:
            main = torch.cuda.current_stream(local.device)
            if self._side is None:
                self._side = torch.cuda.Stream(device=local.device, priority=-1)
            side = self._side
        else:   # CPU (tests): the same schedule, serialised in issue order
            main = side = None
        self._owner_work(local, 0)
        self._bcast(self._panel(local, 0), 0)
        for r in range(R):
            k0, bb = r * B, self._bb(r * B)
            if hasattr(ops, "certify"):
                ops.certify = r < 2
            panel = self._panel(local, r)
            cp = ops.snapshot(local, k0, bb)
            own_r = self.owner(k0) == self.rank
            skip_lo, skip_n = (k0 - self.row0, bb) if own_r else (0, 0)
            if r + 1 < R:
                k1, bb1 = k0 + B, self._bb(k0 + B)
                own_n = self.owner(k1) == self.rank
                lk1 = k1 - self.row0
                if own_n:
                    skip_lo, skip_n = (skip_lo, skip_n + bb1) if own_r else (lk1, bb1)
                fork = main.record_event() if main is not None else None
                with torch.cuda.stream(side) if side is not None else contextlib.nullcontext():
                    if side is not None:
                        side.wait_event(fork)
                    if own_n:                      # 3a: next pivot rows, on the side chain
                        ops.update_rows(local, cp, panel, bb, n, lk1, lk1 + bb1, None)
                    self._owner_work(local, r + 1)
                    self._bcast(self._panel(local, r + 1), k1)
                    join = side.record_event() if side is not None else None
                traced = self.trace is not None and main is not None
                if traced:
                    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    ev0.record(main)
                ops.update_rows(local, cp, panel, bb, n, 0, rows,
                                (skip_lo, skip_n) if skip_n else None)   # 3b
                if traced:
                    ev1.record(main)
                    self.trace.append((ev0, ev1, (rows - skip_n) * n * bb))
                if main is not None:
                    main.wait_event(join)
            else:
                ops.update_rows(local, cp, panel, bb, n, 0, rows, (skip_lo, skip_n) if skip_n else None)
        if hasattr(ops, "certify"):
            ops.certify = False
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


class NativeShardedFW:
    """The same pipelined row-panel closure as one C-ABI call per rank
    (smx_fw_sharded, csrc/sharded.cu): the orchestration runs in C++ and the
    broadcast is enqueued on the library's high-priority side stream.

    transport "nccl": smx_nccl_broadcast on the NCCL communicator of the
    default process group (torch's ProcessGroupNCCL, ``_comm_ptr``).
    transport "callback": a Python broadcast over torch.distributed (gloo in
    the tests); the side stream is synchronised before each broadcast, so no
    kernel ever waits on another rank.
    """

    def __init__(self, n: int, rank: int, world: int, width: int = 16, anti: bool = True,
                 block: int | None = None, group=None, transport: str | None = None, bcast_py=None):
        self.n, self.rank, self.world, self.width = n, rank, world, width
        self.eb = width // 8
        self.kind = _native.SMX_ANTI if anti else _native.SMX_DIST
        lib = _native.lib()
        self.block = block or lib.smx_fw_sharded_block(n, world, self.eb)
        self.row0, self.row1 = row_range(n, world, rank, self.block)
        self.group = group
        if transport is None:
            transport = "nccl" if world > 1 and dist.get_backend(group) == "nccl" else "callback"
        self.transport = transport
        # transport "callback" with bcast_py(view, root, stream_ptr): a custom
        # exchange that enqueues on the given stream (tools/emulate_rank.py)
        self.bcast_py = bcast_py
        self._ws = None
        self._cb = None
        self._local = None

    def _nccl_comm(self, device) -> int:
        pg = self.group or dist.distributed_c10d._get_default_group()
        return pg._get_backend(device)._comm_ptr()

    def _callback(self):
        import ctypes

        def bcast(buf, nbytes, root, ctx, stream):
            try:
                if self.bcast_py is None:
                    # stream may be NULL (torch's legacy default stream)
                    if stream:
                        torch.cuda.ExternalStream(stream).synchronize()
                    else:
                        torch.cuda.synchronize()
                view = None
                for base in (self._local, self._ws):
                    lo = base.data_ptr()
                    if lo <= buf and buf + nbytes <= lo + base.numel() * base.element_size():
                        flat = base.view(torch.uint8).reshape(-1)
                        view = flat[buf - lo: buf - lo + nbytes]
                        break
                if view is None:
                    return -5
                if self.bcast_py is not None:
                    self.bcast_py(view, root, stream)
                    return 0
                dist.broadcast(view, src=root, group=self.group)
                torch.cuda.synchronize()
                return 0
            except Exception:   # never let an exception cross the C frame
                import sys
                import traceback
                traceback.print_exc(file=sys.stderr)
                return -5
        self._cb = _native.BCAST_FN(bcast)
        return ctypes.cast(self._cb, ctypes.c_void_p).value, None

    def run(self, local: torch.Tensor) -> torch.Tensor:
        import ctypes
        lib = _native.lib()
        rows, ld = local.shape[0], local.shape[1]
        nbytes = lib.smx_fw_sharded_workspace_bytes(rows, ld, self.eb, self.block)
        if self._ws is None or self._ws.numel() < nbytes or self._ws.device != local.device:
            self._ws = _native.workspace(nbytes, local.device)
        self._local = local
        if self.world == 1:
            fn, ctx = None, None
        elif self.transport == "nccl":
            fn = ctypes.cast(lib.smx_nccl_broadcast, ctypes.c_void_p).value
            ctx = self._nccl_comm(local.device)
        else:
            fn, ctx = self._callback()
        _native.check(lib.smx_fw_sharded(
            local.data_ptr(), self.n, self.row0, rows, ld, self.eb, self.kind, self.rank, self.world,
            self.block, fn, ctx, self._ws.data_ptr(), nbytes, _native.stream_ptr(local.device)),
            "smx_fw_sharded")
        return local
