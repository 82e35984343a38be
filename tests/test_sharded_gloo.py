"""Multi-rank row-panel-sharded Floyd-Warshall orchestration on the CPU (gloo).

The per-rank compute steps are the pinned CPU oracle (test infrastructure);
what is under test is paper_1705_08743_b200.sharded: row ownership, pivot
owners, the broadcast of each pivot row panel, and the skip ranges -- run as
real world_size-2/3 process groups.  The result must equal the single-process
closure bit for bit (the GPU ops are checked against the same oracle in
tests/test_gpu_parity.py).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1705_08743_b200 import sharded, workloads


class OracleFwOps:
    """CPU stand-in for CudaFwOps with the same contract (test infrastructure)."""

    def __init__(self, width: int, anti: bool, block: int):
        self.width, self.kind, self.block = width, "anti" if anti else "dist", block
        self.fold = np.maximum if anti else np.minimum

    def pivot(self, t, r0, c0, b):
        a = t.numpy()
        tile = np.ascontiguousarray(a[r0:r0 + b, c0:c0 + b])
        a[r0:r0 + b, c0:c0 + b] = oracle.semiring_close(tile, self.width, self.kind)

    def panel_update(self, t, r0, k0, b, n):
        a = t.numpy()
        rp = a[r0:r0 + b].copy()
        prod = oracle.semiring_mul(np.ascontiguousarray(rp[:, k0:k0 + b]), rp, b, self.width, self.kind)
        a[r0:r0 + b, :n] = self.fold(rp[:, :n], prod[:, :n])

    def snapshot(self, t, k0, b):
        return torch.from_numpy(np.ascontiguousarray(t.numpy()[:, k0:k0 + b]))

    def update_rows(self, t, cp, panel, b, n, lo, hi, skip):
        a = t.numpy()
        if hi <= lo:
            return
        prod = oracle.semiring_mul(np.ascontiguousarray(cp.numpy()[lo:hi]), panel.numpy(), b,
                                   self.width, self.kind)
        rows = np.zeros(a.shape[0], dtype=bool)
        rows[lo:hi] = True
        if skip is not None:
            rows[skip[0]:skip[0] + skip[1]] = False
        a[rows, :n] = self.fold(a[rows, :n], prod[rows[lo:hi], :n])

    def rest_update(self, t, panel, k0, b, n, skip):
        self.update_rows(t, self.snapshot(t, k0, b), panel, b, n, 0, t.shape[0], skip)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, width, anti, block, lookahead, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = workloads.CONFIGS["c5_fw_u16"]
        r0, r1 = sharded.row_range(n, world, rank, block)
        (panel,) = workloads.make_inputs(cfg, n, rows=(r0, r1))
        if width != 16:
            lim = (1 << width) - 1
            panel = np.where(panel > 0, lim - (65535 - panel.astype(np.int64)) % 50, 0).astype(
                workloads.DTYPES[width])
            panel = np.pad(panel, ((0, 0), (0, workloads.padded_cols(n, width) - panel.shape[1])))
        if not anti:
            panel = ((1 << width) - 1 - panel.astype(np.int64)).astype(panel.dtype)
        local = torch.from_numpy(np.ascontiguousarray(panel))
        fw = sharded.ShardedFW(n=n, rank=rank, world=world, ops=OracleFwOps(width, anti, block),
                               lookahead=lookahead)
        fw.run(local)
        full = sharded.gather_rows(local, n, world, block)
        if rank == 0:
            q.put(full.numpy().copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,block,width,anti,lookahead", [
    (2, 200, 32, 16, True, True),
    (2, 200, 32, 16, True, False),
    (2, 256, 64, 16, False, True),
    (3, 230, 32, 8, True, True),
    (3, 230, 32, 8, True, False),
    (4, 300, 32, 16, True, True),
])
def test_sharded_fw_matches_single_process(world, n, block, width, anti, lookahead):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, width, anti, block, lookahead, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference: the same generator, the oracle closure
    (full,) = workloads.make_inputs(workloads.CONFIGS["c5_fw_u16"], n)
    if width != 16:
        lim = (1 << width) - 1
        full = np.where(full > 0, lim - (65535 - full.astype(np.int64)) % 50, 0).astype(
            workloads.DTYPES[width])
        full = np.pad(full, ((0, 0), (0, workloads.padded_cols(n, width) - full.shape[1])))
    if not anti:
        full = ((1 << width) - 1 - full.astype(np.int64)).astype(full.dtype)
    want = oracle.semiring_close(np.ascontiguousarray(full), width, "anti" if anti else "dist")
    np.testing.assert_array_equal(got[:, :n], want[:, :n])


def test_row_ranges_cover_and_align():
    for n, world, block in [(32768, 8, 128), (1000, 3, 128), (100, 8, 32)]:
        spans = [sharded.row_range(n, world, r, block) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
            assert a1 == b0
        for a0, _ in spans:
            assert a0 % block == 0 or a0 == n
