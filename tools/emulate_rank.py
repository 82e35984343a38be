"""One rank of the row-panel-sharded closure, alone on one GPU (prediction
aid for the multi-GPU run, which this sandbox cannot launch).

Rank 0 of `world` runs ShardedFW's pipelined schedule on its row panel of the
n = 32768 C5 input with the broadcast replaced by a device copy of some of
its own rows into the receive panel (timing only; the result is not checked).  Rank 0 owns the
first R / world pivot blocks, so its run mixes owner rounds (3a + pivot +
row panel on the side stream, beside its phase 3) and plain rounds (phase 3
only).  Timing the same run with the owner work removed gives the plain
round; the owner round follows.  In the real run every round has an owner
whose broadcast the others wait for, so the closure takes about R owner
rounds: the printed prediction.

    python tools/emulate_rank.py [world ...]
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1705_08743_b200 import sharded, workloads  # noqa: E402


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 1e3 / reps


def main():
    cfg = workloads.CONFIGS["c5_fw_u16"]
    n = cfg.n
    for world in [int(x) for x in sys.argv[1:]] or [2, 4, 8]:
        for block in (256, 512):
            ops = sharded.CudaFwOps(16, anti=True, block=block)
            r0, r1 = sharded.row_range(n, world, 0, block)
            (host,) = workloads.make_inputs(cfg, n, rows=(r0, r1))
            src = torch.from_numpy(host).cuda()
            work = torch.empty_like(src)
            fw = sharded.ShardedFW(n=n, rank=0, world=world, ops=ops)
            # stand-in for the broadcast: the receive panel gets rows of this
            # rank's own (partially closed) panel, so the phase-3 operands have
            # the value distribution of the real run (the bounded fast path
            # depends on it); a 32 MiB device copy on the side stream, about
            # what NCCL's NVLink broadcast costs there

            def fake_bcast(panel, k0):
                if panel.data_ptr() < work.data_ptr() or panel.data_ptr() >= work.data_ptr() + work.numel() * 2:
                    panel.copy_(work[(k0 % (r1 - r0)) // block * block:][:panel.shape[0]])
            fw._bcast = fake_bcast
            rounds = -(-n // block)
            own = sum(1 for r in range(rounds) if fw.owner(r * block) == 0)

            def run():
                work.copy_(src)
                fw.run(work)
            t_all = timed(run)
            real_owner_work = fw._owner_work
            fw._owner_work = lambda local, r: None
            real_owner = fw.owner
            fw.owner = lambda k0: -1      # no owner rounds: phase 3 only (no skips)
            t_plain = timed(run)
            fw._owner_work, fw.owner = real_owner_work, real_owner
            t_round_plain = t_plain / rounds
            t_round_owner = (t_all - (rounds - own) * t_round_plain) / own
            pred = rounds * max(t_round_owner, t_round_plain)
            print(json.dumps({"world": world, "block": block, "rows_per_rank": r1 - r0, "rounds": rounds,
                              "owner_rounds": own, "rank_total_ms": t_all * 1e3,
                              "plain_round_ms": t_round_plain * 1e3, "owner_round_ms": t_round_owner * 1e3,
                              "predicted_closure_ms": pred * 1e3,
                              "predicted_cells_per_s": n ** 3 / pred}), flush=True)


if __name__ == "__main__":
    main()
