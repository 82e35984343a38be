"""One rank of the row-panel-sharded closure, alone on one GPU (prediction
aid for the multi-GPU run, which this sandbox cannot launch).

Rank 0 of `world` runs the pipelined schedule on its row panel of the
n = 32768 C5 input with the broadcast replaced by a device copy of some of
its own rows into the receive panel (timing only; the result is not
checked).  Rank 0 owns the first R / world pivot blocks, so its run mixes
owner rounds (3a + pivot + row panel on the side stream, beside its phase 3)
and plain rounds (phase 3 only).  Modes (where the stand-in copy runs):

  python-high     ShardedFW (Python orchestration); the copy on the
                  high-priority side stream
  python-default  ShardedFW; the copy on a separate DEFAULT-priority stream
                  joined by events -- how torch.distributed's broadcast runs
                  on ProcessGroupNCCL's internal stream unless the group is
                  created with is_high_priority_stream
  native          NativeShardedFW (smx_fw_sharded, C++ orchestration); the
                  copy enqueued on the stream the library hands the exchange
                  callback -- its high-priority side stream, as NCCL is there

For the Python modes the same run with the owner work removed gives the
plain round, and the prediction is R x max(owner round, plain round); the
native mode reports the rank's total, to compare with python-high.

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
    default_stream = torch.cuda.Stream(priority=0)
    for world in [int(x) for x in sys.argv[1:]] or [2, 4, 8]:
        block = sharded.CudaFwOps.block_for(n, world, 16)
        r0, r1 = sharded.row_range(n, world, 0, block)
        (host,) = workloads.make_inputs(cfg, n, rows=(r0, r1))
        src = torch.from_numpy(host).cuda()
        work = torch.empty_like(src)
        rounds = -(-n // block)

        def source_rows(k0, count):
            start = (k0 % (r1 - r0)) // block * block
            return work[start:start + count]

        for mode in ("python-high", "python-default", "native"):
            rec = {"world": world, "block": block, "mode": mode, "rows_per_rank": r1 - r0, "rounds": rounds}
            if mode == "native":
                def bcast_py(view, root, stream):
                    if work.data_ptr() <= view.data_ptr() < work.data_ptr() + work.numel() * 2:
                        return                      # the owner's own rows are the source
                    st = torch.cuda.ExternalStream(stream) if stream else torch.cuda.default_stream()
                    with torch.cuda.stream(st):
                        v = view.view(torch.uint16).view(-1, work.shape[1])
                        v.copy_(source_rows(root * 7919 % n, v.shape[0]))
                fw = sharded.NativeShardedFW(n, 0, world, 16, anti=True, block=block, transport="callback",
                                             bcast_py=bcast_py)

                def run():
                    work.copy_(src)
                    fw.run(work)
                t_all = timed(run)
                rec.update({"rank_total_ms": t_all * 1e3, "round_avg_ms": t_all / rounds * 1e3,
                            "predicted_cells_per_s_if_balanced": n ** 3 / t_all})
                print(json.dumps(rec), flush=True)
                continue
            ops = sharded.CudaFwOps(16, anti=True, block=block)
            fw = sharded.ShardedFW(n=n, rank=0, world=world, ops=ops)

            def fake_bcast(panel, k0, mode=mode):
                if work.data_ptr() <= panel.data_ptr() < work.data_ptr() + work.numel() * 2:
                    return                          # the owner's own rows
                if mode == "python-high":
                    panel.copy_(source_rows(k0, panel.shape[0]))
                    return
                cur = torch.cuda.current_stream()
                default_stream.wait_stream(cur)
                with torch.cuda.stream(default_stream):
                    panel.copy_(source_rows(k0, panel.shape[0]))
                cur.wait_stream(default_stream)
            fw._bcast = fake_bcast
            own = sum(1 for r in range(rounds) if fw.owner(r * block) == 0)

            def run():
                work.copy_(src)
                fw.run(work)
            t_all = timed(run)
            real_owner_work, real_owner = fw._owner_work, fw.owner
            fw._owner_work = lambda local, r: None
            fw.owner = lambda k0: -1      # no owner rounds: phase 3 only (no skips)
            t_plain = timed(run)
            fw._owner_work, fw.owner = real_owner_work, real_owner
            t_round_plain = t_plain / rounds
            t_round_owner = (t_all - (rounds - own) * t_round_plain) / own
            pred = rounds * max(t_round_owner, t_round_plain)
            rec.update({"owner_rounds": own, "rank_total_ms": t_all * 1e3,
                        "plain_round_ms": t_round_plain * 1e3, "owner_round_ms": t_round_owner * 1e3,
                        "predicted_closure_ms": pred * 1e3, "predicted_cells_per_s": n ** 3 / pred})
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
