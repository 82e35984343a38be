"""Per-item timeline of the persistent bit Warshall (development aid).

Runs the C2 closure (n = argv[1], default 4096) with smx_bool_persist_trace_arm
and prints, per round: pivot duration, row-panel (RP) / 3a (A3) / 3b (B3) item
spans and waits, and the critical chain pivot -> RP -> A3 -> next pivot.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_1705_08743_b200 import BoolMatrix, _native, engines, workloads  # noqa: E402

lib = _native.lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
if len(sys.argv) > 2:
    lib.smx_bool_persist_trace_arm(None, -int(sys.argv[2]))   # k-split of RP / A3 items
(t,) = workloads.make_inputs(workloads.CONFIGS["c2_bool_warshall"], n)
m = BoolMatrix.from_numpy(t)
lib.smx_set_graphs(0)
cap = 20000
buf = torch.zeros(4 * cap, dtype=torch.int64, device="cuda")
for _ in range(3):
    engines.bool_closure_bits(m)
lib.smx_bool_persist_trace_arm(buf.data_ptr(), cap)
torch.cuda.synchronize()
engines.bool_closure_bits(m)
torch.cuda.synchronize()
lib.smx_bool_persist_trace_arm(None, 0)
b = buf.view(-1, 4).cpu().tolist()
R = n // 256
items = [x for x in b[:cap - R] if x[0]]
piv = b[cap - R:]
t0 = min(min(x[0] for x in items), piv[0][0])
rounds = []
names = {0: "RP", 1: "A3", 2: "B3"}
for r in range(R):
    rec = {"r": r, "pivot_us": (piv[r][2] - piv[r][0]) / 1e3, "pivot_at_us": (piv[r][0] - t0) / 1e3}
    for ty in (0, 1, 2):
        xs = [x for x in items if (x[3] & 0xFFFF) == r and ((x[3] >> 16) & 0xFFFF) == ty]
        if not xs:
            continue
        rec[names[ty]] = {"items": len(xs), "first_ready_us": (min(x[1] for x in xs) - t0) / 1e3,
                          "last_end_us": (max(x[2] for x in xs) - t0) / 1e3,
                          "avg_item_us": sum(x[2] - x[1] for x in xs) / len(xs) / 1e3,
                          "avg_wait_us": sum(x[1] - x[0] for x in xs) / len(xs) / 1e3}
    rounds.append(rec)
end = max(x[2] for x in items)
print(json.dumps({"n": n, "total_us": (end - t0) / 1e3, "rounds": rounds}, indent=1))
