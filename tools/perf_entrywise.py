"""HBM rates of the device entrywise ops, development aid:
lane |, ^ and ~ on C5-size u16 matrices (2 GiB each) and Boolean | on a
32768-vertex bit matrix, against the driver-measured HBM copy bandwidth
(MEASURED_PEAKS.json).  Prints one JSON object."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1705_08743_b200 import _native  # noqa: E402

REPO = Path(__file__).resolve().parent.parent
lib = _native.lib()
peak = None
mp = REPO / "MEASURED_PEAKS.json"
if mp.exists():
    peak = json.loads(mp.read_text()).get("hbm_gbs")


def t_of(fn, it=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 1e3 / it


res = {"hbm_peak_gbs": peak}
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
a = torch.randint(0, 65535, (n, n), dtype=torch.int32, device="cuda").to(torch.uint16)
b = torch.randint(0, 65535, (n, n), dtype=torch.int32, device="cuda").to(torch.uint16)
c = torch.empty_like(a)
st = _native.stream_ptr()
for name, op, nin in (("lane_max_u16", 1, 2), ("lane_absdiff_u16", 2, 2), ("lane_complement_u16", 3, 1)):
    sec = t_of(lambda: _native.check(lib.smx_lane_entrywise(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n - 3, n, 2,
                                                            op, 0, st), name))
    gbs = (nin + 1) * a.numel() * 2 / sec / 1e9
    res[name] = {"n": n, "ms": sec * 1e3, "gbs": gbs, "frac_of_hbm": gbs / peak if peak else None}
del a, b, c
wa = torch.randint(-2**31, 2**31 - 1, (n, n // 32), dtype=torch.int32, device="cuda")
wb = torch.randint(-2**31, 2**31 - 1, (n, n // 32), dtype=torch.int32, device="cuda")
wc = torch.empty_like(wa)
sec = t_of(lambda: _native.check(lib.smx_bits_entrywise(wa.data_ptr(), wb.data_ptr(), wc.data_ptr(), n, n - 5,
                                                        n // 32, 0, st), "bits or"))
gbs = 3 * wa.numel() * 4 / sec / 1e9
res["bits_or"] = {"n": n, "ms": sec * 1e3, "gbs": gbs, "frac_of_hbm": gbs / peak if peak else None}
# the Boolean bridge: bits -> u16 lanes (from_boolmat) and back (to_boolmat)
lanes = torch.empty((n, n), dtype=torch.uint16, device="cuda")
sec = t_of(lambda: _native.check(lib.smx_lanes_from_bits(wa.data_ptr(), n // 32, lanes.data_ptr(), n, n - 5, n, 2,
                                                         st), "from_bits"))
gbs = (wa.numel() * 4 + lanes.numel() * 2) / sec / 1e9
res["bridge_from_bits_u16"] = {"n": n, "ms": sec * 1e3, "gbs": gbs, "frac_of_hbm": gbs / peak if peak else None}
sec = t_of(lambda: _native.check(lib.smx_lanes_to_bits(lanes.data_ptr(), n, wc.data_ptr(), n // 32, n, n - 5, 2,
                                                       st), "to_bits"))
gbs = (wa.numel() * 4 + lanes.numel() * 2) / sec / 1e9
res["bridge_to_bits_u16"] = {"n": n, "ms": sec * 1e3, "gbs": gbs, "frac_of_hbm": gbs / peak if peak else None}
print(json.dumps(res))
