"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections, csv, sys

SCALE = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
         "s": 1.0, "second": 1.0}


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi or r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        t = float(r[vi].replace(",", "")) * SCALE[r[ui]]
        name = r[ki].split("(")[0][:90]
        agg[name][0] += 1
        agg[name][1] += t
    tot = sum(x[1] for x in agg.values())
    out = [f"== {path}: {sum(x[0] for x in agg.values())} launches, {tot * 1e3:.3f} ms total"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"  {c:6d} launches {t * 1e3:10.3f} ms {100 * t / tot:6.2f}%  avg {t / c * 1e6:9.1f} us  {k}")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarise(p))
