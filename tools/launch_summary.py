"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: time share per kernel."""
import collections
import csv
import sys


def summary(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    out = [f"total kernels {sum(a[0] for a in agg.values())}  total {tot / 1e6:.3f} ms (serialised, cold)"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{k[:58]:58s} {c:7d} {t / 1e6:9.3f} ms {100 * t / tot:5.1f}%  avg {t / c / 1e3:8.2f} us")
    return "\n".join(out)


if __name__ == "__main__":
    print(summary(sys.argv[1]))
