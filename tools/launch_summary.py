"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel totals."""
import collections
import csv
import sys


def summarize(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
    agg = collections.OrderedDict()
    tot = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        name = name.replace("rl::<unnamed>::", "")[:70]
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
        tot += v
    lines = [f"{'ms':>10} {'share':>6} {'count':>6}  kernel"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        lines.append(f"{t:10.3f} {100 * t / tot:5.1f}% {c:6d}  {k}")
    lines.append(f"{tot:10.3f} total ms ({sum(c for c, _ in agg.values())} launches)")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
