"""Top SASS instructions by warp-stall samples from `ncu -i X --page source --csv --print-source=sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ai, si, wi = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((float(r[wi] or 0), r[ai], r[si], r[ie]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for d in sorted(data, reverse=True)[:top]:
    print(f"{100 * d[0] / tot:5.1f}%  {d[1]}  {d[2][:90]}  (exec {d[3]})")
# cumulative by rough region: print running window sums of 40 consecutive instructions
win = 60
best = []
for i in range(0, len(data), win):
    s = sum(d[0] for d in data[i:i + win])
    best.append((s, data[i][1], data[min(i + win, len(data)) - 1][1]))
print("--- hottest 60-instruction windows")
for s, a, b in sorted(best, reverse=True)[:8]:
    print(f"{100 * s / tot:5.1f}%  {a}..{b}")
