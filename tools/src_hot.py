"""Per-CUDA-source-line warp-stall samples from `ncu -i X --page source --csv --print-source=cuda,sass`
(numbered rows carry the line totals)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hi]
wi = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
lines = []
for r in rows[hi + 1:]:
    if not r or not r[0].strip().isdigit() or len(r) <= wi:
        continue
    try:
        v = float(r[wi] or 0)
    except ValueError:
        continue
    why = []
    for c in stall_cols:
        try:
            why.append((float(r[c] or 0), h[c][6:]))
        except ValueError:
            pass
    lines.append((v, int(r[0]), r[1].strip()[:80], sorted(why, reverse=True)[:3]))
tot = sum(x[0] for x in lines) or 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for v, ln, s, why in sorted(lines, reverse=True)[:top]:
    rs = ", ".join(f"{k} {100 * x / v:.0f}%" for x, k in why if v)
    print(f"{100 * v / tot:5.1f}% L{ln:4d} {s}   [{rs}]")
