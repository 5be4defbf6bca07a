"""Per-CUDA-source-line instructions executed and stall samples from
`ncu -i X --page source --csv --print-source=cuda,sass` (dev aid): python tools/src_lines.py src.csv [file-substr] [top] [per]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
per = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
L, fname = [], ""
for i, r in enumerate(rows):
    if r and r[0] == "File Name":
        fname = r[1]
        continue
    if r and r[0] == "Line No":
        h = r
        ie, ws = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
        continue
    if not r or not r[0].strip().isdigit() or want not in fname:
        continue
    try:
        L.append((float(r[ie] or 0), float(r[ws] or 0), int(r[0]), fname.split("/")[-1], r[1].strip()[:70]))
    except (ValueError, IndexError, NameError):
        pass
ti, tw = sum(x[0] for x in L) or 1, sum(x[1] for x in L) or 1
print(f"instructions {ti:.0f} ({ti / per:.0f} per unit), stall samples {tw:.0f}")
for x in sorted(L, key=lambda x: -x[1])[:top]:
    print(f"{x[0] / per:9.0f} inst {100 * x[0] / ti:5.1f}%  {100 * x[1] / tw:5.1f}% stall  {x[3]}:{x[2]} {x[4]}")
