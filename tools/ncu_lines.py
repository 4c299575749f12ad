"""Summarise an ncu --page source --print-source cuda,sass CSV per CUDA source line (dev helper)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
def f(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


hdr = next(r for r in rows if r and r[0] == "Line No")
iw = hdr.index("Warp Stall Sampling (All Samples)")
ix = hdr.index("Instructions Executed")
lines = []
for r in rows:
    if len(r) > ix and r[0] not in ("", "Line No") and r[0].isdigit():
        lines.append((int(r[0]), r[1], f(r[iw]), f(r[ix])))
tw = sum(l[2] for l in lines) or 1
ti = sum(l[3] for l in lines) or 1
print(f"total inst {ti:.3g}  samples {tw:.0f}")
for ln, src, w, i in sorted(lines, key=lambda l: -l[2])[: int(sys.argv[2]) if len(sys.argv) > 2 else 35]:
    print(f"{ln:5d} stall {100*w/tw:5.1f}%  inst {100*i/ti:5.1f}% | {src.strip()[:100]}")
