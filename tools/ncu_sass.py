"""Dev helper: per-SASS-instruction stall breakdown from `ncu --page source --csv` (first kernel instance)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = [r for r in rows if "Instructions Executed" in r][0]
ix, iw = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
st = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]


def f(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


data, seen = [], set()
for r in rows:
    if len(r) > ix and r is not h and r[0] not in seen and r[0].startswith("0x"):
        seen.add(r[0])
        data.append(r)
tot = sum(f(r[iw]) for r in data) or 1
agg = {}
for r in data:
    for i in st:
        agg[h[i]] = agg.get(h[i], 0) + f(r[i])
print("stall mix:", {k: round(100 * v / tot, 1) for k, v in sorted(agg.items(), key=lambda t: -t[1]) if v / tot > 0.01})
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for r in sorted(data, key=lambda r: -f(r[iw]))[:n]:
    top = sorted(((h[i][6:], f(r[i])) for i in st), key=lambda t: -t[1])[:2]
    print(f"{f(r[ix]) / 1e6:8.2f}M {100 * f(r[iw]) / tot:5.1f}% {top} | {r[1].strip()[:70]}")
