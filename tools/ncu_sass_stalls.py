"""Summarise an ncu source-page export (--page source --csv --print-source sass):
stall reasons in total and the top SASS lines by stall samples."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kernels = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
for k, hi in enumerate(kernels):
    end = kernels[k + 1] - 1 if k + 1 < len(kernels) else len(rows)
    h = rows[hi]
    data = [r for r in rows[hi + 1:end] if len(r) == len(h)]
    ix = {n: i for i, n in enumerate(h)}
    name = rows[hi - 1][1] if hi > 0 and len(rows[hi - 1]) > 1 else "?"

    def f(r, n):
        try:
            return float(r[ix[n]].replace(",", ""))
        except (KeyError, ValueError):
            return 0.0

    stalls = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
    tot = Counter()
    for r in data:
        for n in stalls:
            tot[n] += f(r, n)
    s = sum(tot.values()) or 1
    print(f"== {name[:100]}")
    print("stall mix:", ", ".join(f"{n[6:]} {100 * v / s:.1f}%" for n, v in tot.most_common(8)))
    data.sort(key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))
    for r in data[:top]:
        mix = sorted(((f(r, n), n[6:]) for n in stalls), reverse=True)[:2]
        print(f"{r[ix['Address']][-5:]} {r[ix['Source']][:60]:60s} samples {int(f(r, 'Warp Stall Sampling (All Samples)')):6d} "
              + " ".join(f"{n}:{int(v)}" for v, n in mix))
