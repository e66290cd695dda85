"""Summarise an ncu source-page CSV (--page source --csv --print-source sass):
total stall samples by reason, and the hottest instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
col = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {r: 0 for r in reasons}
samples = []
for row in data:
    if len(row) < len(hdr):
        continue
    try:
        s = int(row[col["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    samples.append((s, row[col["Address"]], row[col["Source"]]))
    for r in reasons:
        try:
            tot[r] += int(row[col[r]] or 0)
        except ValueError:
            pass
S = sum(tot.values()) or 1
print("stall reasons (share of samples):")
for r, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {r:28s} {100 * v / S:5.1f}%")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print(f"hottest {n} instructions:")
for s, a, src in sorted(samples, reverse=True)[:n]:
    print(f"  {s:6d} {a[-5:]} {src.strip()[:90]}")
