"""Per-kernel launch count, mean duration and share of an ncu launch list (--csv --log-file)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
iK, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
t = defaultdict(list)
for r in rows[1:]:
    t[r[iK].split("(")[0][:70]].append(float(r[iV].replace(",", "")))
tot = sum(sum(v) for v in t.values())
print(f"{'kernel':70s} {'n':>5s} {'mean us':>9s} {'share':>7s}")
for k, v in sorted(t.items(), key=lambda x: -sum(x[1])):
    print(f"{k:70s} {len(v):5d} {sum(v) / len(v) / 1e3:9.2f} {sum(v) / tot:7.1%}")
