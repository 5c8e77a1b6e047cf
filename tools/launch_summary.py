"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel count / total / avg,
optionally skipping the first `skip` launches of our library (setup)."""
import collections
import csv
import sys

path = sys.argv[1]
only = sys.argv[2] if len(sys.argv) > 2 else None
rows = [r for r in csv.reader(open(path)) if r]
hdr = next(i for i, r in enumerate(rows) if r[0] == "ID")
H = rows[hdr]
data = [dict(zip(H, r)) for r in rows[hdr + 1:] if len(r) == len(H)]
agg = collections.OrderedDict()
tot = 0.0
for d in data:
    nm = d["Kernel Name"].split("(")[0].replace("void ", "")
    if only and only not in nm:
        continue
    v = float(d["Metric Value"].replace(",", "")) / 1e3  # us
    a = agg.setdefault(nm, [0, 0.0])
    a[0] += 1
    a[1] += v
    tot += v
print(f"{'kernel':58s} {'launches':>8s} {'total us':>10s} {'avg us':>8s} {'share':>6s}")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:58]:58s} {c:8d} {t:10.1f} {t / c:8.2f} {100 * t / tot:5.1f}%")
print(f"{'TOTAL':58s} {sum(c for c, _ in agg.values()):8d} {tot:10.1f}")
