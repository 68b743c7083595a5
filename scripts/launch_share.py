"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name:
launches, total µs, share of the listed time."""
import csv, sys, collections
rows = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
r = list(csv.reader(lines))
h = r[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
ui = h.index("Metric Unit")
agg = collections.OrderedDict()
for row in r[1:]:
    if row[mi] != "gpu__time_duration.sum":
        continue
    v = float(row[vi].replace(",", ""))
    u = row[ui]
    us = v / 1e3 if u == "nsecond" else v * 1e3 if u == "msecond" else v if u == "usecond" else v / 1e3
    name = row[ki].split("(")[0][:70]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':72s} {'n':>5s} {'total_us':>10s} {'share':>6s}")
for name, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{name:72s} {n:5d} {us:10.1f} {100*us/tot:5.1f}%")
print(f"{'TOTAL':72s} {sum(a[0] for a in agg.values()):5d} {tot:10.1f}")
