"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv, sys
f = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
r = list(csv.reader(open(f)))
h = r[1]
rows = [x for x in r[2:] if len(x) == len(h) and x[0].startswith("0x")]
si = h.index('Warp Stall Sampling (All Samples)'); ei = h.index('Instructions Executed')
val = lambda x: int(x[si]) if x[si].isdigit() else 0
tot = sum(val(x) for x in rows)
print('total samples', tot, 'n instr', len(rows))
top = sorted(range(len(rows)), key=lambda i: -val(rows[i]))[:n]
for i in sorted(top):
    x = rows[i]
    print(f"{i:5d} {val(x):7d} {100*val(x)/tot:5.1f}% ex={x[ei]:>10s}  {x[1].strip()[:100]}")
