"""Summarise an ncu --page source --csv export (SASS): shared-memory wavefronts per tile by
instruction class, and the top warp-stall instructions.  usage: ncu_src_summary.py src.csv tiles"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
tiles = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
agg, stalls = {}, []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]]
    try:
        wf = float(r[ix["L1 Wavefronts Shared"]] or 0)
        ideal = float(r[ix["L1 Wavefronts Shared Ideal"]] or 0)
        ex = float(r[ix["Instructions Executed"]] or 0)
        st = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    stalls.append((st, src[:80]))
    if wf == 0:
        continue
    op = src.split()[1] if src.startswith("@") else src.split()[0]
    if op.startswith("STS") and "RZ" in src:
        op += " (zero)"
    a = agg.setdefault(op, [0.0, 0.0, 0.0])
    a[0] += wf; a[1] += ideal; a[2] += ex
tot = sum(v[0] for v in agg.values())
print("shared wavefronts per tile: %.1f" % (tot / tiles))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print("  %-22s wf %7.1f  ideal %7.1f  instr %6.1f" % (k, v[0] / tiles, v[1] / tiles, v[2] / tiles))
ts = sum(s for s, _ in stalls) or 1.0
print("top warp-stall samples:")
for s, src in sorted(stalls, reverse=True)[:12]:
    print("  %5.1f%%  %s" % (100 * s / ts, src))
