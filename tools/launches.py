"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (per-kernel share)."""
import csv, io, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith('"')]
rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
tot, agg = 0.0, {}
for r in rows:
    t = float(r['Metric Value'].replace(',', '')) / 1e3
    tot += t
    k = r['Kernel Name'].split('(')[0]
    agg.setdefault(k, [0.0, 0])
    agg[k][0] += t
    agg[k][1] += 1
print(f"total {tot:.1f} us over {len(rows)} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:40s} {v[0]:10.1f} us  n={v[1]:3d}  share={v[0] / tot:6.2%}")
