"""Aggregate ncu 'cuda,sass' source CSV to per-source-line stall samples and instructions.
usage: ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, out, tot, toti = None, [], 0.0, 0.0
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r[0] in ('Function Name', 'Line No') or len(r) < 8:
        continue
    if r[0] and r[2] == '-':
        s, ins = float(r[4] or 0), float(r[7] or 0)
        out.append((s, ins, f"{fname}:{r[0]}", r[1]))
        tot += s; toti += ins
print(f"total samples {tot:.0f}  instructions {toti:.3g}")
for s, ins, loc, src in sorted(out, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% {100*ins/toti:5.1f}%i {loc:16s} {src[:100]}")
