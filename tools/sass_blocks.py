"""Basic-block view of an `ncu --page source --csv --print-source sass` dump: runs of SASS
instructions with the same execution count, by share of executed warp instructions.
usage: python tools/sass_blocks.py x_sass.csv [n]"""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))[2:]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
tot = sum(float(r[5]) for r in rows)
smp = sum(float(r[4]) for r in rows)
print('total warp instructions %.4g, samples %.0f' % (tot, smp))
blocks, cur = [], None
for idx, r in enumerate(rows):
    c, s = float(r[5]), float(r[4])
    if cur and cur['c'] == c:
        cur['n'] += 1; cur['s'] += s; cur['end'] = idx
    else:
        cur = {'c': c, 'n': 1, 's': s, 'start': idx, 'end': idx}; blocks.append(cur)
blocks.sort(key=lambda b: -b['c'] * b['n'])
for b in blocks[:n]:
    ops = []
    for i in range(b['start'], b['end'] + 1):
        t = rows[i][1].split()
        ops.append(t[1] if t[0].startswith('@') else t[0])
    print(f"{100*b['c']*b['n']/tot:5.1f}% inst {100*b['s']/smp:5.1f}% stall  count {b['c']:.3g} x {b['n']:4d}  [{b['start']}-{b['end']}]",
          Counter(ops).most_common(6))
