"""Per-opcode warp-instruction and stall-sample totals from `ncu -i rep --page source --csv --print-source sass`.
usage: python tools/sass_ops.py x.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "Address")
ii, si, ti = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Thread Instructions Executed")
agg, tot, tots = {}, 0, 0
for r in rows:
    if len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    op = r[1].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    o = o.split(".")[0]
    n, s, t = float(r[ii] or 0), float(r[si] or 0), float(r[ti] or 0)
    a = agg.setdefault(o, [0, 0, 0])
    a[0] += n; a[1] += s; a[2] += t
    tot += n; tots += s
print(f"total warp instructions {tot:.4g}, samples {tots:.0f}")
for o, (n, s, t) in sorted(agg.items(), key=lambda x: -x[1][0])[:30]:
    print(f"{o:10s} {n:12.4g} {100*n/tot:5.1f}%  samples {100*s/max(tots,1):5.1f}%  lanes/inst {t/max(n,1):5.1f}")
