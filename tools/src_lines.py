"""Per-CUDA-source-line aggregates from `ncu -i rep --page source --csv --print-source sass,cuda`:
top lines by warp-stall samples and by executed instructions.  usage: python tools/src_lines.py x.csv [n]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur, data = "", []
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        smp, inst = float(r[4] or 0), float(r[7] or 0)
    except ValueError:
        continue
    data.append((smp, inst, f"{cur}:{r[0]}", r[1].strip()[:100]))
ts = sum(d[0] for d in data) or 1.0
ti = sum(d[1] for d in data) or 1.0
print(f"total samples {ts:.0f}, warp instructions {ti:.4g}")
for smp, inst, loc, src in sorted(data, reverse=True)[:n_top]:
    print(f"{100 * smp / ts:5.1f}% stall {100 * inst / ti:5.1f}% inst {loc:>14} {src}")
