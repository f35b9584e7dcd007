# per-class ERI kernel times (ncu launch list) for the current build and variants: bash tools/eri_cls.sh v1 v2 ...
for x in cur "$@"; do
  if [ $x = cur ]; then L=""; else L="QM1B_B200_DEV_LIB=build_ab/$x.so"; fi
  env $L ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,dram__bytes_write.sum --clock-control none -k regex:k_eri --csv python tools/prof_run.py 256 1 2>/dev/null > gpurun_out/eri_cls_$x.csv
  echo "== $x"; python - gpurun_out/eri_cls_$x.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
d = {}
for r in rows[1:]:
    d.setdefault(r[ki][:48], {})[r[mi].split("__")[1][:22]] = (r[vi], r[ui])
for k, v in d.items(): print(k, {a: b[0] + b[1] for a, b in v.items()})
PY
done
