# usage: bash tools/prof_k.sh <tag> <kernel-regex> [prof_run args...]
# source-level ncu capture of one kernel launch -> gpurun_out/<tag>_ops.txt, <tag>_metrics.json
tag=$1; k=$2; shift 2
args=${@:-256 3}
ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/$tag python tools/prof_run.py $args > gpurun_out/${tag}_ncu.log 2>&1
ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv 2>/dev/null
python tools/sass_ops.py gpurun_out/${tag}_sass.csv > gpurun_out/${tag}_ops.txt 2>&1
python tools/ncu_summary.py gpurun_out/${tag}_metrics.json k=gpurun_out/$tag.ncu-rep > /dev/null 2>&1
rm -f gpurun_out/$tag.ncu-rep
head -12 gpurun_out/${tag}_ops.txt
