# per-CUDA-source-line profile of one kernel: bash tools/prof_src.sh <tag> <kernel-regex> [prof_run args]
tag=$1; k=$2; shift 2; args=${@:-256 3}
ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/$tag python tools/prof_run.py $args > gpurun_out/${tag}_ncu.log 2>&1
ncu -i gpurun_out/$tag.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/${tag}_src.csv 2>/dev/null
rm -f gpurun_out/$tag.ncu-rep
python tools/src_lines.py gpurun_out/${tag}_src.csv ${NLINES:-45} > gpurun_out/${tag}_lines.txt
rm -f gpurun_out/${tag}_src.csv
