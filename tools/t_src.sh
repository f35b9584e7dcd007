ncu --set full --clock-control none --import-source on -k regex:k_jk32 -c 1 -o gpurun_out/jk1 python tools/prof_run.py 64 2 > /dev/null 2>&1
for opt in "cuda" "sass,cuda" "cuda,sass"; do
  echo "== $opt"; ncu -i gpurun_out/jk1.ncu-rep --page source --csv --print-source $opt 2>&1 | head -4 | cut -c1-400
done
ncu -i gpurun_out/jk1.ncu-rep --page source --csv --print-source sass --print-source-line-info 2>&1 | head -3 | cut -c1-400
ncu --help | grep -A3 "print-source" | head -20
