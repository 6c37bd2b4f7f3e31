#!/bin/bash
# One `ncu --set full` capture of attend_kernel (one C2 layer) + SASS source page.
# usage (under gpurun): bash scripts/gpu_ncu_attend.sh <tag>
TAG=${1:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_kernel -s 8 -c 1 \
  -o gpurun_out/prof_attend_$TAG -f python bench.py --steps 1 --warmup 3 --layers 4 --no-e2e \
  --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_full_$TAG.err
tail -2 gpurun_out/ncu_full_$TAG.err
ncu -i gpurun_out/prof_attend_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_$TAG.csv 2>&1
ls -la gpurun_out/prof_attend_$TAG.ncu-rep gpurun_out/sass_$TAG.csv
