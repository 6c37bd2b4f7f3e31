#!/bin/bash
# ncu --set full (+ SASS source page with stall reasons) of attend_kernel for one config.
# usage (under gpurun): bash scripts/gpu_ncu_cfg.sh <tag> <config> <rank_of G>
TAG=${1:-x}; CFG=${2:-c2}; G=${3:-1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_kernel -s 8 -c 1 \
  -o gpurun_out/prof_${TAG} -f python bench.py --config $CFG --rank-of $G --steps 1 --warmup 3 --layers 4 --no-e2e \
  --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_${TAG}.err
tail -2 gpurun_out/ncu_${TAG}.err
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_${TAG}.csv 2>&1
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}.csv 2>&1
ls -la gpurun_out/prof_${TAG}.ncu-rep
