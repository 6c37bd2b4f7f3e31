#!/bin/bash
# Targeted ncu metrics of one attend_kernel launch per config (c3, c5, reduce; G = 1) and of
# one rank of 8 (c2, c3).  usage (under gpurun): bash scripts/gpu_ncu_configs.sh <tag>
TAG=${1:-x}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpc__cycles_elapsed.avg.per_second
for spec in "c3:" "c5:" "reduce:" "c2:--rank-of 8" "c3:--rank-of 8"; do
  c=${spec%%:*}; extra=${spec#*:}
  name=$c$(echo $extra | tr -d ' -')
  timeout 600 ncu --clock-control none -k regex:attend_kernel -s 8 -c 1 --metrics $M --csv \
    python bench.py --config $c $extra --steps 1 --warmup 3 --layers 4 --no-e2e --no-cpu-baseline \
    > gpurun_out/ncu_cfg_${TAG}_$name.csv 2> /dev/null
  echo "== $name"; grep -E "gpu__time|dram__bytes|lts__|pipe_tensor|sm__throughput|gpc__cycles" gpurun_out/ncu_cfg_${TAG}_$name.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
