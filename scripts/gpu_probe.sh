#!/bin/bash
# usage (under gpurun): bash scripts/gpu_probe.sh <tag> <config> [extra bench args]
# admission parity tests + targeted ncu metrics of one attend_kernel launch of <config>.
TAG=${1:-p}; CFG=${2:-c3}; shift 2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_admit.py -q 2>&1 | tail -3
timeout 600 ncu --clock-control none -k regex:attend_kernel -s 8 -c 1 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum \
  --csv python bench.py --config $CFG --steps 1 --warmup 3 --layers 4 --no-e2e --no-cpu-baseline "$@" \
  > gpurun_out/ncu_probe_$TAG.csv 2> gpurun_out/ncu_probe_$TAG.err
tail -2 gpurun_out/ncu_probe_$TAG.err
grep -E "gpu__time|dram__bytes|lts__|pipe_tensor|sm__throughput|inst_executed" gpurun_out/ncu_probe_$TAG.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
