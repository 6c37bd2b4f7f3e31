#!/bin/bash
# Full GPU pass: build, parity tests, smoke, bench, ncu launch list + one full capture.
# usage (under gpurun): bash scripts/gpu_full.sh [tag] [--quick]
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()" || exit 1
if [ "$2" != "--quick" ]; then
  timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -5 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
# launch list of our kernels (cold-cache, serialised: compare shares, not absolutes)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"admit|attend|merge" \
  -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 \
  --no-e2e --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_launch_$TAG.err
tail -3 gpurun_out/ncu_launch_$TAG.err
# one full capture of the dominant kernel
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_kernel -s 8 -c 1 \
  -o gpurun_out/prof_attend_$TAG -f python bench.py --steps 1 --warmup 3 --layers 4 --no-e2e \
  --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_full_$TAG.err
tail -3 gpurun_out/ncu_full_$TAG.err
ls -la gpurun_out
