#!/bin/bash
# usage: scripts/gpu_round.sh  -- experiment driver run on the GPU box
set -x
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -m pytest tests/test_gpu_admit.py -x -q 2>&1 | tail -5
for v in default fp16 split; do
  if [ $v = default ]; then export TAPER_LIB=$PWD/paper_2605_06914_b200/libtaper.so; else export TAPER_LIB=$PWD/build/libtaper_$v.so; fi
  echo "=== variant $v"
  timeout 600 python -m pytest tests/test_gpu_attention.py -q 2>&1 | grep -E "passed|failed|Error:" | tail -8
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; tail -3 gpurun_out/bench_$v.err; cat gpurun_out/bench_$v.json
done
