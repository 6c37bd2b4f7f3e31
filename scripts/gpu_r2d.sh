#!/bin/bash
# round 2 (late): snapshot-validated first claim -- full GPU suite, smoke, bench + ncu,
# rank-of-G lines
mkdir -p gpurun_out
bash scripts/gpu_full.sh r2d > gpurun_out/full_r2d.log 2>&1
tail -12 gpurun_out/full_r2d.log | cut -c1-400
# (compute-sanitizer is closed on this pool: runs under it left GPUs needing a reset)
for cfg in "c2 8" "c3 8" "c5 8" "c3 1" "c5 1" "c2 2" "c3 2"; do
  set -- $cfg
  timeout 600 python bench.py --config $1 --rank-of $2 --no-cpu-baseline --no-e2e --steps 20 --warmup 3 \
    > gpurun_out/bench_r2d_${1}_$2.json 2> gpurun_out/bench_r2d_${1}_$2.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value'],2), round(d['roofline']['frac'],3), round(d['kernel_us']['attend'],1), round(d['kernel_us']['attention_call_in_step'],1), d['clocks']['sm_mhz'])" gpurun_out/bench_r2d_${1}_$2.json
done
