#!/bin/bash
# full GPU pass of a build: suite, smoke, bench + ncu (scripts/gpu_full.sh), per-config ncu,
# rank-of-G and per-config bench lines.  usage (under gpurun): bash scripts/gpu_final.sh TAG
TAG=${1:-final}
mkdir -p gpurun_out
bash scripts/gpu_full.sh $TAG > gpurun_out/full_$TAG.log 2>&1
head -8 gpurun_out/full_$TAG.log | cut -c1-300
bash scripts/gpu_ncu_configs.sh $TAG > gpurun_out/ncu_cfg_$TAG.log 2>&1
for cfg in "c2 8" "c3 8" "c5 8" "c2 2" "c3 2" "c3 1" "c5 1" "reduce 1"; do
  set -- $cfg
  timeout 600 python bench.py --config $1 --rank-of $2 --no-cpu-baseline --no-e2e --steps 20 --warmup 3 \
    > gpurun_out/bench_${TAG}_${1}_$2.json 2> gpurun_out/bench_${TAG}_${1}_$2.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value'],2), round(d['roofline']['frac'],3), round(d['kernel_us']['attend'],1), round(d['kernel_us']['attention_call_in_step'],1), d['clocks']['sm_mhz'])" gpurun_out/bench_${TAG}_${1}_$2.json
done
