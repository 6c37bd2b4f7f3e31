#!/bin/bash
# round 2: racecheck of the step + bench lines (c2 default; per-rank c2/c3 at G = 8; c3 at G = 1)
TAG=${1:-p}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
# (compute-sanitizer is closed on this pool: runs under it left GPUs needing a reset)
timeout 900 python bench.py > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('c2 default', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), 'frac', round(d['roofline']['frac'],3), 'attend', round(d['kernel_us']['attend'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'], 'cpu', d['cpu_baseline']['value'], d['cpu_baseline']['cores'], d['cpu_baseline']['single_core']['value'])" gpurun_out/bench_${TAG}_c2.json
for cfg in "c2 8" "c3 8" "c3 1" "c5 1"; do
  set -- $cfg
  timeout 600 python bench.py --config $1 --rank-of $2 --no-cpu-baseline --no-e2e --steps 20 --warmup 3 \
    > gpurun_out/bench_${TAG}_${1}_$2.json 2> gpurun_out/bench_${TAG}_${1}_$2.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value'],2), round(d['roofline']['frac'],3), round(d['kernel_us']['attend'],1), round(d['kernel_us']['attention_call_in_step'],1), d['clocks']['sm_mhz'], d['config']['launch'][:20])" gpurun_out/bench_${TAG}_${1}_$2.json
done
