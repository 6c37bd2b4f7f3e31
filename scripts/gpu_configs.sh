#!/bin/bash
# Parity tests + bench lines of every single-GPU config (c2 default, c3, c5; taper and eager).
# usage (under gpurun): bash scripts/gpu_configs.sh <tag>
TAG=${1:-cfg}
mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
for c in c2 c3 c5; do
  for p in taper eager; do
    timeout 600 python bench.py --config $c --policy $p --no-cpu-baseline --steps 20 --warmup 3 \
      > gpurun_out/bench_${TAG}_${c}_${p}.json 2> gpurun_out/bench_${TAG}_${c}_${p}.err
    tail -2 gpurun_out/bench_${TAG}_${c}_${p}.err
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['value'], d.get('attn_frac_of_measured_hbm'), d['roofline']['frac'], d['kernel_us']['attend'], d['clocks'], d['config'].get('admitted_slots'))" gpurun_out/bench_${TAG}_${c}_${p}.json
  done
done
