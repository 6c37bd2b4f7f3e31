#!/bin/bash
# c3 probe + bench (taper) of the current build
TAG=${1:-x}
bash scripts/gpu_probe.sh $TAG c3
for c in c3 c2; do
timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 --warmup 3 2>/dev/null | tail -1 | python -c \
  "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['kernel_us']['attend'], d['roofline']['frac'], d['clocks'])"
done
