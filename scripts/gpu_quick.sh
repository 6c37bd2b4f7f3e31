#!/bin/bash
# Quick GPU iteration: build, GPU parity tests, CTA-0 trace of one C2 layer, two bench runs.
# usage (under gpurun): bash scripts/gpu_quick.sh <tag>
TAG=${1:-q}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python scripts/trace_attend.py c2 > gpurun_out/trace_$TAG.txt 2>&1
sed -n 13,25p gpurun_out/trace_$TAG.txt
for i in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c \
    "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernel_us'], d['roofline']['frac'], d['clocks'])"
done
