#!/bin/bash
# round-2 start: fresh-box baseline of the current build (parity suite + per-config timings)
mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for cfg in "c2 1" "c2 8" "c3 1" "c3 8" "c5 8"; do
  set -- $cfg
  timeout 600 python bench.py --config $1 --rank-of $2 --no-cpu-baseline --no-e2e --steps 20 --warmup 3 \
    > gpurun_out/base_${1}_$2.json 2> gpurun_out/base_${1}_$2.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value'],2), round(d['roofline']['frac'],3), round(d['kernel_us']['attend'],1), d['clocks']['sm_mhz'])" gpurun_out/base_${1}_$2.json
done
for cfg in "c2 8" "c3 8" "c3 1"; do
  set -- $cfg
  timeout 300 python scripts/layer_time.py $1 8 32 $((8 / $2))
done
