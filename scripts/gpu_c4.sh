#!/bin/bash
# final build: c4 trace replay per policy (per-regime steps/s)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for pol in taper eager off; do
  timeout 900 python bench.py --config c4 --policy $pol --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_$pol.json 2> gpurun_out/bench_c4_$pol.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value'],2), {k: round(v['steps_per_s'],1) for k, v in d['regimes'].items()})" gpurun_out/bench_c4_$pol.json
done
