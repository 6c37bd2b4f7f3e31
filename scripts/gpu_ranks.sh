#!/bin/bash
# per-rank work of a G-GPU KV-head shard on one B200 (bench.py --rank-of G), configs c2 c3 c5
TAG=${1:-rk}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for c in c3 c5 c2; do
  for G in 1 2 4 8; do
    timeout 600 python bench.py --config $c --rank-of $G --no-cpu-baseline --no-e2e --steps 20 --warmup 3 \
      > gpurun_out/rank_${TAG}_${c}_$G.json 2> gpurun_out/rank_${TAG}_${c}_$G.err
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value'],2), round(d['roofline']['frac'],3), round(d['kernel_us']['attend'],1), d['clocks']['sm_mhz'])" gpurun_out/rank_${TAG}_${c}_$G.json
  done
done
