#!/bin/bash
# round 2 (late): L2 prefetch of the first item before the grid dependency -- same-box A/B on
# chained calls (layer_time.py) + bench lines + CTA timeline of one C2 rank-of-8 layer
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c3 8 32 1|c2 8 32 8" pf64= pf0=TAPER_PREFETCH_TILES=0 pf16=TAPER_PREFETCH_TILES=16 2>&1 | tee gpurun_out/ab_pf.txt
for cfg in "c2 8" "c3 8"; do
  set -- $cfg
  timeout 600 python bench.py --config $1 --rank-of $2 --no-cpu-baseline --no-e2e --steps 20 --warmup 3 \
    > gpurun_out/bench_pf_${1}_$2.json 2> gpurun_out/bench_pf_${1}_$2.err
done
timeout 600 python bench.py --no-cpu-baseline --steps 30 --warmup 3 > gpurun_out/bench_pf_c2.json 2> gpurun_out/bench_pf_c2.err
TAPER_EXTRA_DEFINES=TAPER_TRACE_ITEMS=1 timeout 300 python scripts/trace_attend.py c2 1 > gpurun_out/trace_c2_h1.txt 2>&1
head -40 gpurun_out/trace_c2_h1.txt
