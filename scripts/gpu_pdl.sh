#!/bin/bash
# round 2 (late): PDL / early-claim A/B on C2 rank-of-8 layers, chained and interleaved
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c3 8 32 1" base= ec0=TAPER_EARLY_CLAIM=0 nopdl=TAPER_PDL=0 2>&1 | tee gpurun_out/ab_pdl.txt
export INTERLEAVE=1
bash scripts/gpu_ab_multi.sh "c2 8 32 1" base= ec0=TAPER_EARLY_CLAIM=0 nopdl=TAPER_PDL=0 2>&1 | tee gpurun_out/ab_pdl_inter.txt
