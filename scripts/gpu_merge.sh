#!/bin/bash
# round 2 (late): merge CTAs occupying SMs the next attend call needs -- launch variants
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c2 8 32 8|c3 8 32 1" base= mpdl0=TAPER_MERGE_PDL=0 mg64=TAPER_MERGE_GRID=64 mg148=TAPER_MERGE_GRID=148 2>&1 | tee gpurun_out/ab_merge.txt
