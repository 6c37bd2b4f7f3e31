#!/bin/bash
# round 2 (late): skewed prefix chunks (first 1.5x, last 0.5x) on the current build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c3 8 32 1|c5 8 32 1|c2 8 32 2|c2 8 32 8" base= skew=TAPER_SKEW_CHUNKS=1 skew768=TAPER_SKEW_CHUNKS=1,TAPER_CHUNK_MIN=768 2>&1 | tee gpurun_out/ab_skew.txt
