#!/bin/bash
# round 2 (late): prefix chunk floor at h = 1 / 2 (A/B on chained calls)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c3 8 32 1|c5 8 32 1|c2 8 32 2" base= m1536=TAPER_CHUNK_MIN=1536 m2048=TAPER_CHUNK_MIN=2048 2>&1 | tee gpurun_out/ab_chunk.txt
