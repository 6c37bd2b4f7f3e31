#!/bin/bash
# round 2 (late): with later claims, re-check finer prefix chunks at small h
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c3 8 32 1|c5 8 32 1|c2 8 32 2" base= m768=TAPER_CHUNK_MIN=768 m512=TAPER_CHUNK_MIN=512 l6=TAPER_CLAIM_LEAD=6 2>&1 | tee gpurun_out/ab_lead2.txt
