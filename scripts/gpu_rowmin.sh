#!/bin/bash
# round 2 (late): row mode from 5 ready slots (M = 64 row items) at small h
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c2 8 32 2|c5 8 32 1|c2 8 32 4" base= rm5=TAPER_ROW_MIN=5 rm7=TAPER_ROW_MIN=7 2>&1 | tee gpurun_out/ab_rowmin.txt
