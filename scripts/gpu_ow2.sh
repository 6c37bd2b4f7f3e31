#!/bin/bash
# round 2 (late): merge knobs again on the final build (later claims)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c3 8 32 1|c5 8 32 1|c2 8 32 2" base= ow=TAPER_MERGE_ONE_WAITER=1 rpw2=TAPER_MERGE_MIN_RPW=2 2>&1 | tee gpurun_out/ab_ow2.txt
