#!/bin/bash
# round 2 (late): double-buffered P^T for wide swap items (odd tiles in the Q buffer's upper half)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_step_replay.py tests/test_gpu_reresolve.py -x -q 2>&1 | tail -3
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c2 8 32 8|c5 8 32 1|c2 8 32 2" pt2= pt1=TAPER_WIDE_PT2=0 2>&1 | tee gpurun_out/ab_pt2.txt
AB_SCRIPT=steady.py AB_ARGS="c2" timeout 900 python scripts/ab.py pt2= pt1=TAPER_WIDE_PT2=0 2>&1 | tail -2 | tee gpurun_out/ab_pt2_steady.txt
