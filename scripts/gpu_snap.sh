#!/bin/bash
# round 2 (late): first snapshot load issued before the prologue barrier
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1500 python -m pytest tests/test_gpu_attention.py tests/test_gpu_reresolve.py tests/test_gpu_step_replay.py -x -q 2>&1 | tail -3
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c2 8 32 8|c3 8 32 1|c2 8 32 2" snap= r2h=@build/libtaper_r2h.so 2>&1 | tee gpurun_out/ab_snap.txt
INTERLEAVE=1 bash scripts/gpu_ab_multi.sh "c2 8 32 1" snap= r2h=@build/libtaper_r2h.so 2>&1 | tee gpurun_out/ab_snap_inter.txt
