#!/bin/bash
# round 2 (late): cross-item QK lookahead in the MMA warp -- parity, then same-box A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_step_replay.py -x -q 2>&1 | tail -3
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c2 8 32 8|c3 8 32 1|c3 4 16 8|c5 8 32 1|c2 8 32 2" la= nola=TAPER_QK_LOOKAHEAD=0 la512=TAPER_CHUNK_MIN=512 2>&1 | tee gpurun_out/ab_la.txt
