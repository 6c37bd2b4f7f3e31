#!/bin/bash
# round 2 (late): re-resolve test build + more prefix chunk floors at h <= 2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_reresolve.py -x -q 2>&1 | tail -3
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c3 8 32 1|c2 8 32 2" base= f640=TAPER_CHUNK_MIN=640 f832=TAPER_CHUNK_MIN=832 f896=TAPER_CHUNK_MIN=896 2>&1 | tee gpurun_out/ab_chunk2.txt
