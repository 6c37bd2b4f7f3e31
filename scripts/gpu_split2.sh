#!/bin/bash
# round 2 (late): tail splits again, now with later claims (lead 8)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_attention.py -x -q -k "full_size_one_rank or kv_head or row_mode or multi_chunk" 2>&1 | tail -3
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c3 8 32 1|c5 8 32 1|c2 8 32 2|c2 8 32 8" split= nosplit=TAPER_TAIL_SPLIT=0 2>&1 | tee gpurun_out/ab_split2.txt
