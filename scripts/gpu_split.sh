#!/bin/bash
# round 2 (late): tail splits of dynamically claimed items
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c3 8 32 1|c5 8 32 1|c2 8 32 2|c2 8 32 8" split= nosplit=TAPER_TAIL_SPLIT=0 r2h=@build/libtaper_r2h.so 2>&1 | tee gpurun_out/ab_split.txt
TAPER_EXTRA_DEFINES=TAPER_TRACE_ITEMS=1 timeout 300 python scripts/trace_attend.py c2 1 > gpurun_out/trace_c2_h1_split.txt 2>&1; grep -E "per-CTA|10 latest|tiles per" gpurun_out/trace_c2_h1_split.txt
