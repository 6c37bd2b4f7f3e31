#!/bin/bash
# round 2 (late): two slots per merge CTA at h = 1 (two rows per warp)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1200 python -m pytest tests/test_gpu_attention.py tests/test_gpu_gather.py -x -q 2>&1 | tail -3
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c3 8 32 1|c5 8 32 1|c2 8 32 2|c2 8 32 8" ow1= ow0=TAPER_MERGE_ONE_WAITER=0 2>&1 | tee gpurun_out/ab_ow.txt
timeout 300 python scripts/trace_chain.py c2 1 > gpurun_out/trace_chain_ow.txt 2>&1; grep -v Warn gpurun_out/trace_chain_ow.txt
