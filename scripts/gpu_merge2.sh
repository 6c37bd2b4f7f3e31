#!/bin/bash
# round 2 (late): merge with one warp per (KV head, GQA row) and 8 partials in flight
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c2 8 32 8|c3 8 32 1|c5 8 32 1|c2 8 32 2|c2 8 32 4|c3 4 16 8" new= head=@build/libtaper_head.so 2>&1 | tee gpurun_out/ab_merge2.txt
TAPER_LIB=$PWD/build/libtaper_head.so timeout 300 python scripts/trace_chain.py c2 1 > gpurun_out/trace_chain_head.txt 2>&1
timeout 300 python scripts/trace_chain.py c2 1 > gpurun_out/trace_chain_new.txt 2>&1
grep -v Warn gpurun_out/trace_chain_head.txt gpurun_out/trace_chain_new.txt
