#!/bin/bash
# round 2 (late): first record published before its validation (poisoned on mismatch)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c2 8 32 8|c3 8 32 1|c5 8 32 1|c2 8 32 2" pub= r2g=@build/libtaper_r2g.so 2>&1 | tee gpurun_out/ab_pub.txt
INTERLEAVE=1 bash scripts/gpu_ab_multi.sh "c2 8 32 1" pub= r2g=@build/libtaper_r2g.so 2>&1 | tee gpurun_out/ab_pub_inter.txt
