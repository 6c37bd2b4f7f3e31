#!/bin/bash
# round 2 (late): P = hi + lo with a truncated hi (byte permute) -- parity of the variant, then
# same-box A/B at full clock (chained calls) and at the power cap (steady state)
mkdir -p gpurun_out build
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
python -c "from paper_2605_06914_b200 import build as B; B.build(force=True, defines=['TAPER_PHI_TRUNC=1'], out='build/libtaper_trunc.so')" || exit 1
TAPER_LIB=$PWD/build/libtaper_trunc.so timeout 900 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -3
bash scripts/gpu_ab_multi.sh "c2 8 32 8|c3 4 16 8|c2 8 32 1" base= trunc=@build/libtaper_trunc.so 2>&1 | tee gpurun_out/ab_trunc.txt
AB_SCRIPT=steady.py AB_ARGS="c2" timeout 900 python scripts/ab.py base= trunc=@build/libtaper_trunc.so 2>&1 | tail -2 | tee gpurun_out/ab_trunc_steady.txt
AB_SCRIPT=steady.py AB_ARGS="c3" timeout 900 python scripts/ab.py base= trunc=@build/libtaper_trunc.so 2>&1 | tail -2 | tee -a gpurun_out/ab_trunc_steady.txt
