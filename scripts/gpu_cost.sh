#!/bin/bash
# round 2 (late): claim-order cost model (admit's LPT keys) -- order only, outputs unchanged
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c3 8 32 1|c2 8 32 8|c2 8 32 2" base= c0_16=TAPER_ITEM_COST0=16 wide4=TAPER_WIDE_COST=4 wide2=TAPER_WIDE_COST=2 2>&1 | tee gpurun_out/ab_cost.txt
