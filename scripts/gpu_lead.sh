#!/bin/bash
# round 2 (late): claim the next item kClaimLead tiles before the current one ends
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c3 8 32 1|c5 8 32 1|c2 8 32 2|c2 8 32 8" base= l4=TAPER_CLAIM_LEAD=4 l8=TAPER_CLAIM_LEAD=8 l12=TAPER_CLAIM_LEAD=12 2>&1 | tee gpurun_out/ab_lead.txt
