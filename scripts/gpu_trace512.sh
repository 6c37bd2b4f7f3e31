#!/bin/bash
# CTA timelines of one C2 rank-of-8 layer: default 1024-token chunk floor vs 512
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
TAPER_EXTRA_DEFINES=TAPER_TRACE_ITEMS=1 timeout 300 python scripts/trace_attend.py c2 1 > gpurun_out/trace_c2_h1_base.txt 2>&1
TAPER_EXTRA_DEFINES=TAPER_TRACE_ITEMS=1,TAPER_CHUNK_MIN=512 timeout 300 python scripts/trace_attend.py c2 1 > gpurun_out/trace_c2_h1_512.txt 2>&1
for f in base 512; do echo "== $f"; grep -E 'per-CTA|CTA end|10 latest|tiles per CTA|first Q landed|first K/V' gpurun_out/trace_c2_h1_$f.txt; sed -n '/per item/,/epilogue per item/p' gpurun_out/trace_c2_h1_$f.txt; done
