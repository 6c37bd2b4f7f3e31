#!/bin/bash
# round 2: GPU parity suite + compute-sanitizer on c1 / c2 (logs under gpurun_out/sanitizer_*)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for tool in memcheck racecheck synccheck; do
  for cfg in c1 c2; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_step.py $cfg \
      > gpurun_out/sanitizer_${tool}_${cfg}.log 2>&1
    echo "$tool $cfg rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_step' gpurun_out/sanitizer_${tool}_${cfg}.log | tr '\n' ' ')"
  done
done
