#!/bin/bash
# round 2 (late): balanced schedule + snapshot-validated first claim -- parity tests, then
# same-box A/B (AUTO = balanced at h <= 4 vs dynamic everywhere) and bench lines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_admit.py tests/test_gpu_step_replay.py -x -q 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
bash scripts/gpu_ab_multi.sh "c2 8 32 1|c3 8 32 1|c5 8 32 1|c2 8 32 2|c2 8 32 4|c2 8 32 8" bal= dyn=TAPER_AUTO_BALANCED_MAX_H=0 2>&1 | tee gpurun_out/ab_bal.txt
for cfg in "c2 8" "c3 8" "c5 8"; do
  set -- $cfg
  timeout 600 python bench.py --config $1 --rank-of $2 --no-cpu-baseline --no-e2e --steps 20 --warmup 3 \
    > gpurun_out/bench_bal_${1}_$2.json 2> gpurun_out/bench_bal_${1}_$2.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value'],2), round(d['roofline']['frac'],3), round(d['kernel_us']['attend'],1), round(d['kernel_us']['attention_call_in_step'],1), d['clocks']['sm_mhz'])" gpurun_out/bench_bal_${1}_$2.json
done
