#!/bin/bash
# round 2: GPU parity suite (the sanitizer logs under profiles/r2/ came from an earlier pass)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
# (compute-sanitizer is closed on this pool: runs under it left GPUs needing a reset)
