#!/bin/bash
# same-box A/B of build variants on one config: bash scripts/gpu_ab.sh <config> NAME=DEFS ...
CFG=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
AB_SCRIPT=layer_time.py AB_ARGS="$CFG" timeout 1500 python scripts/ab.py "$@" 2>&1 | tail -12
