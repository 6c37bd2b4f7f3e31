#!/bin/bash
# same-box A/B of build variants over several layer shapes:
#   bash scripts/gpu_ab_multi.sh "c2|c3|c5|c2 8 32 1" NAME=DEFS|@lib ...
SHAPES=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
first=1
IFS='|' read -ra SH <<< "$SHAPES"
for shp in "${SH[@]}"; do
  echo "== $shp"
  if [ $first = 1 ]; then args=("$@"); first=0; else
    args=(); for a in "$@"; do n=${a%%=*}; d=${a#*=}; if [ "${d:0:1}" = "@" ]; then args+=("$a"); else args+=("$n=@/tmp/libtaper_$n.so"); fi; done
    # the working-tree variant (empty defines) was built to /tmp/libtaper_<name>.so too
  fi
  AB_SCRIPT=layer_time.py AB_ARGS="$shp" timeout 1200 python scripts/ab.py "${args[@]}" 2>&1 | tail -${#args[@]}
done
