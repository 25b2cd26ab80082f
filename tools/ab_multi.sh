#!/bin/bash
# Same-box A/B of several environment settings of the bench step (ms per step, alternating, R rounds).
# usage (GPU box): bash tools/ab_multi.sh R "ENV1" "ENV2" ...   (an ENV is "A=1 B=2" or "-" for none)
R=$1; shift
for i in $(seq 1 $R); do
  for e in "$@"; do
    [ "$e" = "-" ] && ee="" || ee="$e"
    v=$(env $ee timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu --no-library 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'])")
    echo "[$e] $v"
  done
done
