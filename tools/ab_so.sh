#!/bin/bash
# Same-box A/B of two builds of libds.so (run under gpurun from the repo root).
#   old build: abtmp/libds_old.so (e.g. `git stash; make -C paper_1904_04956_b200/csrc;
#   cp paper_1904_04956_b200/libds.so abtmp/libds_old.so; git stash pop; make ...`)
#   usage: bash tools/ab_so.sh ncu <kernel-name>   # per-launch ncu durations (serialised; relative only)
#          bash tools/ab_so.sh bench               # three alternating bench runs per build
MODE=${1:-bench}
cp paper_1904_04956_b200/libds.so /tmp/new.so
use() { if [ $1 = old ]; then cp abtmp/libds_old.so paper_1904_04956_b200/libds.so; else cp /tmp/new.so paper_1904_04956_b200/libds.so; fi; }
if [ $MODE = ncu ]; then
  for v in new old; do
    use $v
    ncu --kernel-name $2 --launch-skip 2 -c 6 --metrics gpu__time_duration.sum --clock-control none --csv \
      python bench.py --steps 2 --warmup 3 > gpurun_out/ab_ncu_$v.csv 2>/dev/null
    echo -n "$v "; grep gpu__time_duration gpurun_out/ab_ncu_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' '; echo
  done
else
  for i in 1 2 3; do for v in new old; do
    use $v
    echo -n "$v "; python bench.py --steps 60 --warmup 5 --no-cpu --no-library 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['value'])"
  done; done
fi
cp /tmp/new.so paper_1904_04956_b200/libds.so
