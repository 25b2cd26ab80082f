#!/bin/bash
# One GPU round trip: gpu tests, smoke, bench, ncu launch list, ncu --set full of the top kernels.
# usage (from the repo root, under gpurun):  bash tools/gpu_round.sh [tag] [what...]
TAG=${1:-r1}; shift
WHAT=${@:-tests smoke bench launches full}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/${TAG}_smi.txt 2>&1
for w in $WHAT; do
case $w in
tests)  timeout 1200 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" ;;
smoke)  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" ;;
bench)  timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"; cat $O/${TAG}_bench.json ;;
ref)    timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/${TAG}_bench_ref.json 2>&1; echo "ref rc=$?"; cat $O/${TAG}_bench_ref.json ;;
launches) # ncu serialises launches: the bench's gated side streams would wait on kernels that cannot run
          # beside them, so the launch list comes from the profiling-mode step (same kernels, GEMMs in order)
          timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
          --log-file $O/${TAG}_launches.csv python tools/phase_profile.py \
          > $O/${TAG}_launches_bench.log 2>&1; echo "launches rc=$?" ;;
full)   for k in lstm_bwd lstm_fwd gemm_kernel sgd_kernel; do
          timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 2 \
            -o $O/${TAG}_prof_$k -f python tools/phase_profile.py > $O/${TAG}_prof_$k.log 2>&1; echo "ncu $k rc=$?"
        done ;;
esac
done
