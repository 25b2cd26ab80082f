#!/bin/bash
# Round-2 final evidence (ncu), run on the GPU box:  gpurun -- 'bash tools/r2f_profile.sh [tag] [kernel:skip ...]'
# ncu serialises kernels, so the overlapped schedule (gated streams, start waits) cannot run under it:
# every capture profiles the profiling-mode step of tools/phase_profile.py (same kernels, each layer's
# GEMMs on the main stream).  Outputs under gpurun_out/r2f/; summarise here with tools/ncu_summary.py,
# tools/traffic_json.py and tools/kernel_traffic_json.py.
TAG=${1:-r2f}; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
X="--metrics sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__sass_inst_executed_op_utcmma.sum,sm__inst_executed_pipe_tc.sum,sm__cycles_elapsed.max"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $OUT/dram.csv python tools/phase_profile.py > $OUT/dram.log 2>&1
echo "dram rc=$?"
# -s: launches of the kernel to skip (phase_profile: 3 warm-up steps + the measured one; 6 recurrences per step)
SPECS=${@:-lstm_bwd3_kernel:12 lstm_fwd2_kernel:12 lstm_fwd2_kernel:13 ce_grad_dz_kernel:2 ce_stats_kernel:2 gemm_kernel:1}
for spec in $SPECS; do
  K=${spec%%:*}; S=${spec##*:}
  timeout 600 ncu --set full $X --clock-control none --import-source on -k regex:$K -s $S -c 1 -o $OUT/full_${K}_$S -f \
    python tools/phase_profile.py > $OUT/full_${K}_$S.log 2>&1
  echo "full $K $S rc=$?"
done
ls -la $OUT
