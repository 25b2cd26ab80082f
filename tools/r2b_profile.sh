#!/bin/bash
# Round-2 (second half) evidence, run on the GPU box:  gpurun -- 'bash tools/r2b_profile.sh'
# ncu serialises kernels, so the overlapped schedule (gated streams, start waits) cannot run under it:
# every capture profiles the profiling-mode step of tools/phase_profile.py (same kernels, each layer's
# GEMMs on the main stream).  Outputs under gpurun_out/r2b/ (summarised into profiles/ here).
OUT=gpurun_out/r2b
mkdir -p $OUT
X="--metrics sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__sass_inst_executed_op_utcmma.sum,sm__inst_executed_pipe_tc.sum,sm__cycles_elapsed.max"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $OUT/launches.csv \
  python tools/phase_profile.py > $OUT/launches.log 2>&1
echo "launches rc=$?"
for K in lstm_bwd3_kernel lstm_fwd2_kernel ce_grad_dz_kernel ce_stats_kernel; do
  timeout 600 ncu --set full $X --clock-control none --import-source on -k regex:$K -s $([ ${K#ce} != $K ] && echo 2 || echo 12) -c 1 -o $OUT/full_$K -f \
    python tools/phase_profile.py > $OUT/full_$K.log 2>&1
  echo "full $K rc=$?"
done
# a forward layer-input projection (gemm launch 2 of the third step: 21 gemm launches per step)
timeout 600 ncu --set full $X --clock-control none --import-source on -k regex:gemm_kernel -s 46 -c 1 -o $OUT/full_gemm_a -f \
  python tools/phase_profile.py > $OUT/full_gemm_a.log 2>&1
echo "full gemm rc=$?"
ls -la $OUT
