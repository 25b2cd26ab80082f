#!/bin/bash
# Round-2 evidence, run on the GPU box:  gpurun -- 'bash tools/r2_profile.sh'
# Outputs under gpurun_out/r2/ (summarised into profiles/ by tools/ncu_summary.py here).
set -x
OUT=gpurun_out/r2
mkdir -p $OUT
X="--metrics sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__sass_inst_executed_op_utcmma.sum,sm__inst_executed_pipe_tc.sum,sm__cycles_elapsed.max"
# 1. launch list of the bench command (per-launch device time, cold cache, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-library > $OUT/launches_bench.log 2>&1
# 2. full captures of the dominant kernels of the step
for K in lstm_bwd_kernel lstm_fwd2_kernel ce_grad_dz_kernel ce_stats_kernel; do
  ncu --set full $X --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o $OUT/full_$K -f \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-library > $OUT/full_$K.log 2>&1
done
# a backward layer group GEMM (dW_ih + 2 dW_hh + dX) and a forward projection
ncu --set full $X --clock-control none --import-source on -k regex:gemm_kernel -s 24 -c 1 -o $OUT/full_gemm_bwd -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-library > $OUT/full_gemm_bwd.log 2>&1
ncu --set full $X --clock-control none --import-source on -k regex:gemm_kernel -s 15 -c 1 -o $OUT/full_gemm_fwd -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-library > $OUT/full_gemm_fwd.log 2>&1
# 3. FP32-parity 3xTF32 GEMM (a layer input projection of the parity step) + parity step timing
python tools/parity_step.py > $OUT/parity_step.json 2> $OUT/parity_step.err
ncu --set full $X --clock-control none -k regex:gemm3_kernel -s 2 -c 1 -o $OUT/full_gemm3 -f \
  python tools/parity_step.py > $OUT/full_gemm3.log 2>&1
# 4. sync kernels: HBM roofline at paper size (two learners on one device)
python tools/sync_bench.py > $OUT/sync_kernels.json 2> $OUT/sync_kernels.err
ncu --set full --clock-control none -k regex:"update_mix|pair_mix|shard_step|sgd_kernel" -c 4 -o $OUT/full_sync -f \
  python tools/sync_bench.py > $OUT/full_sync.log 2>&1
ls -la $OUT
