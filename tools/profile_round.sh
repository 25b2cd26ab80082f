#!/bin/bash
# ncu evidence for one round (run under gpurun, one GPU):
#   launch list of 3 bench steps, dram bytes of every GEMM launch of one step,
#   --set full captures of the top kernels.  Summarise here with tools/ncu_summary.py.
TAG=${1:-r1c}
O=gpurun_out
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --n-seq 4096 > $O/${TAG}_launches_bench.log 2>&1
echo "launches rc=$?"
# all kernels of the 4th gradient step of phase_profile: time + dram bytes
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/${TAG}_dram.csv python tools/phase_profile.py > $O/${TAG}_dram.log 2>&1
echo "dram rc=$?"
# 14 gemm_kernel launches per step: 0-5 forward inputs, 6 bottleneck, 7 dW_o+dW_b+dY, 8-13 backward
# layer groups; launch 25 (step 1, #11) = a backward layer group, 15 = a forward input projection
for spec in "lstm_bwd:2" "lstm_fwd2:2" "gemm_kernel:25" "gemm_kernel:15" "ce_stats:1" "ce_grad_dz:1" "sgd_lr:0"; do
  k=${spec%%:*}; sk=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $sk -c 1 \
    -o $O/${TAG}_full_${k}_${sk} -f python bench.py --steps 2 --warmup 3 --no-cpu --n-seq 4096 > $O/${TAG}_full_${k}_${sk}.log 2>&1
  echo "full $k rc=$?"
done
