# bwd/fwd recurrence timing under DS_LSTM_VARIANT experiment switches
mkdir -p gpurun_out
for v in 7 135 263 391; do
  echo "variant $v" >> gpurun_out/variants.txt
  DS_LSTM_VARIANT=$v DS_FWD_UNITS=16 timeout 120 python tools/lstm_trace.py 2>&1 | grep "us per launch" >> gpurun_out/variants.txt
done
