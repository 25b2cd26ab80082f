mkdir -p gpurun_out; rm -f gpurun_out/variants.txt
for v in 7; do
  echo "variant $v" >> gpurun_out/variants.txt
  DS_LSTM_VARIANT=$v timeout 120 python tools/lstm_trace.py 2>&1 | grep "us per launch" >> gpurun_out/variants.txt
done
