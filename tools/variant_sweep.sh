mkdir -p gpurun_out; rm -f gpurun_out/variants.txt
for v in 0 50 200 500; do
  echo "nap $v" >> gpurun_out/variants.txt
  DS_NAP=$v timeout 120 python tools/lstm_trace.py 2>&1 | grep "us per launch" >> gpurun_out/variants.txt
done
