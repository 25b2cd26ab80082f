set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_p2p.py -m gpu -x -q > gpurun_out/p2p_test.log 2>&1; echo "p2p test rc=$?"
for st in ssgd adpsgd; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --n-seq 2048 --same-device --strategy $st > gpurun_out/p2p_bench_$st.log 2>&1; echo "bench $st rc=$?"
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 3 --warmup 3 --no-cpu --n-seq 2048 --same-device --strategy hadpsgd --batch 160 > gpurun_out/p2p_bench_hadpsgd.log 2>&1; echo "bench hadpsgd rc=$?"
