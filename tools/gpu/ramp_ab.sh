# Ramped vs uniform staged-pull chunks on the batch-1 c4 pair (N=2), and the one-GPU
# transport tests (ramp parity).
set -x
mkdir -p gpurun_out/ramp
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
timeout 600 python -m pytest tests/test_gpu_transport.py tests/test_abi.py -m "gpu or not gpu" -x -q > gpurun_out/ramp/pytest_transport.log 2>&1; echo "rc=$?" >> gpurun_out/ramp/pytest_transport.log
port=29600
for rep in 1 2; do
for arg in "--layer-chunk 20" "--layer-chunk 20 --no-ramp" "--layer-chunk 40" "--layer-chunk 40 --no-ramp" "--layer-chunk 16" "--layer-chunk 16 --no-ramp"; do
  port=$((port+1))
  echo "ARGS $arg" >> gpurun_out/ramp/batch1.err
  timeout 300 $TR --master-port $port bench.py --gpus 2 --requests 1 $arg --warmup 5 --steps 30 --no-e2e --no-cpu-baseline --no-nvlink-probe >> gpurun_out/ramp/batch1.jsonl 2>> gpurun_out/ramp/batch1.err
done
done
timeout 600 $TR --master-port 29650 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/ramp/bench_n2_full.jsonl 2> gpurun_out/ramp/bench_n2_full.err
