# HEAD verification on a 4-GPU box: multi-GPU tests, N=2 / N=4 bench lines (the driver's
# scaling run), a batch-1 c4 pair sweep over layer chunks.
set -x
mkdir -p gpurun_out/v4
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_fullsize.py -m gpu -x -q > gpurun_out/v4/pytest_gpu_multi_n4.log 2>&1; echo "rc=$?" >> gpurun_out/v4/pytest_gpu_multi_n4.log
timeout 600 $TR --nproc-per-node 2 --master-port 29511 bench.py --gpus 2 > gpurun_out/v4/bench_n2.jsonl 2> gpurun_out/v4/bench_n2.err
timeout 600 $TR --nproc-per-node 4 --master-port 29512 bench.py --gpus 4 > gpurun_out/v4/bench_n4.jsonl 2> gpurun_out/v4/bench_n4.err
timeout 600 $TR --nproc-per-node 2 --master-port 29513 bench.py --gpus 2 --impl reference --steps 3 --warmup 3 > gpurun_out/v4/bench_ref_n2.jsonl 2> gpurun_out/v4/bench_ref_n2.err
port=29530
for lc in 0 10 20 40; do
  port=$((port+1))
  timeout 300 $TR --nproc-per-node 2 --master-port $port bench.py --gpus 2 --requests 1 --layer-chunk $lc --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/v4/batch1_chunks.jsonl 2>> gpurun_out/v4/batch1_chunks.err
done
