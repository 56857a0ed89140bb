# HEAD on a 4-GPU box: multi-GPU tests and the N=2 / N=4 default lines (the driver's scaling run)
set -x
mkdir -p gpurun_out/f4
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_fullsize.py -m gpu -x -q > gpurun_out/f4/pytest_gpu_multi_n4.log 2>&1; echo "rc=$?" >> gpurun_out/f4/pytest_gpu_multi_n4.log
timeout 600 $TR --nproc-per-node 2 --master-port 29811 bench.py --gpus 2 > gpurun_out/f4/bench_n2.jsonl 2> gpurun_out/f4/bench_n2.err
timeout 600 $TR --nproc-per-node 4 --master-port 29812 bench.py --gpus 4 > gpurun_out/f4/bench_n4.jsonl 2> gpurun_out/f4/bench_n4.err
timeout 600 $TR --nproc-per-node 4 --master-port 29813 bench.py --gpus 4 --impl reference --steps 3 --warmup 3 > gpurun_out/f4/bench_ref_n4.jsonl 2> gpurun_out/f4/bench_ref_n4.err
