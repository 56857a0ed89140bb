# after the chunk-plan overflow fix: one-GPU transport tests, the two-GPU multi tests (incl.
# the persistent-P staged pull) and the default N=2 line
set -x
mkdir -p gpurun_out/f2b
timeout 900 python -m pytest tests/test_gpu_transport.py tests/test_gpu_multi.py -m gpu -x -q > gpurun_out/f2b/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f2b/pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2 --master-port 29871 bench.py --gpus 2 > gpurun_out/f2b/bench_n2.jsonl 2> gpurun_out/f2b/bench_n2.err
