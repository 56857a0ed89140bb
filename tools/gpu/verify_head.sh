set -x
mkdir -p gpurun_out/v1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v1/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v1/pytest_gpu_n1.log 2>&1; echo "rc=$?" >> gpurun_out/v1/pytest_gpu_n1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v1/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/v1/smoke.log
timeout 600 python bench.py > gpurun_out/v1/bench_n1.jsonl 2> gpurun_out/v1/bench_n1.err; echo "rc=$?" >> gpurun_out/v1/bench_n1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v1/bench_ref.jsonl 2> gpurun_out/v1/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v1/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v1/ncu_smoke.log 2>&1
