# HEAD after the chunk-schedule work: one-GPU suite, smoke, default N=1 line, smoke launch list
set -x
mkdir -p gpurun_out/f3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f3/pytest_gpu_n1.log 2>&1; echo "rc=$?" >> gpurun_out/f3/pytest_gpu_n1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f3/smoke.log
timeout 600 python bench.py > gpurun_out/f3/bench_n1.jsonl 2> gpurun_out/f3/bench_n1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f3/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3/ncu_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f3/ncu_smoke.log
timeout 300 python bench.py --workload c2 --no-cpu-baseline > gpurun_out/f3/bench_n1_c2.jsonl 2> gpurun_out/f3/bench_n1_c2.err
