# smoke() under ncu (serialised launches): its launch list; the serialised-launch test.
set -x
mkdir -p gpurun_out/v2
timeout 600 python -m pytest tests/test_gpu_transport.py -m gpu -x -q > gpurun_out/v2/pytest_transport.log 2>&1; echo "rc=$?" >> gpurun_out/v2/pytest_transport.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v2/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v2/ncu_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/v2/ncu_smoke.log
