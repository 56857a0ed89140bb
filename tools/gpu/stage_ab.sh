# persistent k_stage_rows: one-GPU transport tests + smoke (incl. serialised), then the
# batch-1 and full c4 pair with / without it and with / without the chunk ramp
set -x
mkdir -p gpurun_out/stage
timeout 900 python -m pytest tests/test_gpu_transport.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/stage/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/stage/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/stage/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/stage/smoke.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
port=29700
for rep in 1 2; do
for env in "" "KVX_STAGE_CHUNKED=1"; do
for arg in "--layer-chunk 20" "--layer-chunk 20 --no-ramp" "--layer-chunk 10 --no-ramp" "--layer-chunk 40 --no-ramp" "--layer-chunk 40"; do
  port=$((port+1))
  echo "ENV $env ARGS $arg" >> gpurun_out/stage/batch1.err
  env $env timeout 300 $TR --master-port $port bench.py --gpus 2 --requests 1 $arg --warmup 5 --steps 30 --no-e2e --no-cpu-baseline --no-nvlink-probe >> gpurun_out/stage/batch1.jsonl 2>> gpurun_out/stage/batch1.err
done
done
done
for lc in 20 40 -20 -40 10 -10; do
  timeout 300 python tools/pull_probe.py --requests 1 --layer-chunk $lc --ring 3 --iters 9 --modes overlap >> gpurun_out/stage/probe_b1.jsonl 2>> gpurun_out/stage/probe.err
done
timeout 600 $TR --master-port 29790 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/stage/bench_n2_full.jsonl 2> gpurun_out/stage/bench_n2_full.err
