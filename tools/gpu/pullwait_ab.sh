# k_pull_rows with CTA-token ready polling: transport tests, batch-1 chunk sweep (incl. ramp),
# single transfers (per-chunk and persistent P), full c4 pair
set -x
mkdir -p gpurun_out/pw
timeout 900 python -m pytest tests/test_gpu_transport.py -m gpu -x -q > gpurun_out/pw/pytest_transport.log 2>&1; echo "rc=$?" >> gpurun_out/pw/pytest_transport.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
port=29900
for arg in "--layer-chunk 20" "--layer-chunk 10" "--layer-chunk 40" "--layer-chunk 20 --chunk-ramp" "--layer-chunk 40 --chunk-ramp" "--layer-chunk 10 --chunk-ramp"; do
  port=$((port+1))
  echo "ARGS $arg" >> gpurun_out/pw/batch1.err
  timeout 300 $TR --master-port $port bench.py --gpus 2 --requests 1 $arg --warmup 5 --steps 30 --no-e2e --no-cpu-baseline --no-nvlink-probe >> gpurun_out/pw/batch1.jsonl 2>> gpurun_out/pw/batch1.err
done
for env in "" "KVX_STAGE_PERSISTENT=1"; do
for lc in 20 10 40 -20 -40 -10; do
  env $env timeout 300 python tools/pull_probe.py --requests 1 --layer-chunk $lc --ring 3 --iters 9 --modes overlap >> gpurun_out/pw/probe_b1_$([ -z "$env" ] && echo chunked || echo persistent).jsonl 2>> gpurun_out/pw/probe.err
done
done
timeout 600 $TR --master-port 29990 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/pw/bench_n2_full.jsonl 2> gpurun_out/pw/bench_n2_full.err
