# c2 on one GPU: k_tile_copy with / without L2 evict-first hints (KVX_TC_EVICT=1); parity on
mkdir -p gpurun_out/c2ev
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "tile" > gpurun_out/c2ev/pytest_tile.log 2>&1
KVX_TC_EVICT=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "tile" > gpurun_out/c2ev/pytest_tile_evict.log 2>&1
for rep in 1 2 3; do
for env in "" "KVX_TC_EVICT=1"; do
  echo "ENV $env" >> gpurun_out/c2ev/c2.err
  env $env timeout 300 python bench.py --workload c2 --steps 30 --no-e2e --no-cpu-baseline --no-verify >> gpurun_out/c2ev/c2.jsonl 2>> gpurun_out/c2ev/c2.err
done
done
