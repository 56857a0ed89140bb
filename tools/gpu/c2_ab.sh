# c2 on one GPU (same dtype fp16, TP2 -> 1): k_tile_copy (default) vs k_tile_cast (KVX_TT_SAME=1) vs rows
mkdir -p gpurun_out/c2ab
for rep in 1 2 3; do
for env in "" "KVX_TT_SAME=1" "KVX_TILE=0"; do
  echo "ENV $env" >> gpurun_out/c2ab/c2.err
  env $env timeout 300 python bench.py --workload c2 --steps 30 --no-e2e --no-cpu-baseline --no-parity --no-verify >> gpurun_out/c2ab/c2.jsonl 2>> gpurun_out/c2ab/c2.err
done
done
