# Batch-1 c4 staged pull, single transfers (tools/pull_probe.py): D kernel alone (all chunks
# pre-staged) vs the real P/D overlap, per chunk schedule.
mkdir -p gpurun_out/probe
for lc in 80 40 20 10 5 -20 -40; do
  timeout 300 python tools/pull_probe.py --requests 1 --layer-chunk $lc --ring 3 --iters 9 >> gpurun_out/probe/b1.jsonl 2>> gpurun_out/probe/b1.err
done
timeout 300 python tools/pull_probe.py --layer-chunk 4 --ring 3 --iters 3 >> gpurun_out/probe/full.jsonl 2>> gpurun_out/probe/full.err
