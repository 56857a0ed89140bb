mkdir -p gpurun_out/tl2
for lc in 20 10; do
  timeout 300 python tools/pull_timeline.py --layer-chunk $lc --iters 3 --sleep-ms 3 >> gpurun_out/tl2/timeline.jsonl 2>> gpurun_out/tl2/timeline.err
  timeout 300 python tools/pull_timeline.py --layer-chunk $lc --iters 3 --sleep-ms 3 --p-only >> gpurun_out/tl2/timeline.jsonl 2>> gpurun_out/tl2/timeline.err
done
timeout 300 python tools/pull_timeline.py --layer-chunk 5 --iters 3 --sleep-ms 3 --p-only >> gpurun_out/tl2/timeline.jsonl 2>> gpurun_out/tl2/timeline.err
