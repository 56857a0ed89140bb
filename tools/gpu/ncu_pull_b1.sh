# ncu --set full of the D-side persistent pull (k_pull_rows) for ONE c4 pair request with every
# chunk staged first (d_only: P and D never run concurrently, so serialised replay is safe)
mkdir -p gpurun_out/ncu_b1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pull_rows -c 1 -o gpurun_out/ncu_b1/pull_b1 \
  python tools/pull_probe.py --requests 1 --layer-chunk 20 --modes d_only --iters 1 > gpurun_out/ncu_b1/ncu.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_b1/ncu.log
