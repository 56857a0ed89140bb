# Occupancy A/B for the ALU-bound fnuz -> e4m3 row kernel: tools/variants_bench.py with the default
# build (KVX_MINB=4, 64 registers), then rebuilt with -DKVX_MINB=5 and 6.  Run from the repo root
# under gpurun; writes gpurun_out/ab_minb.txt.
mkdir -p gpurun_out
for mb in ${MINBS:-4 5 6}; do
  if [ $mb != 4 ]; then
    KVX_NVCC_FLAGS=-DKVX_MINB=$mb python -c "import sys; sys.path.insert(0,'paper_2509_17542_b200'); import build; build.build(force=True)" >> gpurun_out/ab_minb_err.txt 2>&1
  fi
  for d in e4m3 bf16; do
    echo "== minb $mb $d" >> gpurun_out/ab_minb.txt
    timeout 300 python tools/variants_bench.py --src fnuz --dst $d 2>>gpurun_out/ab_minb_err.txt | head -n 1 >> gpurun_out/ab_minb.txt
  done
  echo "== minb $mb bf16->e4m3" >> gpurun_out/ab_minb.txt
  timeout 300 python tools/variants_bench.py --src bf16 --dst e4m3 2>>gpurun_out/ab_minb_err.txt | head -n 1 >> gpurun_out/ab_minb.txt
done
