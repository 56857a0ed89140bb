# A/B of the widening-cast occupancy cap (KVX_MINB_WIDEN): default build (3), then rebuilt with 4.
# fp8 -> wider and one narrowing control through tools/variants_bench.py (first line: the row kernel).
# Run from the repo root under gpurun; writes gpurun_out/ab_widen.txt.
mkdir -p gpurun_out
for mw in 3 4; do
  if [ $mw != 3 ]; then
    KVX_NVCC_FLAGS=-DKVX_MINB_WIDEN=$mw python -c "import sys; sys.path.insert(0,'paper_2509_17542_b200'); import build; build.build(force=True)" >> gpurun_out/ab_widen_err.txt 2>&1
  fi
  for sd in "fnuz bf16" "e4m3 bf16" "fnuz f32" "e4m3 f32" "fnuz e4m3" "bf16 e4m3" "bf16 f32"; do
    set -- $sd
    echo "== widen $mw $1 -> $2" >> gpurun_out/ab_widen.txt
    timeout 300 python tools/variants_bench.py --src $1 --dst $2 2>>gpurun_out/ab_widen_err.txt | head -n 1 >> gpurun_out/ab_widen.txt
  done
done
