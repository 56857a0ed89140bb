# A/B of the e4m3fnuz decode on one GPU: GPU suite + tools/variants_bench.py (fnuz -> e4m3 / bf16)
# with KVX_FNUZ_SHIFT=1 (default build), then rebuilt with -DKVX_FNUZ_SHIFT=0.  Run from the repo root
# under gpurun; writes gpurun_out/ab_fnuz.txt.

mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1; echo "pytest $?" >> gpurun_out/ab_pytest.log
for r in 1 2; do
echo "== new" >> gpurun_out/ab_fnuz.txt
for d in e4m3 bf16; do timeout 300 python tools/variants_bench.py --src fnuz --dst $d >> gpurun_out/ab_fnuz.txt 2>>gpurun_out/ab_err.txt; done
done
KVX_NVCC_FLAGS=-DKVX_FNUZ_SHIFT=0 python -c "import sys; sys.path.insert(0,'paper_2509_17542_b200'); import build; build.build(force=True)" >> gpurun_out/ab_err.txt 2>&1
for r in 1 2; do
echo "== old" >> gpurun_out/ab_fnuz.txt
for d in e4m3 bf16; do timeout 300 python tools/variants_bench.py --src fnuz --dst $d >> gpurun_out/ab_fnuz.txt 2>>gpurun_out/ab_err.txt; done
done
tail -n 3 gpurun_out/ab_pytest.log
