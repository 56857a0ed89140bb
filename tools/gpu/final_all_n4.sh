# the whole GPU suite at HEAD on a 4-GPU box (one-GPU tests + 2/4-GPU tests)
mkdir -p gpurun_out/fa
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/fa/pytest_gpu_all_n4.log 2>&1; echo "rc=$?" >> gpurun_out/fa/pytest_gpu_all_n4.log
