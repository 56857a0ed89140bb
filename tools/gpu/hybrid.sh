mkdir -p gpurun_out/hy
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/peer_read_bench tools/peer_read_bench.cu && timeout 120 build/peer_read_bench hybrid > gpurun_out/hy/hybrid.txt 2>&1
