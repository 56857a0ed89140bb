// NVLink read-ceiling microbenchmark (not part of the library): peer-read bandwidth GPU1 -> GPU0 by
//   (a) SM loads (16 B / lane, U loads in flight), stored locally,
//   (b) 1-D bulk TMA (cp.async.bulk G->S from the peer, S->G bulk store locally),
//   (c) the copy engine (cudaMemcpyAsync).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/peer_read_bench tools/peer_read_bench.cu  (2 GPUs)
// build/peer_read_bench sizes: isolated single launches at one request's transfer sizes
// build/peer_read_bench hybrid: one read split between the copy engine and SM loads, concurrently
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <string>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int U>
__global__ void k_ldg(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t i = ((size_t)blockIdx.x * blockDim.x) * U + threadIdx.x; i < n; i += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t j = i + (size_t)u * blockDim.x;
      if (j < n) v[u] = __ldcs(src + j);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t j = i + (size_t)u * blockDim.x;
      if (j < n) __stcs(dst + j, v[u]);
    }
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_bulk(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, size_t nchunks, int chunk, int S) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t mbar[16];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  auto load = [&](size_t c, int s) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar[s])), "r"(chunk));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                     "r"(smem_u32(sm + (size_t)s * chunk)), "l"(src + c * chunk), "r"(chunk), "r"(smem_u32(&mbar[s]))
                 : "memory");
  };
  size_t it_n = nchunks > blockIdx.x ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  for (size_t it = 0; it < (size_t)S && it < it_n; ++it) load(blockIdx.x + it * gridDim.x, (int)it);
  uint32_t phase[16] = {0};
  for (size_t it = 0; it < it_n; ++it) {
    int s = (int)(it % S);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(smem_u32(&mbar[s])), "r"(phase[s]) : "memory");
    phase[s] ^= 1;
    size_t c = blockIdx.x + it * gridDim.x;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * chunk),
                 "r"(smem_u32(sm + (size_t)s * chunk)), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    if (it >= 1 && it - 1 + S < it_n) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      size_t p = it - 1;
      load(blockIdx.x + (p + S) * gridDim.x, (int)(p % S));
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  int nd = 0;
  CK(cudaGetDeviceCount(&nd));
  if (nd < 2) { printf("need 2 GPUs\n"); return 1; }
  const size_t N = (size_t)2 << 30;
  uint8_t *src, *dst;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&src, N));
  CK(cudaMemset(src, 1, N));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&dst, N));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](const char* name, auto fn) {
    std::vector<float> ts;
    for (int i = 0; i < 6; ++i) {
      CK(cudaEventRecord(e0, st));
      fn();
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (i) ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    printf("%-36s %8.3f ms  %7.1f GB/s\n", name, ts[ts.size() / 2], N / (ts[ts.size() / 2] * 1e-3) / 1e9);
  };
  if (argc > 1 && std::string(argv[1]) == "hybrid") {
    // one peer read of N bytes split between the copy engine (fraction f, its own stream) and
    // SM loads (the rest) running at the same time: does the CE's protocol add to the SMs'?
    cudaStream_t st2;
    CK(cudaStreamCreate(&st2));
    cudaEvent_t ej;
    CK(cudaEventCreateWithFlags(&ej, cudaEventDisableTiming));
    for (double f : {0.0, 0.2, 0.35, 0.5, 0.65, 0.8, 1.0}) {
      const size_t nce = (size_t)(N * f) / 4096 * 4096, nsm = N - nce;
      std::vector<float> ts;
      for (int i = 0; i < 6; ++i) {
        CK(cudaEventRecord(e0, st));
        CK(cudaStreamWaitEvent(st2, e0, 0));
        if (nce) CK(cudaMemcpyAsync(dst, src, nce, cudaMemcpyDeviceToDevice, st2));
        if (nsm) k_ldg<4><<<148 * 4, 256, 0, st>>>((const uint4*)(src + nce), (uint4*)(dst + nce), nsm / 16);
        CK(cudaEventRecord(ej, st2));
        CK(cudaStreamWaitEvent(st, ej, 0));
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (i) ts.push_back(ms);
      }
      std::sort(ts.begin(), ts.end());
      const float m = ts[ts.size() / 2];
      printf("hybrid: %3.0f%% by copy engine + %3.0f%% by SM loads  %7.3f ms  %6.1f GB/s\n", 100 * f, 100 * (1 - f), m,
             N / (m * 1e-3) / 1e9);
    }
    return 0;
  }
  if (argc > 1 && std::string(argv[1]) == "sizes") {
    // one isolated launch per timing (launch, ramp and tail included) at transfer sizes of one
    // request: the floor of a single-request pull (c4 pair: 168 MB of fp8 per request)
    for (size_t n : {(size_t)4 << 20, (size_t)21 << 20, (size_t)42 << 20, (size_t)84 << 20, (size_t)168 << 20,
                     (size_t)336 << 20}) {
      std::vector<float> tc, tk;
      for (int i = 0; i < 12; ++i) {
        float ms;
        CK(cudaEventRecord(e0, st));
        CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, st));
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (i >= 2) tc.push_back(ms);
        CK(cudaEventRecord(e0, st));
        k_ldg<4><<<148 * 4, 256, 0, st>>>((const uint4*)src, (uint4*)dst, n / 16);
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (i >= 2) tk.push_back(ms);
      }
      std::sort(tc.begin(), tc.end());
      std::sort(tk.begin(), tk.end());
      const float mc = tc[tc.size() / 2], mk = tk[tk.size() / 2];
      printf("size %7.1f MB  copy engine %7.4f ms %6.1f GB/s   ldg16 U=4 4 CTA/SM %7.4f ms %6.1f GB/s\n", n / 1048576.0,
             mc, n / (mc * 1e-3) / 1e9, mk, n / (mk * 1e-3) / 1e9);
    }
    return 0;
  }
  timeit("copy engine cudaMemcpyAsync", [&] { CK(cudaMemcpyAsync(dst, src, N, cudaMemcpyDeviceToDevice, st)); });
  for (int cpsm : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, 64, "ldg16 U=2 %d CTA/SM x256", cpsm);
    timeit(nm, [&] { k_ldg<2><<<148 * cpsm, 256, 0, st>>>((const uint4*)src, (uint4*)dst, N / 16); });
    snprintf(nm, 64, "ldg16 U=4 %d CTA/SM x256", cpsm);
    timeit(nm, [&] { k_ldg<4><<<148 * cpsm, 256, 0, st>>>((const uint4*)src, (uint4*)dst, N / 16); });
  }
  for (int chunk : {4096, 8192, 16384, 32768}) {
    for (int S : {2, 4, 6}) {
      size_t smem = (size_t)chunk * S;
      if (smem > 200 * 1024) continue;
      CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int per_sm = std::max(1, std::min(8, (int)((220 * 1024) / (smem + 2048))));
      char nm[64];
      snprintf(nm, 64, "bulk chunk %5d x %d stages, %d CTA/SM", chunk, S, per_sm);
      timeit(nm, [&] { k_bulk<<<148 * per_sm, 32, smem, st>>>(src, dst, N / chunk, chunk, S); });
    }
  }
  // reads by GPU0's SMs from GPU1 and writes by GPU1's SMs into GPU0 at the same time:
  // both carry data GPU1 -> GPU0 -- does mixing them beat either alone?
  {
    uint8_t *src1b, *dst0b;   // GPU1 -> GPU0 write pair: source on GPU1, destination on GPU0
    CK(cudaSetDevice(0));
    CK(cudaMalloc(&dst0b, N));
    CK(cudaSetDevice(1));
    CK(cudaDeviceEnablePeerAccess(0, 0));
    CK(cudaMalloc(&src1b, N));
    CK(cudaMemset(src1b, 2, N));
    cudaStream_t st1;
    CK(cudaStreamCreate(&st1));
    cudaEvent_t f0, f1;
    CK(cudaEventCreate(&f0));
    CK(cudaEventCreate(&f1));
    for (double frac : {0.0, 0.25, 0.4, 0.5, 0.6, 1.0}) {
      const size_t nr = (size_t)(N * frac) / 4096 * 4096, nw = N - nr;   // bytes read by GPU0 / written by GPU1
      std::vector<float> ts;
      for (int i = 0; i < 6; ++i) {
        CK(cudaSetDevice(0));
        CK(cudaDeviceSynchronize());
        CK(cudaSetDevice(1));
        CK(cudaDeviceSynchronize());
        CK(cudaSetDevice(0));
        CK(cudaEventRecord(e0, st));
        CK(cudaStreamWaitEvent(st1, e0, 0));   // start both together
        if (nr) k_ldg<4><<<148 * 4, 256, 0, st>>>((const uint4*)src, (uint4*)dst, nr / 16);
        CK(cudaSetDevice(1));
        if (nw) k_ldg<4><<<148 * 4, 256, 0, st1>>>((const uint4*)src1b, (uint4*)dst0b, nw / 16);   // stores go over NVLink
        CK(cudaEventRecord(f1, st1));
        CK(cudaSetDevice(0));
        CK(cudaStreamWaitEvent(st, f1, 0));
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (i) ts.push_back(ms);
      }
      std::sort(ts.begin(), ts.end());
      const float ms = ts[ts.size() / 2];
      printf("mixed: %.0f%% by GPU0 SM reads + %.0f%% by GPU1 SM writes  %8.3f ms  %7.1f GB/s GPU1->GPU0\n",
             100 * frac, 100 * (1 - frac), ms, N / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
