// Per-SM limits of random gathers on B200: lanes active per LDG, shared-memory
// staging of part of the index range, and the L1 carve-out left by a large
// dynamic shared allocation (.ca vs .cg).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_mix gather_mix.cu && ./gather_mix
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// frac_hot: lanes whose index < K read shared memory (indices drawn so that
// a fraction hot of them fall below K); CG: ld.cg instead of ld.ca
template <bool CG>
__global__ void __launch_bounds__(1024, 1) k_mix(const uint32_t* __restrict__ P, uint32_t mask, uint32_t K,
                                                 uint32_t hot_thr, uint32_t iters, uint32_t* out) {
  extern __shared__ uint32_t sh[];
  for (uint32_t i = threadIdx.x; i < K; i += blockDim.x) sh[i] = P[i];
  __syncthreads();
  uint32_t acc = 0;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  for (uint32_t it = 0; it < iters; ++it) {
    uint32_t u[8], w[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t h = hsh(t * 7919u + (it * 8 + k) * 104729u);
      u[k] = (h >> 24) < hot_thr ? (K ? h % K : 0u) : (K + (h & mask));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const bool hot = u[k] < K;
      uint32_t x = 0;
      if (hot) x = sh[u[k]];
      if (!hot) x = CG ? __ldcg(P + u[k]) : __ldca(P + u[k]);
      w[k] = x;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc = max(acc, w[k]);
  }
  if (acc == 0xdeadbeef) out[0] = acc;
}

int main() {
  uint32_t *P, *out;
  cudaMalloc(&P, (1ull << 26) * 4);
  cudaMemset(P, 1, (1ull << 26) * 4);
  cudaMalloc(&out, 4);
  cudaFuncSetAttribute(k_mix<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k_mix<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint32_t iters = 256, mask = (1u << 23) - 1;  // 32 MB cold region
  struct { uint32_t K, thr, dyn; } cases[] = {
      {0, 0, 0}, {0, 0, 64 << 10}, {0, 0, 128 << 10}, {0, 0, 200 << 10},
      {16384, 64, 64 << 10}, {16384, 128, 64 << 10}, {16384, 256, 64 << 10},
      {32768, 85, 128 << 10}, {32768, 128, 128 << 10}, {32768, 256, 128 << 10},
      {51200, 85, 200 << 10}, {51200, 256, 200 << 10}};
  for (int cg = 0; cg < 2; ++cg)
    for (auto c : cases) {
      const size_t dyn = c.dyn > c.K * 4 ? c.dyn : c.K * 4;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (cg) k_mix<true><<<148, 1024, dyn>>>(P, mask, c.K, c.thr, iters, out);
        else k_mix<false><<<148, 1024, dyn>>>(P, mask, c.K, c.thr, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double g = 148.0 * 1024 * iters * 8 / (ms * 1e-3) / 1e9;
        if (rep)
          printf("%s K=%6u hot=%5.1f%% smem=%3zu KB: %7.1f G gathers/s total, %7.1f G/s from L2\n", cg ? "cg" : "ca",
                 c.K, 100.0 * c.thr / 256, dyn >> 10, g, g * (1.0 - c.thr / 256.0));
      }
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
