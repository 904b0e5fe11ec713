// Random 4-byte gather throughput on one B200: G gathers/s for a region of
// `words` u32 (indices from a hash, ILP loads in flight per thread), to find
// the L2-resident random-access ceiling that bounds the MAP pull step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bw gather_bw.cu && ./gather_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int ILP, int MODE>
__global__ void __launch_bounds__(1024, 1) k_gather(const uint32_t* __restrict__ P, uint32_t mask, uint32_t iters,
                                                    uint32_t* out, const uint32_t* __restrict__ idx) {
  uint32_t acc = 0;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t T = gridDim.x * blockDim.x;
  for (uint32_t it = 0; it < iters; ++it) {
    uint32_t u[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      if (MODE == 0) u[k] = hsh(t * 7919u + (it * ILP + k) * 104729u) & mask;
      else u[k] = __ldcs(idx + ((size_t)(it * ILP + k) * T + t) % (64u << 20));  // streamed indices
    }
    uint32_t w[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) w[k] = MODE == 2 ? __ldcg(P + u[k]) : __ldca(P + u[k]);
#pragma unroll
    for (int k = 0; k < ILP; ++k) acc = max(acc, w[k]);
  }
  if (acc == 0xdeadbeef) out[0] = acc;
}

__global__ void k_idx(uint32_t* idx, uint32_t n, uint32_t mask) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) idx[i] = hsh(i * 2654435761u) & mask;
}

int main() {
  uint32_t *P, *out, *idx;
  const size_t maxw = 1ull << 28;
  cudaMalloc(&P, maxw * 4);
  cudaMemset(P, 1, maxw * 4);
  cudaMalloc(&out, 4);
  cudaMalloc(&idx, (64u << 20) * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint32_t iters = 256;
  for (int mode = 0; mode < 3; ++mode) {
    for (int lg = 18; lg <= 28; lg += 1) {
      const uint32_t mask = (1u << lg) - 1u;
      if (mode) { k_idx<<<1184, 256>>>(idx, 64u << 20, mask); cudaDeviceSynchronize(); }
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k_gather<8, 0><<<148, 1024>>>(P, mask, iters, out, idx);
        else if (mode == 1) k_gather<8, 1><<<148, 1024>>>(P, mask, iters, out, idx);
        else k_gather<8, 2><<<148, 1024>>>(P, mask, iters, out, idx);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double g = 148.0 * 1024 * iters * 8 / (ms * 1e-3) / 1e9;
        if (rep) printf("mode %d (%s) region %7.1f MB: %8.1f G gathers/s (%.2f ms)\n", mode,
                        mode == 0 ? "hash idx, ld.ca" : mode == 1 ? "streamed idx, ld.ca" : "streamed idx, ld.cg",
                        (4.0 * (1u << lg)) / 1e6, g, ms);
      }
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
