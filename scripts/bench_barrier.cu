// Microbenchmark: cost of the engine's grid barrier (common.cuh grid_sync)
// and of a cooperative-groups grid.sync(), in a cooperative persistent grid.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/bench_barrier.cu -o /tmp/bb
#include <cooperative_groups.h>
#include <cstdio>

#include "../paper_0912_2555_b200/csrc/common.cuh"

namespace cg = cooperative_groups;
using namespace cyc;

__global__ void __launch_bounds__(1024, 1) k_bar(GridBar* b, int iters, unsigned long long* out) {
  unsigned long long epoch = 0;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) grid_sync(b, epoch);
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

__global__ void __launch_bounds__(1024, 1) k_cg(int iters, unsigned long long* out) {
  cg::grid_group g = cg::this_grid();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

// flag + counter pattern without the initial __syncthreads fence storm:
// hierarchical: 148 blocks arrive on 8 sub-counters, leaders combine.
std::atomic<uint64_t> cyc::g_launches{0};
void cyc::throw_cuda(cudaError_t e, const char* w, const char* f, int l) {
  fprintf(stderr, "%s %s %s:%d\n", cudaGetErrorString(e), w, f, l);
  exit(1);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  GridBar* b;
  unsigned long long* out;
  cudaMalloc(&b, sizeof(GridBar));
  cudaMalloc(&out, 16);
  for (int threads : {1024, 512, 256}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(b, 0, sizeof(GridBar));
      int iters = 20000;
      void* args[] = {&b, &iters, &out};
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      CYC_CUDA(cudaLaunchCooperativeKernel((void*)k_bar, sms, threads, args, 0, 0));
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("grid_sync  blocks=%d threads=%d: %.3f us/barrier\n", sms, threads, ms * 1e3 / iters);
      void* args2[] = {&iters, &out};
      cudaEventRecord(e0);
      CYC_CUDA(cudaLaunchCooperativeKernel((void*)k_cg, sms, threads, args2, 0, 0));
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("cg::sync   blocks=%d threads=%d: %.3f us/barrier\n", sms, threads, ms * 1e3 / iters);
    }
  }
  return 0;
}
