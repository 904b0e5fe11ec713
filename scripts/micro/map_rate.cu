// First-touch cost of device memory on one B200: how fast the driver maps new
// physical memory into a stream-ordered pool (cudaMallocAsync growth) and
// through cudaMalloc, vs reuse of memory the pool already holds.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o map_rate map_rate.cu && ./map_rate
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  double t = now_ms();
  cudaFree(0);
  printf("context %.1f ms\n", now_ms() - t);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaMemPool_t pool;
  cudaDeviceGetDefaultMemPool(&pool, 0);
  uint64_t thr = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  const size_t blk = 8ull << 30;
  void* p[8];
  for (int round = 0; round < 2; ++round) {
    t = now_ms();
    for (int i = 0; i < 7; ++i) cudaMallocAsync(&p[i], blk, s);
    cudaStreamSynchronize(s);
    const double ta = now_ms() - t;
    t = now_ms();
    for (int i = 0; i < 7; ++i) cudaMemsetAsync(p[i], 0, blk, s);
    cudaStreamSynchronize(s);
    const double tm = now_ms() - t;
    for (int i = 0; i < 7; ++i) cudaFreeAsync(p[i], s);
    cudaStreamSynchronize(s);
    printf("pool round %d: alloc 56 GB %.1f ms, first memset %.1f ms (%.0f GB/s)\n", round, ta, tm, 56.0 / tm * 1e3);
  }
  // other sizes out of the held pool
  t = now_ms();
  for (int i = 0; i < 8; ++i) cudaMallocAsync(&p[i], 6ull << 30, s);
  cudaStreamSynchronize(s);
  printf("pool resplit 8 x 6 GB %.1f ms\n", now_ms() - t);
  for (int i = 0; i < 8; ++i) cudaFreeAsync(p[i], s);
  cudaStreamSynchronize(s);
  thr = 0;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  cudaMemPoolTrimTo(pool, 0);
  t = now_ms();
  void* q;
  cudaMalloc(&q, 56ull << 30);
  const double ta = now_ms() - t;
  t = now_ms();
  cudaMemset(q, 0, 56ull << 30);
  cudaDeviceSynchronize();
  printf("cudaMalloc 56 GB %.1f ms, memset %.1f ms\n", ta, now_ms() - t);
  cudaFree(q);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
