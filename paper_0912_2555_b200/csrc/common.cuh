// common.cuh — error plumbing, device buffers and warp/grid primitives shared
// by every kernel of the B200 MAP engine.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/cycheck_b200.h"

namespace cyc {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kFlag = 0x80000000u;  // accepting bit packed above the map code
constexpr uint32_t kCode = 0x7FFFFFFFu;

struct Error : std::runtime_error {
  cyc_status code;
  Error(cyc_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);

#define CYC_CUDA(call)                                                  \
  do {                                                                  \
    cudaError_t e_ = (call);                                            \
    if (e_ != cudaSuccess) ::cyc::throw_cuda(e_, #call, __FILE__, __LINE__); \
  } while (0)

extern std::atomic<uint64_t> g_launches;

#define CYC_LAUNCHED()                          \
  do {                                          \
    ::cyc::g_launches.fetch_add(1);             \
    CYC_CUDA(cudaGetLastError());               \
  } while (0)

inline uint32_t div_up(uint64_t a, uint64_t b) { return (uint32_t)((a + b - 1) / b); }

// Blocks of >= kBigBlock (16 MB) go through a process-wide grow-only cache
// (abi.cu) instead of straight back to the pool: the pool splits freed
// multi-GB blocks for small requests, and the fragmentation made later GB-sized
// requests map new memory — 100-700 ms stalls per call on config 3
// (restriction outputs). Cached blocks are reused whole (stream-ordered via
// an event recorded at release) and given back to the pool on exhaustion.
constexpr size_t kBigBlock = 16ull << 20;

// Every persistent (cooperative) kernel of the process goes through here:
// it is ordered after the previous one on the device, whatever its stream.
// Two grids spinning at grid barriers on different streams (contexts on
// separate threads) could each be partly resident and wait for each other
// forever; regular kernels beside one grid only delay it.
void coop_launch(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t st);
void* big_alloc(size_t n, cudaStream_t st, size_t* cap);
void big_free(void* p, size_t cap, cudaStream_t st);

// Stream-ordered device allocation from the context's pool.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  size_t cap = 0;  // > 0: block from the big-block cache
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t n, cudaStream_t st) { alloc(n, st); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; bytes = o.bytes; cap = o.cap; s = o.s;
      o.p = nullptr; o.bytes = 0; o.cap = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  // On failure the buffer is left empty (bytes == 0), never sized but null.
  void alloc(size_t n, cudaStream_t st) {
    release();
    s = st;
    if (n == 0) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (n >= kBigBlock && cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) {
      p = big_alloc(n, st, &cap);
      bytes = n;
      return;
    }
    cudaError_t e = cudaMallocAsync(&p, n, st);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      p = nullptr;
      throw Error(CYC_E_RESOURCE, "device memory exhausted allocating " + std::to_string(n) + " bytes");
    }
    CYC_CUDA(e);
    bytes = n;
  }
  void release() {
    if (p && cap) big_free(p, cap, s);
    else if (p) cudaFreeAsync(p, s);
    p = nullptr;
    bytes = 0;
    cap = 0;
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// ---------------------------------------------------------------- device side
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ unsigned long long ld_cg64(const unsigned long long* p) {
  return __ldcg(p);
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Inclusive warp scan (full warp converged).
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  return x;
}

__device__ __forceinline__ bool acc_bit(const uint32_t* words, uint32_t v) {
  return (__ldg(words + (v >> 5)) >> (v & 31u)) & 1u;
}

// Sense-free grid barrier for a cooperative (co-resident) grid: a monotone
// 64-bit arrival counter and a released-generation word. Thread 0 of each
// block arrives; the last arrival publishes the generation.
struct GridBar {
  unsigned long long count;
  unsigned long long pad0[15];
  unsigned long long gen;
  unsigned long long pad1[15];
};

__device__ __forceinline__ void grid_sync(GridBar* b, unsigned long long& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long target = ++epoch;
    __threadfence();
    unsigned long long arrived = atomicAdd(&b->count, 1ull) + 1ull;
    if (arrived == target * gridDim.x) {
      st_release64(&b->gen, target);
    } else {
      while (ld_acquire64(&b->gen) < target) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

}  // namespace cyc
