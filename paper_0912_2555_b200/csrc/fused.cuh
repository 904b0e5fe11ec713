// fused.cuh — row-sharded MAP with the per-step exchange fused into the step
// kernel over peer memory (CUDA IPC / NVLink); see fused.cu.
#pragma once

#include <cstring>

#include "build.cuh"

namespace cyc {

constexpr int kFusedMaxWorld = 16;

inline void require_fused(bool ok, const char* msg) {
  if (!ok) throw Error(CYC_E_CONTRACT, msg);
}

struct FusedShard {
  const DevCsr* gath = nullptr;  // the graph's gather index (owned by the cyc_graph)
  uint32_t lo = 0, hi = 0;
  int rank = 0, world = 1;
  void* base = nullptr;                    // X[2] | flags | barrier counter (cudaMalloc, IPC-exported)
  void* peer_base[kFusedMaxWorld] = {};    // every rank's base (self = base)
  size_t off_x0 = 0, off_x1 = 0, off_flags = 0, off_bar = 0, bytes = 0;
  bool connected = false;
  int final_cur = 0;
  unsigned long long barriers_done = 0;    // cross-rank barriers completed (identical on every rank)

  ~FusedShard();
  // allocates the shared block and writes its cudaIpcMemHandle_t (64 bytes)
  void open(const DevCsr& gath, uint32_t lo, uint32_t hi, int rank, int world, void* handle_out);
  // handles: world x 64 bytes, in rank order
  void connect(const void* handles);
  // one run_map over the sharded rows; res = {cycle, witness, iterations,
  // kernel_calls, demoted_total, final buffer index}
  void run(const uint64_t* acc_words, int early_exit, cudaStream_t s, unsigned long long res[6]);
  void final_vector(uint32_t* out, cudaStream_t s) const;
};

}  // namespace cyc
