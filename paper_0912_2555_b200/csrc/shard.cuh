// shard.cuh — one rank's part of a row-sharded MAP run.
#pragma once

#include <vector>

#include "map_run.cuh"

namespace cyc {

// A rank builds only its rows: from the full edge log it derives the (shared,
// deterministic) storage order and edge-balanced row ranges, keeps the logged
// edges whose gather row falls in [row_lo, row_hi), and builds from those
// alone its gather rows and the push rows that target them. Map vector and
// frontier bitmaps are replicated; the exchange buffers are plain cudaMalloc
// so they can be shared with peers by CUDA IPC or peer access.
struct ShardGraph {
  int device = 0;
  uint32_t n = 0, n_pad = 0;
  uint64_t m_global = 0;  // snapshot edges of the whole graph (sum over ranks)
  uint64_t m_local = 0;
  int world = 1, rank = 0;
  uint32_t row_lo = 0, row_hi = 0;
  bool relabel = false;
  DevBuf orig, perm;       // storage layout (degree order) when relabel
  DevCsr gath, push;       // this rank's gather rows / push rows restricted to its targets
  DevBuf sell, sdesc, hcol, hrow;
  uint32_t n_hchunks = 0;
  uint64_t sell_words = 0;
  DevBuf acc;              // accepting words (u64) in vertex-id order
  RunWs ws;
  // exchange buffers (cudaMalloc): map words [2], frontier bitmaps [2], records, barrier
  uint32_t* xP[2] = {nullptr, nullptr};
  uint32_t* xFB[2] = {nullptr, nullptr};
  ShardRec* rec = nullptr;
  unsigned long long* bar = nullptr;
  unsigned long long bars_done = 0;
  // peers (index = rank; self included)
  uint32_t* peerP[kMaxWorld][2] = {};
  uint32_t* peerFB[kMaxWorld][2] = {};
  ShardRec* peerRec[kMaxWorld] = {};
  unsigned long long* peerBar[kMaxWorld] = {};
  std::vector<void*> opened;  // IPC mappings to close
  bool emulated = false;
  ~ShardGraph();
  uint64_t device_bytes() const;
};

// IPC handles of a rank's exchange buffers.
struct ShardHandles {
  cudaIpcMemHandle_t h[6];
  unsigned long long m_local;  // the rank's snapshot edges (the ranks' sum is the graph's)
  int world, rank;
};

void build_shard(const uint32_t* d_edges, uint64_t m_log, uint32_t n, const uint64_t* acc_words,
                 int orientation, int world, int rank, int layout, ShardGraph& sh, BuildArena& ar,
                 cudaStream_t s);
void shard_export(const ShardGraph& sh, ShardHandles& out);
void shard_connect_ipc(ShardGraph& sh, const ShardHandles* all, int world);
// Same-process peers (distinct devices with peer access, or one device: emulated).
void shard_connect_local(ShardGraph* const* shards, int world);
// Runs run_map on every rank of the process: one cooperative grid per device,
// or one emulated grid holding all ranks when they share a device.
void shard_run(ShardGraph* const* shards, int world_here, const uint64_t* acc_words, int early_exit, int mode,
               unsigned long long max_iterations, unsigned long long max_steps, uint32_t alpha,
               unsigned long long cap, cudaStream_t const* streams, cudaEvent_t e0, cudaEvent_t e1,
               RunOut* outs);
// Final vector (vertex-id order) of a rank's replica.
void shard_values(const ShardGraph& sh, int cur, uint32_t* dst, cudaStream_t s);

}  // namespace cyc
