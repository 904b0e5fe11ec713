// shard.cu — building one rank's part of a row-sharded graph, and wiring the
// ranks' exchange buffers together (the partition rule is the
// reference's worker split, map_engine.cpp:35-43: contiguous row ranges
// balanced by edge count).
//
// Every rank reads the whole edge log (generated on its device, or copied
// in) but keeps only the edges of its own rows:
//   1. gather-column and gather-row counts of the log (one pass, atomics);
//   2. the storage order (degree layout: descending gather count, the same
//      stable sort as plan.cu on the log's counts, so identical on every rank);
//   3. edge-balanced row ranges over the storage order, rounded to the
//      kRowPad padding (identical on every rank, no communication);
//   4. the log's edges whose gather row is one of this rank's, relabelled;
//   5. from those alone: the gather rows (K1 build_csr, rows keyed by the
//      gather row) and the push rows restricted to this rank's targets (K1,
//      keyed by the gather column), then the sliced ELL and heavy slab.
// Per-rank edge memory is ~1/world of the graph; the map vector and frontier
// bitmaps (O(n)) are replicated.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "plan.cuh"
#include "shard.cuh"

namespace cyc {

namespace {

// counts: gcol[u] = edges whose gather column is u (the gather frequency),
// grow[v] = edges of gather row v. Transposed snapshot: gather row = source.
__global__ void k_shard_counts(const uint2* __restrict__ e, uint64_t m, uint32_t n, int transposed,
                               uint32_t* __restrict__ gcol, uint32_t* __restrict__ grow, uint32_t* err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 x = e[i];
    if (x.x >= n || x.y >= n) {
      atomicExch(err, 1u);
      continue;
    }
    const uint32_t r = transposed ? x.x : x.y, c = transposed ? x.y : x.x;
    atomicAdd(gcol + c, 1u);
    atomicAdd(grow + r, 1u);
  }
}

// row lengths in storage order
__global__ void k_shard_rowlen(uint32_t n, const uint32_t* __restrict__ orig, const uint32_t* __restrict__ grow,
                               uint32_t* __restrict__ out) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    out[p] = grow[orig ? orig[p] : p];
}

// bounds[r] = first storage row whose exclusive prefix reaches r * total / world
__global__ void k_shard_bounds(const uint32_t* __restrict__ pre, uint32_t n, int world, uint32_t* bounds) {
  const int r = threadIdx.x;
  if (r > world) return;
  const uint64_t total = pre[n];
  const uint64_t target = total * (uint64_t)r / (uint64_t)world;
  uint32_t lo = 0, hi = n;  // first p with pre[p] >= target
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (pre[mid] < target) lo = mid + 1; else hi = mid;
  }
  bounds[r] = lo;
}

// Edges whose gather row (in storage order) is in [lo, hi), as (gather row,
// gather column) pairs in VERTEX ids (K1's buckets balance on the id order;
// in degree order the first bucket would hold the hubs). PASS 0 counts, PASS 1 writes.
template <int PASS>
__global__ void k_shard_filter(const uint2* __restrict__ e, uint64_t m, int transposed,
                               const uint32_t* __restrict__ perm, uint32_t lo, uint32_t hi,
                               unsigned long long* cnt, uint2* __restrict__ out) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t base0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) & ~31ull;
  for (uint64_t b = base0; b < m; b += stride) {
    const uint64_t i = b + lane;
    bool keep = false;
    uint2 y = make_uint2(0u, 0u);
    if (i < m) {
      const uint2 x = e[i];
      const uint32_t r = transposed ? x.x : x.y, c = transposed ? x.y : x.x;
      const uint32_t pr = perm ? __ldg(perm + r) : r;
      keep = pr >= lo && pr < hi;
      y = make_uint2(r, c);
    }
    const uint32_t bal = __ballot_sync(kFull, keep);
    if (!bal) continue;
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(cnt, (unsigned long long)__popc(bal));
    pos = __shfl_sync(kFull, pos, 0);
    if (PASS == 1 && keep) out[pos + __popc(bal & ((1u << lane) - 1u))] = y;
  }
}

// final vector of a replica in vertex-id order
__global__ void k_shard_values(const uint32_t* __restrict__ P, const uint32_t* __restrict__ orig, uint32_t n,
                               uint32_t* __restrict__ out) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    out[orig ? orig[p] : p] = P[p] & kCode;
}

void* xalloc(size_t bytes) {  // exchange buffers: plain cudaMalloc (IPC-exportable)
  void* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw Error(CYC_E_RESOURCE, "device memory exhausted allocating shard exchange buffers");
  }
  CYC_CUDA(e);
  CYC_CUDA(cudaMemset(p, 0, bytes));
  return p;
}

}  // namespace

ShardGraph::~ShardGraph() {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  for (void* p : opened) cudaIpcCloseMemHandle(p);
  for (void* p : {(void*)xP[0], (void*)xP[1], (void*)xFB[0], (void*)xFB[1], (void*)rec, (void*)bar})
    if (p) cudaFree(p);
  cudaSetDevice(prev);
}

uint64_t ShardGraph::device_bytes() const {
  auto b = [](const DevBuf& x) { return (uint64_t)x.bytes; };
  return b(gath.off) + b(gath.col) + b(gath.heavy) + b(push.off) + b(push.col) + b(sell) + b(sdesc) + b(hcol) +
         b(hrow) + b(orig) + b(perm) + 2ull * ((uint64_t)n_pad + 1) * 4 + 2ull * ((uint64_t)n_pad / 32 + 2) * 4;
}

void build_shard(const uint32_t* d_edges, uint64_t m_log, uint32_t n, const uint64_t* acc_words, int orientation,
                 int world, int rank, int layout, ShardGraph& sh, BuildArena& ar, cudaStream_t s) {
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
    throw Error(CYC_E_CONTRACT, "shard: bad world/rank");
  CYC_CUDA(cudaGetDevice(&sh.device));
  const bool dbg = std::getenv("CYC_DEBUG_TIMING") != nullptr;
  auto tm = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {  // CYC_DEBUG_TIMING=1: host-observed phase times
    if (!dbg) return;
    CYC_CUDA(cudaStreamSynchronize(s));
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[cyc shard %d/%d] %-10s %8.3f ms\n", rank, world, what,
                 std::chrono::duration<double, std::milli>(now - tm).count());
    tm = now;
  };
  const int transposed = orientation == CYC_TRANSPOSED;
  const uint2* e2 = reinterpret_cast<const uint2*>(d_edges);
  sh.n = n;
  sh.n_pad = (uint32_t)(((uint64_t)n + kRowPad - 1) / kRowPad * kRowPad);
  sh.world = world;
  sh.rank = rank;
  const uint32_t np = sh.n_pad;
  DevBuf gcol(((size_t)n + 1) * 4, s), grow(((size_t)n + 1) * 4, s), err(16, s), scratch;
  CYC_CUDA(cudaMemsetAsync(gcol.p, 0, gcol.bytes, s));
  CYC_CUDA(cudaMemsetAsync(grow.p, 0, grow.bytes, s));
  CYC_CUDA(cudaMemsetAsync(err.p, 0, 16, s));
  if (m_log) {
    k_shard_counts<<<grid_for(m_log, 256, 8), 256, 0, s>>>(e2, m_log, n, transposed, gcol.as<uint32_t>(),
                                                            grow.as<uint32_t>(), err.as<uint32_t>());
    CYC_LAUNCHED();
  }
  uint32_t herr = 0;
  CYC_CUDA(cudaMemcpyAsync(&herr, err.p, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  if (herr) throw Error(CYC_E_CONTRACT, "build_snapshot: edge endpoint >= n (not interned)");
  mark("counts");
  // storage order (degree layout: descending gather frequency of the log);
  // auto as plan.cu: a map vector beyond ~40 MB whose n/8 most-gathered
  // vertices take at least half of the gathers
  const bool want = n >= 64 && (layout == 2 || (layout == 0 && (uint64_t)n * 4 > (40ull << 20)));
  if (want) {
    DevBuf koff(((size_t)n + 1) * 4, s), toff(((size_t)n + 1) * 4, s);
    exclusive_scan(gcol.as<uint32_t>(), koff.as<uint32_t>(), n, nullptr, s, scratch);
    exclusive_scan(grow.as<uint32_t>(), toff.as<uint32_t>(), n, nullptr, s, scratch);
    sh.orig.alloc(((size_t)np + 1) * 4, s);
    sh.perm.alloc((size_t)n * 4, s);
    degree_order(koff.as<uint32_t>(), toff.as<uint32_t>(), n, sh.orig.as<uint32_t>(), sh.perm.as<uint32_t>(), s);
    sh.relabel = true;
    if (layout == 0) {
      DevBuf hl(((size_t)n + 1) * 4, s), hp(((size_t)n + 1) * 4, s);
      k_shard_rowlen<<<grid_for(n, 256, 8), 256, 0, s>>>(n, sh.orig.as<uint32_t>(), gcol.as<uint32_t>(),
                                                         hl.as<uint32_t>());
      CYC_LAUNCHED();
      exclusive_scan(hl.as<uint32_t>(), hp.as<uint32_t>(), n, nullptr, s, scratch);
      uint32_t hot = 0, all = 0;
      CYC_CUDA(cudaMemcpyAsync(&hot, hp.as<uint32_t>() + n / 8, 4, cudaMemcpyDeviceToHost, s));
      CYC_CUDA(cudaMemcpyAsync(&all, hp.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, s));
      CYC_CUDA(cudaStreamSynchronize(s));
      if ((double)hot < 0.5 * (double)all) {
        sh.relabel = false;
        sh.orig = DevBuf();
        sh.perm = DevBuf();
      }
    }
  }
  // edge-balanced row ranges (every rank computes the same ones)
  std::vector<uint32_t> bounds(world + 1);
  {
    DevBuf rl(((size_t)n + 1) * 4, s), pre(((size_t)n + 1) * 4, s), bd(((size_t)world + 1) * 4, s);
    k_shard_rowlen<<<grid_for(n ? n : 1, 256, 8), 256, 0, s>>>(n, sh.relabel ? sh.orig.as<uint32_t>() : nullptr,
                                                               grow.as<uint32_t>(), rl.as<uint32_t>());
    CYC_LAUNCHED();
    exclusive_scan(rl.as<uint32_t>(), pre.as<uint32_t>(), n, nullptr, s, scratch);
    k_shard_bounds<<<1, 32, 0, s>>>(pre.as<uint32_t>(), n, world, bd.as<uint32_t>());
    CYC_LAUNCHED();
    CYC_CUDA(cudaMemcpyAsync(bounds.data(), bd.p, (world + 1) * 4, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
  }
  for (int r = 0; r <= world; ++r) {  // rank boundaries on whole row-padding groups
    uint32_t b = (uint32_t)(((uint64_t)bounds[r] + kRowPad / 2) / kRowPad * kRowPad);
    if (r == 0) b = 0;
    if (r == world) b = np;
    bounds[r] = std::min(np, std::max(b, r ? bounds[r - 1] : 0u));
  }
  sh.row_lo = bounds[rank];
  sh.row_hi = bounds[rank + 1];
  mark("order");
  // this rank's edges, relabelled
  DevBuf cnt(16, s);
  CYC_CUDA(cudaMemsetAsync(cnt.p, 0, 16, s));
  const uint32_t* perm = sh.relabel ? sh.perm.as<uint32_t>() : nullptr;
  unsigned long long mine = 0;
  if (m_log) {
    k_shard_filter<0><<<grid_for(m_log, 256, 8), 256, 0, s>>>(e2, m_log, transposed, perm, sh.row_lo, sh.row_hi,
                                                              cnt.as<unsigned long long>(), nullptr);
    CYC_LAUNCHED();
    CYC_CUDA(cudaMemcpyAsync(&mine, cnt.p, 8, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
  }
  DevBuf pairs((mine ? mine : 1) * 8, s);
  if (mine) {
    CYC_CUDA(cudaMemsetAsync(cnt.p, 0, 16, s));
    k_shard_filter<1><<<grid_for(m_log, 256, 8), 256, 0, s>>>(e2, m_log, transposed, perm, sh.row_lo, sh.row_hi,
                                                              cnt.as<unsigned long long>(), pairs.as<uint2>());
    CYC_LAUNCHED();
  }
  mark("filter");
  // gather rows keyed by the pair's first element, push rows by its second
  // (vertex ids), then both relabelled to the storage order
  if (sh.relabel) {
    DevCsr g0, p0;
    build_csr(pairs.as<uint32_t>(), mine, n, 0, s, g0, err.as<uint32_t>(), ar);
    build_csr(pairs.as<uint32_t>(), mine, n, 1, s, p0, err.as<uint32_t>(), ar);
    mark("csrs");
    pairs = DevBuf();
    build_heavy(g0, kHeavyDeg, kHeavyChunk, s, 1u);
    build_heavy(p0, kHeavyDeg, kHeavyChunk, s, 1u);
    relayout(g0, sh.orig.as<uint32_t>(), sh.perm.as<uint32_t>(), sh.gath, scratch, s);
    relayout(p0, sh.orig.as<uint32_t>(), sh.perm.as<uint32_t>(), sh.push, scratch, s);
    mark("relayout");
  } else {
    build_csr(pairs.as<uint32_t>(), mine, n, 0, s, sh.gath, err.as<uint32_t>(), ar);
    build_csr(pairs.as<uint32_t>(), mine, n, 1, s, sh.push, err.as<uint32_t>(), ar);
    mark("csrs");
    pairs = DevBuf();
  }
  sh.m_local = sh.gath.m;
  build_hslab(sh.gath, np, sh.hcol, sh.hrow, sh.n_hchunks, s);
  sh.sell_words = build_sell(sh.gath, sh.row_lo, sh.row_hi, np, sh.sell, sh.sdesc, s);
  mark("slabs");
  // accepting words (vertex-id order), the workspace and the exchange buffers
  sh.acc.alloc((((size_t)n + 63) / 64 + 1) * 8, s);
  CYC_CUDA(cudaMemsetAsync(sh.acc.p, 0, sh.acc.bytes, s));
  if (acc_words && n) CYC_CUDA(cudaMemcpyAsync(sh.acc.p, acc_words, ((size_t)n + 63) / 64 * 8, cudaMemcpyDefault, s));
  sh.ws.ensure(n, sh.gath.m, sh.push.o(), s);
  CYC_CUDA(cudaStreamSynchronize(s));
  for (int b = 0; b < 2; ++b) {
    sh.xP[b] = static_cast<uint32_t*>(xalloc(((size_t)np + 1) * 4));
    sh.xFB[b] = static_cast<uint32_t*>(xalloc(((size_t)np / 32 + 2) * 4));
  }
  sh.rec = static_cast<ShardRec*>(xalloc(sizeof(ShardRec) * 2 * kMaxWorld));
  sh.bar = static_cast<unsigned long long*>(xalloc(64));
  mark("buffers");
  // the global snapshot edge count: every rank's rows are disjoint, so
  // m_global = sum over ranks; a rank alone knows only its own. Ranks agree
  // on it when connected (shard_connect_*); until then it is the local one.
  sh.m_global = sh.m_local;
  for (int p = 0; p < kMaxWorld; ++p) {
    sh.peerP[p][0] = sh.peerP[p][1] = nullptr;
  }
  sh.peerP[rank][0] = sh.xP[0];
  sh.peerP[rank][1] = sh.xP[1];
  sh.peerFB[rank][0] = sh.xFB[0];
  sh.peerFB[rank][1] = sh.xFB[1];
  sh.peerRec[rank] = sh.rec;
  sh.peerBar[rank] = sh.bar;
}

void shard_export(const ShardGraph& sh, ShardHandles& out) {
  void* bufs[6] = {sh.xP[0], sh.xP[1], sh.xFB[0], sh.xFB[1], sh.rec, sh.bar};
  for (int k = 0; k < 6; ++k) CYC_CUDA(cudaIpcGetMemHandle(&out.h[k], bufs[k]));
  out.m_local = sh.m_local;
  out.world = sh.world;
  out.rank = sh.rank;
}

void shard_connect_ipc(ShardGraph& sh, const ShardHandles* all, int world) {
  if (world != sh.world) throw Error(CYC_E_CONTRACT, "shard connect: world size mismatch");
  uint64_t m = 0;
  for (int p = 0; p < world; ++p) {
    if (all[p].world != world || all[p].rank != p) throw Error(CYC_E_CONTRACT, "shard connect: handles out of order");
    m += all[p].m_local;
  }
  sh.m_global = m;
  for (int p = 0; p < world; ++p) {
    if (p == sh.rank) continue;
    void* m[6];
    for (int k = 0; k < 6; ++k) {
      CYC_CUDA(cudaIpcOpenMemHandle(&m[k], all[p].h[k], cudaIpcMemLazyEnablePeerAccess));
      sh.opened.push_back(m[k]);
    }
    sh.peerP[p][0] = static_cast<uint32_t*>(m[0]);
    sh.peerP[p][1] = static_cast<uint32_t*>(m[1]);
    sh.peerFB[p][0] = static_cast<uint32_t*>(m[2]);
    sh.peerFB[p][1] = static_cast<uint32_t*>(m[3]);
    sh.peerRec[p] = static_cast<ShardRec*>(m[4]);
    sh.peerBar[p] = static_cast<unsigned long long*>(m[5]);
  }
}

void shard_connect_local(ShardGraph* const* shards, int world) {
  const int dev0 = shards[0]->device;
  bool same = true;
  uint64_t m = 0;
  for (int i = 0; i < world; ++i) {
    if (shards[i]->world != world || shards[i]->rank != i) throw Error(CYC_E_CONTRACT, "shard connect: ranks out of order");
    same &= shards[i]->device == dev0;
    m += shards[i]->m_local;
  }
  for (int i = 0; i < world; ++i) {
    ShardGraph& a = *shards[i];
    a.emulated = same && world > 1;
    a.m_global = m;
    for (int j = 0; j < world; ++j) {
      const ShardGraph& b = *shards[j];
      if (!same && i != j) {
        int ok = 0;
        CYC_CUDA(cudaDeviceCanAccessPeer(&ok, a.device, b.device));
        if (!ok) throw Error(CYC_E_RESOURCE, "shard connect: devices without peer access");
        CYC_CUDA(cudaSetDevice(a.device));
        const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError(); else CYC_CUDA(e);
      }
      a.peerP[j][0] = b.xP[0];
      a.peerP[j][1] = b.xP[1];
      a.peerFB[j][0] = b.xFB[0];
      a.peerFB[j][1] = b.xFB[1];
      a.peerRec[j] = b.rec;
      a.peerBar[j] = b.bar;
    }
  }
  CYC_CUDA(cudaSetDevice(dev0));
}

void shard_run(ShardGraph* const* shards, int k, const uint64_t* acc_words, int early_exit, int mode,
               unsigned long long max_iterations, unsigned long long max_steps, uint32_t alpha, unsigned long long cap,
               cudaStream_t const* streams, cudaEvent_t, cudaEvent_t, RunOut* outs) {
  std::vector<ShardRunIn> in(k);
  for (int i = 0; i < k; ++i) {
    ShardGraph& sh = *shards[i];
    cudaStream_t s = streams[i];
    CYC_CUDA(cudaSetDevice(sh.device));
    for (int p = 0; p < sh.world; ++p)
      if (!sh.peerP[p][0]) throw Error(CYC_E_CONTRACT, "run_map: shard not connected to all peers");
    // F in storage order (u32 words), from the call's or the graph's accepting words
    const size_t nw64 = ((size_t)sh.n + 63) / 64;
    DevBuf f((nw64 + 1) * 8, s);
    CYC_CUDA(cudaMemsetAsync(f.p, 0, f.bytes, s));
    CYC_CUDA(cudaMemcpyAsync(f.p, acc_words ? (const void*)acc_words : sh.acc.p, nw64 * 8, cudaMemcpyDefault, s));
    // trim the tail like load_acc (bits >= n must be clear)
    if (sh.n & 63u) {
      uint64_t last = 0;
      CYC_CUDA(cudaMemcpyAsync(&last, f.as<uint64_t>() + (sh.n >> 6), 8, cudaMemcpyDeviceToHost, s));
      CYC_CUDA(cudaStreamSynchronize(s));
      last &= (1ull << (sh.n & 63u)) - 1ull;
      CYC_CUDA(cudaMemcpyAsync(f.as<uint64_t>() + (sh.n >> 6), &last, 8, cudaMemcpyHostToDevice, s));
    }
    if (sh.relabel) {
      permute_bits(f.as<uint32_t>(), sh.orig.as<uint32_t>(), sh.n, sh.ws.F.as<uint32_t>(), s);
    } else {
      CYC_CUDA(cudaMemcpyAsync(sh.ws.F.p, f.p, nw64 * 8, cudaMemcpyDeviceToDevice, s));
    }
    CYC_CUDA(cudaStreamSynchronize(s));
    ShardRunIn& r = in[i];
    std::memset(&r, 0, sizeof r);
    r.device = sh.device;
    r.s = s;
    r.push = &sh.push;
    r.gath = &sh.gath;
    r.orig = sh.relabel ? sh.orig.as<uint32_t>() : nullptr;
    r.perm = sh.relabel ? sh.perm.as<uint32_t>() : nullptr;
    r.sdesc = sh.sdesc.as<uint4>();
    r.sell = sh.sell.as<uint32_t>();
    r.hcol = sh.hcol.as<uint32_t>();
    r.hrow = sh.hrow.as<uint32_t>();
    r.n_hchunks = sh.n_hchunks;
    r.ws = &sh.ws;
    for (int b = 0; b < 2; ++b) {
      r.P[b] = sh.xP[b];
      r.FB[b] = sh.xFB[b];
    }
    r.bigm = sh.ws.bigm.as<uint32_t>();  // push degree > kBigDeg over this rank's push rows
    r.n = sh.n;
    r.m_global = sh.m_global;
    r.world = sh.world;
    r.rank = sh.rank;
    r.row_lo = sh.row_lo;
    r.row_hi = sh.row_hi;
    std::memcpy(r.peerP, sh.peerP, sizeof r.peerP);
    std::memcpy(r.peerFB, sh.peerFB, sizeof r.peerFB);
    r.rec = sh.rec;
    std::memcpy(r.peerRec, sh.peerRec, sizeof r.peerRec);
    r.bar = sh.bar;
    std::memcpy(r.peerBar, sh.peerBar, sizeof r.peerBar);
    r.bar_base = sh.bars_done;
  }
  launch_map_run_shards(in.data(), k, shards[0]->emulated, early_exit, mode, max_iterations, max_steps, alpha, cap,
                        outs);
  for (int i = 0; i < k; ++i) shards[i]->bars_done = outs[i].res[kResBars];
}

void shard_values(const ShardGraph& sh, int cur, uint32_t* dst, cudaStream_t s) {
  if (!sh.n) return;
  k_shard_values<<<grid_for(sh.n, 256, 8), 256, 0, s>>>(sh.xP[cur], sh.relabel ? sh.orig.as<uint32_t>() : nullptr,
                                                        sh.n, dst);
  CYC_LAUNCHED();
}

}  // namespace cyc
