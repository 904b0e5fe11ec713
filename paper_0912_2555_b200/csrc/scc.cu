// scc.cu — K2: keep exactly the vertices of cyclic SCCs that hold an
// accepting vertex, renumber them in ascending order and keep every edge with
// both endpoints kept (reference graph.cpp:190-221; Tarjan at :125-186).
//
// Tarjan is inherently sequential. The kept set is set-defined, so any
// correct SCC decomposition reproduces it; on the device we use:
//   1. reachability pruning: a kept vertex is reachable from F and reaches F
//      (both computed by dense OR-propagation over the CSR pair);
//   2. trimming: a vertex with no active predecessor or successor is a
//      trivial acyclic SCC;
//   3. max-colour rounds (Orzan / Barnat et al.'s coloring): colour[v] = max
//      active id reaching v; each root r (colour[r] == r) owns the SCC of
//      vertices with colour r that reach r through colour-r vertices.
// Every SCC found is kept iff it holds an accepting vertex and is cyclic
// (size >= 2 or a self-loop). Passes are dense; convergence flags are read
// by the host every few passes.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "scc.cuh"

namespace cyc {

namespace {

constexpr int kT = 256;

__device__ __forceinline__ bool accb(const uint64_t* acc, uint32_t v) {
  return (acc[v >> 6] >> (v & 63u)) & 1ull;
}

__global__ void k_reach_init(uint32_t n, const uint64_t* __restrict__ acc, uint8_t* fw, uint8_t* bw) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    uint8_t a = accb(acc, v) ? 1 : 0;
    fw[v] = a;
    bw[v] = a;
  }
}

// flag |= 1 if any vertex newly reached. rows: for fw use the gather index
// (predecessors), for bw the snapshot rows (successors).
// Heavy rows (degree > heavy) are left to the *_chunks kernels, one warp per
// 256-edge chunk (R-MAT hubs would otherwise serialise a pass on one thread).
__global__ void k_reach(uint32_t n, const uint32_t* __restrict__ off, const uint32_t* __restrict__ col,
                        uint32_t heavy, uint8_t* mark, uint32_t* flag) {
  bool ch = false;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (mark[v] || off[v + 1] - off[v] > heavy) continue;
    for (uint32_t i = off[v]; i < off[v + 1]; ++i) {
      if (((volatile uint8_t*)mark)[col[i]]) {
        mark[v] = 1;
        ch = true;
        break;
      }
    }
  }
  if (ch) *flag = 1;
}

__global__ void k_reach_chunks(const uint4* __restrict__ chunks, uint32_t nch,
                               const uint32_t* __restrict__ col, uint8_t* mark, uint32_t* flag) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t c = gw; c < nch; c += nw) {
    const uint4 ch = chunks[c];
    if (((volatile uint8_t*)mark)[ch.x]) continue;
    bool hit = false;
    for (uint32_t i = ch.y + lane; i < ch.z; i += 32u) hit |= ((volatile uint8_t*)mark)[col[i]] != 0;
    if (__any_sync(kFull, hit) && lane == 0) {
      mark[ch.x] = 1;
      *flag = 1;
    }
  }
}

__global__ void k_and(uint32_t n, const uint8_t* fw, const uint8_t* bw, uint8_t* active) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    active[v] = fw[v] & bw[v];
}

__device__ __forceinline__ bool any_active(const uint32_t* off, const uint32_t* col, uint32_t v,
                                           const uint8_t* active) {
  for (uint32_t i = off[v]; i < off[v + 1]; ++i)
    if (((volatile const uint8_t*)active)[col[i]]) return true;
  return false;
}

__global__ void k_trim(uint32_t n, const uint32_t* __restrict__ soff, const uint32_t* __restrict__ scol,
                       const uint32_t* __restrict__ goff, const uint32_t* __restrict__ gcol,
                       uint8_t* active, uint32_t* flag) {
  bool ch = false;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (!active[v]) continue;
    if (!any_active(goff, gcol, v, active) || !any_active(soff, scol, v, active)) {
      active[v] = 0;
      ch = true;
    }
  }
  if (ch) *flag = 1;
}

__global__ void k_color_init(uint32_t n, const uint8_t* active, uint32_t* color, uint8_t* inscc) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    color[v] = active[v] ? v : 0xFFFFFFFFu;
    inscc[v] = 0;
  }
}

__global__ void k_color_prop(uint32_t n, const uint32_t* __restrict__ goff,
                             const uint32_t* __restrict__ gcol, uint32_t heavy, const uint8_t* active,
                             uint32_t* color, uint32_t* flag) {
  bool ch = false;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (!active[v] || goff[v + 1] - goff[v] > heavy) continue;
    uint32_t c = ((volatile uint32_t*)color)[v], best = c;
    for (uint32_t i = goff[v]; i < goff[v + 1]; ++i) {
      uint32_t u = gcol[i];
      if (active[u]) best = max(best, ((volatile uint32_t*)color)[u]);
    }
    if (best != c) {
      atomicMax(color + v, best);
      ch = true;
    }
  }
  if (ch) *flag = 1;
}

__global__ void k_color_chunks(const uint4* __restrict__ chunks, uint32_t nch,
                               const uint32_t* __restrict__ gcol, const uint8_t* active,
                               uint32_t* color, uint32_t* flag) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t c = gw; c < nch; c += nw) {
    const uint4 ch = chunks[c];
    if (!active[ch.x]) continue;
    uint32_t best = 0;
    for (uint32_t i = ch.y + lane; i < ch.z; i += 32u) {
      const uint32_t u = gcol[i];
      if (active[u]) best = max(best, ((volatile uint32_t*)color)[u]);
    }
    best = __reduce_max_sync(kFull, best);
    if (lane == 0 && best > ((volatile uint32_t*)color)[ch.x]) {
      atomicMax(color + ch.x, best);
      *flag = 1;
    }
  }
}

__global__ void k_roots(uint32_t n, const uint8_t* active, const uint32_t* color, uint8_t* inscc,
                        uint32_t* rsize, uint32_t* rflag) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (active[v] && color[v] == v) {
      inscc[v] = 1;
      rsize[v] = 0;
      rflag[v] = 0;
    }
  }
}

__global__ void k_bw_color(uint32_t n, const uint32_t* __restrict__ soff,
                           const uint32_t* __restrict__ scol, uint32_t heavy, const uint8_t* active,
                           const uint32_t* color, uint8_t* inscc, uint32_t* flag) {
  bool ch = false;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (!active[v] || inscc[v] || soff[v + 1] - soff[v] > heavy) continue;
    const uint32_t c = color[v];
    for (uint32_t i = soff[v]; i < soff[v + 1]; ++i) {
      uint32_t w = scol[i];
      if (active[w] && color[w] == c && ((volatile uint8_t*)inscc)[w]) {
        inscc[v] = 1;
        ch = true;
        break;
      }
    }
  }
  if (ch) *flag = 1;
}

__global__ void k_bw_chunks(const uint4* __restrict__ chunks, uint32_t nch,
                            const uint32_t* __restrict__ scol, const uint8_t* active,
                            const uint32_t* color, uint8_t* inscc, uint32_t* flag) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t c = gw; c < nch; c += nw) {
    const uint4 ch = chunks[c];
    const uint32_t v = ch.x;
    if (!active[v] || ((volatile uint8_t*)inscc)[v]) continue;
    const uint32_t cv = color[v];
    bool hit = false;
    for (uint32_t i = ch.y + lane; i < ch.z; i += 32u) {
      const uint32_t w = scol[i];
      hit |= active[w] && color[w] == cv && ((volatile uint8_t*)inscc)[w];
    }
    if (__any_sync(kFull, hit) && lane == 0) {
      inscc[v] = 1;
      *flag = 1;
    }
  }
}

__device__ bool has_self_loop(const uint32_t* off, const uint32_t* col, uint32_t v) {
  uint32_t lo = off[v], hi = off[v + 1];
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    uint32_t c = col[mid];
    if (c == v) return true;
    if (c < v) lo = mid + 1; else hi = mid;
  }
  return false;
}

__global__ void k_scc_stats(uint32_t n, const uint32_t* __restrict__ soff,
                            const uint32_t* __restrict__ scol, const uint64_t* __restrict__ acc,
                            const uint8_t* inscc, const uint32_t* color, uint32_t* rsize,
                            uint32_t* rflag) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (!inscc[v]) continue;
    uint32_t r = color[v];
    atomicAdd(rsize + r, 1u);
    uint32_t f = (accb(acc, v) ? 1u : 0u) | (has_self_loop(soff, scol, v) ? 2u : 0u);
    if (f) atomicOr(rflag + r, f);
  }
}

__global__ void k_scc_apply(uint32_t n, const uint32_t* color, const uint32_t* rsize,
                            const uint32_t* rflag, uint8_t* inscc, uint8_t* active, uint8_t* keep,
                            uint32_t* flag) {
  bool any = false;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (inscc[v]) {
      uint32_t r = color[v];
      keep[v] = (rflag[r] & 1u) && (rsize[r] >= 2u || (rflag[r] & 2u));
      active[v] = 0;
      inscc[v] = 0;
    }
    any |= active[v] != 0;
  }
  if (any) *flag = 1;
}

__global__ void k_keep_acc32(uint32_t n, const uint8_t* keep, const uint64_t* __restrict__ acc,
                             uint32_t* k32) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    k32[v] = keep[v] && accb(acc, v);
}

__global__ void k_list_from_flags(uint32_t n, const uint32_t* flags, const uint32_t* pos, uint32_t* out) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (flags[v]) out[pos[v]] = v;
}

// ---- compaction of the kept subgraph
__global__ void k_keep32(uint32_t n, const uint8_t* keep, uint32_t* k32) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    k32[v] = keep[v];
}

__global__ void k_kept_list(uint32_t n, const uint8_t* keep, const uint32_t* newid, uint32_t* kept) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (keep[v]) kept[newid[v]] = v;
}

// One warp per kept row (rows of R-MAT hubs are long): count, then an
// order-preserving ballot compaction of the kept columns.
__global__ void k_filter_count(uint32_t k, const uint32_t* kept, const uint32_t* __restrict__ off,
                               const uint32_t* __restrict__ col, const uint8_t* keep, uint32_t* cnt) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t a = gw; a < k; a += nw) {
    const uint32_t v = kept[a];
    uint32_t c = 0;
    for (uint32_t i = off[v] + lane; i < off[v + 1]; i += 32u) c += keep[col[i]];
    c = __reduce_add_sync(kFull, c);
    if (lane == 0) cnt[a] = c;
  }
}

__global__ void k_filter_fill(uint32_t k, const uint32_t* kept, const uint32_t* __restrict__ off,
                              const uint32_t* __restrict__ col, const uint8_t* keep,
                              const uint32_t* newid, const uint32_t* noff, uint32_t* ncol) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t a = gw; a < k; a += nw) {
    const uint32_t v = kept[a];
    uint32_t o = noff[a];
    const uint32_t b = off[v], e = off[v + 1];
    for (uint32_t i0 = b; i0 < e; i0 += 32u) {
      const uint32_t i = i0 + lane;
      const uint32_t w = i < e ? col[i] : 0u;
      const bool in = i < e && keep[w];
      const uint32_t bal = __ballot_sync(kFull, in);
      if (in) ncol[o + __popc(bal & lanemask_lt())] = newid[w];
      o += __popc(bal);
    }
  }
}

__global__ void k_pack_acc(uint32_t k, const uint32_t* kept, const uint64_t* __restrict__ acc,
                           uint64_t* out) {
  const uint32_t words = (k + 63) / 64;
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x) {
    uint64_t bits = 0;
    for (uint32_t j = 0; j < 64; ++j) {
      uint32_t a = w * 64 + j;
      if (a < k && accb(acc, kept[a])) bits |= 1ull << j;
    }
    out[w] = bits;
  }
}

// Runs `pass` until it leaves the flag clear; returns the number of passes.
template <class F>
int until_stable(uint32_t* dflag, cudaStream_t s, F&& pass) {
  int k = 0;
  for (;;) {
    uint32_t h = 0;
    CYC_CUDA(cudaMemsetAsync(dflag, 0, 4, s));
    pass();
    ++k;
    CYC_CUDA(cudaMemcpyAsync(&h, dflag, 4, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
    if (!h) break;
  }
  return k;
}

struct SccLog {
  bool on = std::getenv("CYC_DEBUG_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what, int passes) {
    if (!on) return;
    auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[cyc scc] %-12s passes %5d %9.3f ms\n", what, passes,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

void filter_csr(const DevCsr& in, const uint8_t* keep, const uint32_t* newid, const uint32_t* kept,
                uint32_t k, cudaStream_t s, DevCsr& out) {
  out.n = k;
  out.off.alloc(((size_t)k + 1) * 4, s);
  DevBuf cnt(((size_t)k + 1) * 4, s), scratch;
  if (k) {
    k_filter_count<<<sm_count() * 8, kT, 0, s>>>(k, kept, in.o(), in.c(), keep, cnt.as<uint32_t>());
    CYC_LAUNCHED();
  }
  exclusive_scan(cnt.as<uint32_t>(), out.off.as<uint32_t>(), k, nullptr, s, scratch);
  uint32_t m = 0;
  CYC_CUDA(cudaMemcpyAsync(&m, out.off.as<uint32_t>() + k, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  out.m = m;
  out.col.alloc(((size_t)m + 1) * 4, s);
  if (k) {
    k_filter_fill<<<sm_count() * 8, kT, 0, s>>>(k, kept, in.o(), in.c(), keep, newid,
                                                out.off.as<uint32_t>(), out.col.as<uint32_t>());
    CYC_LAUNCHED();
  }
}

}  // namespace

void scc_keep_mask(const DevCsr& snap, const DevCsr& gath, const uint64_t* acc, cudaStream_t s,
                   uint8_t* keep) {
  const uint32_t n = snap.n;
  CYC_CUDA(cudaMemsetAsync(keep, 0, (size_t)n + 1, s));
  if (!n) return;
  DevBuf fw((size_t)n + 1, s), bw((size_t)n + 1, s), active((size_t)n + 1, s), inscc((size_t)n + 1, s);
  DevBuf color(((size_t)n + 1) * 4, s), rsize(((size_t)n + 1) * 4, s), rflag(((size_t)n + 1) * 4, s);
  DevBuf flag(16, s);
  uint32_t* f = flag.as<uint32_t>();
  const uint32_t grid = grid_for(n, kT, 8);
  SccLog lg;
  k_reach_init<<<grid, kT, 0, s>>>(n, acc, fw.as<uint8_t>(), bw.as<uint8_t>());
  CYC_LAUNCHED();
  const uint32_t hg = gath.heavy_deg ? gath.heavy_deg : kNone, hs = snap.heavy_deg ? snap.heavy_deg : kNone;
  const uint32_t cgrid = sm_count() * 8;
  int np = until_stable(f, s, [&] {
    k_reach<<<grid, kT, 0, s>>>(n, gath.o(), gath.c(), hg, fw.as<uint8_t>(), f);
    CYC_LAUNCHED();
    if (gath.n_heavy_chunks) {
      k_reach_chunks<<<cgrid, kT, 0, s>>>(gath.heavy.as<uint4>(), gath.n_heavy_chunks, gath.c(),
                                          fw.as<uint8_t>(), f);
      CYC_LAUNCHED();
    }
  });
  lg.mark("reach-fw", np);
  np = until_stable(f, s, [&] {
    k_reach<<<grid, kT, 0, s>>>(n, snap.o(), snap.c(), hs, bw.as<uint8_t>(), f);
    CYC_LAUNCHED();
    if (snap.n_heavy_chunks) {
      k_reach_chunks<<<cgrid, kT, 0, s>>>(snap.heavy.as<uint4>(), snap.n_heavy_chunks, snap.c(),
                                          bw.as<uint8_t>(), f);
      CYC_LAUNCHED();
    }
  });
  lg.mark("reach-bw", np);
  k_and<<<grid, kT, 0, s>>>(n, fw.as<uint8_t>(), bw.as<uint8_t>(), active.as<uint8_t>());
  CYC_LAUNCHED();
  int rounds = 0;
  for (;;) {
    ++rounds;
    np = until_stable(f, s, [&] {
      k_trim<<<grid, kT, 0, s>>>(n, snap.o(), snap.c(), gath.o(), gath.c(), active.as<uint8_t>(), f);
      CYC_LAUNCHED();
    });
    lg.mark("trim", np);
    k_color_init<<<grid, kT, 0, s>>>(n, active.as<uint8_t>(), color.as<uint32_t>(), inscc.as<uint8_t>());
    CYC_LAUNCHED();
    np = until_stable(f, s, [&] {
      k_color_prop<<<grid, kT, 0, s>>>(n, gath.o(), gath.c(), hg, active.as<uint8_t>(),
                                       color.as<uint32_t>(), f);
      CYC_LAUNCHED();
      if (gath.n_heavy_chunks) {
        k_color_chunks<<<cgrid, kT, 0, s>>>(gath.heavy.as<uint4>(), gath.n_heavy_chunks, gath.c(),
                                            active.as<uint8_t>(), color.as<uint32_t>(), f);
        CYC_LAUNCHED();
      }
    });
    lg.mark("color", np);
    k_roots<<<grid, kT, 0, s>>>(n, active.as<uint8_t>(), color.as<uint32_t>(), inscc.as<uint8_t>(),
                                rsize.as<uint32_t>(), rflag.as<uint32_t>());
    CYC_LAUNCHED();
    np = until_stable(f, s, [&] {
      k_bw_color<<<grid, kT, 0, s>>>(n, snap.o(), snap.c(), hs, active.as<uint8_t>(),
                                     color.as<uint32_t>(), inscc.as<uint8_t>(), f);
      CYC_LAUNCHED();
      if (snap.n_heavy_chunks) {
        k_bw_chunks<<<cgrid, kT, 0, s>>>(snap.heavy.as<uint4>(), snap.n_heavy_chunks, snap.c(),
                                         active.as<uint8_t>(), color.as<uint32_t>(),
                                         inscc.as<uint8_t>(), f);
        CYC_LAUNCHED();
      }
    });
    lg.mark("bw-color", np);
    k_scc_stats<<<grid, kT, 0, s>>>(n, snap.o(), snap.c(), acc, inscc.as<uint8_t>(),
                                    color.as<uint32_t>(), rsize.as<uint32_t>(), rflag.as<uint32_t>());
    CYC_LAUNCHED();
    uint32_t any = 0;
    CYC_CUDA(cudaMemsetAsync(f, 0, 4, s));
    k_scc_apply<<<grid, kT, 0, s>>>(n, color.as<uint32_t>(), rsize.as<uint32_t>(),
                                    rflag.as<uint32_t>(), inscc.as<uint8_t>(), active.as<uint8_t>(),
                                    keep, f);
    CYC_LAUNCHED();
    CYC_CUDA(cudaMemcpyAsync(&any, f, 4, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
    if (!any) break;
  }
}

uint32_t scc_cyclic_accepting(const DevCsr& snap, const DevCsr& gath, const uint64_t* acc,
                              cudaStream_t s, DevBuf& list) {
  const uint32_t n = snap.n;
  DevBuf keep((size_t)n + 1, s), f32(((size_t)n + 1) * 4, s), pos(((size_t)n + 2) * 4, s), scratch;
  scc_keep_mask(snap, gath, acc, s, keep.as<uint8_t>());
  if (n) {
    k_keep_acc32<<<grid_for(n, kT, 8), kT, 0, s>>>(n, keep.as<uint8_t>(), acc, f32.as<uint32_t>());
    CYC_LAUNCHED();
  }
  exclusive_scan(f32.as<uint32_t>(), pos.as<uint32_t>(), n, nullptr, s, scratch);
  uint32_t k = 0;
  CYC_CUDA(cudaMemcpyAsync(&k, pos.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  list.alloc(((size_t)k + 1) * 4, s);
  if (n && k) {
    k_list_from_flags<<<grid_for(n, kT, 8), kT, 0, s>>>(n, f32.as<uint32_t>(), pos.as<uint32_t>(),
                                                        list.as<uint32_t>());
    CYC_LAUNCHED();
  }
  CYC_CUDA(cudaStreamSynchronize(s));
  return k;
}

void restrict_graph(const DevCsr& snap, const DevCsr& gath, const uint64_t* acc, cudaStream_t s,
                    DevCsr& out_snap, DevCsr& out_gath, DevBuf& out_acc, DevBuf& out_kept) {
  const uint32_t n = snap.n;
  DevBuf keep((size_t)n + 1, s), k32(((size_t)n + 1) * 4, s), newid(((size_t)n + 2) * 4, s), scratch;
  scc_keep_mask(snap, gath, acc, s, keep.as<uint8_t>());
  if (n) {
    k_keep32<<<grid_for(n, kT, 8), kT, 0, s>>>(n, keep.as<uint8_t>(), k32.as<uint32_t>());
    CYC_LAUNCHED();
  }
  exclusive_scan(k32.as<uint32_t>(), newid.as<uint32_t>(), n, nullptr, s, scratch);
  uint32_t k = 0;
  CYC_CUDA(cudaMemcpyAsync(&k, newid.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  out_kept.alloc(((size_t)k + 1) * 4, s);
  if (n) {
    k_kept_list<<<grid_for(n, kT, 8), kT, 0, s>>>(n, keep.as<uint8_t>(), newid.as<uint32_t>(),
                                                  out_kept.as<uint32_t>());
    CYC_LAUNCHED();
  }
  filter_csr(snap, keep.as<uint8_t>(), newid.as<uint32_t>(), out_kept.as<uint32_t>(), k, s, out_snap);
  filter_csr(gath, keep.as<uint8_t>(), newid.as<uint32_t>(), out_kept.as<uint32_t>(), k, s, out_gath);
  const size_t words = ((size_t)k + 63) / 64;
  out_acc.alloc((words + 1) * 8, s);
  CYC_CUDA(cudaMemsetAsync(out_acc.p, 0, (words + 1) * 8, s));
  if (k) {
    k_pack_acc<<<grid_for(words, kT, 8), kT, 0, s>>>(k, out_kept.as<uint32_t>(), acc,
                                                     out_acc.as<uint64_t>());
    CYC_LAUNCHED();
  }
  CYC_CUDA(cudaStreamSynchronize(s));
}

}  // namespace cyc
