// scc.cu — K2: keep exactly the vertices of cyclic SCCs that hold an
// accepting vertex, renumber them in ascending order and keep every edge with
// both endpoints kept (reference graph.cpp:190-221; Tarjan at :125-186).
//
// Tarjan is inherently sequential. The kept set is set-defined, so any
// correct SCC decomposition reproduces it; on the device we use:
//   0. orientation: colours flow along whichever of the two relations (the
//      snapshot relation or its reverse) has mostly ascending edges, so a
//      vertex's ancestors tend to have smaller ids and most SCCs are found in
//      the first colouring round (config 2 transposed: 65 rounds -> 1);
//   1. reachability pruning: a kept vertex is reachable from F and reaches F;
//   2. trimming: a vertex with no active predecessor or successor is a
//      trivial acyclic SCC (dense passes, usually two);
//   3. max-colour rounds (Orzan / Barnat et al.'s coloring): colour[v] = max
//      active id reaching v; each root r (colour[r] == r) owns the SCC of
//      vertices with colour r that reach r through colour-r vertices.
// Steps 1 and 3 are closures computed by the frontier engine (frontier.cuh):
// one persistent kernel per closure, levels touch only changed vertices.
// Every SCC found is kept iff it holds an accepting vertex and is cyclic
// (size >= 2 or a self-loop).
#include <chrono>
#include <pthread.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "frontier.cuh"
#include "scc.cuh"

namespace cyc {

namespace {

constexpr int kT = 256;
constexpr uint32_t kNoColor = 0xFFFFFFFFu;  // inactive: never raised, never equal

__device__ __forceinline__ bool accb(const uint64_t* acc, uint32_t v) {
  return (acc[v >> 6] >> (v & 63u)) & 1ull;
}
__device__ __forceinline__ bool bit(const uint32_t* b, uint32_t v) { return (b[v >> 5] >> (v & 31u)) & 1u; }

// ---- frontier ops
struct OpReach {  // mark = vertices reached so far (seeds included); act: optional vertex filter
  uint32_t* mark;
  const uint8_t* act = nullptr;
  __device__ uint32_t token(uint32_t) const { return 0u; }
  __device__ bool relax(uint32_t, uint32_t, uint32_t w, uint32_t) const {
    return (!act || act[w]) && test_and_set_bit(mark, w);
  }
};

struct OpColor {  // colour[w] = max(colour[w], colour[u]) along the relation
  uint32_t* color;
  uint32_t* stamp;  // level + 1 at which w was last queued (zeroed per round)
  __device__ uint32_t token(uint32_t u) const { return __ldcg(color + u); }
  __device__ bool relax(uint32_t, uint32_t tok, uint32_t w, uint32_t L) const {
    if (__ldcg(color + w) >= tok) return false;  // also every inactive w
    if (atomicMax(color + w, tok) >= tok) return false;
    return atomicMax(stamp + w, L + 1u) < L + 1u;
  }
};

struct OpSameColor {  // backward reach from roots through equal colours
  const uint32_t* color;
  uint32_t* inscc;
  __device__ uint32_t token(uint32_t w) const { return __ldcg(color + w); }
  __device__ bool relax(uint32_t, uint32_t tok, uint32_t v, uint32_t) const {
    // membership first: the bitmap is L2-resident, colours are not
    return !bit(inscc, v) && __ldcg(color + v) == tok && test_and_set_bit(inscc, v);
  }
};

struct SeedBits {
  const uint32_t* b;
  __device__ bool operator()(uint32_t v) const { return bit(b, v); }
};
struct SeedActive {
  const uint8_t* a;
  __device__ bool operator()(uint32_t v) const { return a[v] != 0; }
};
struct SeedRoots {
  const uint32_t* color;
  __device__ bool operator()(uint32_t v) const { return color[v] == v + 1u; }
};

// ---- dense kernels
// Light rows one per lane, rows longer than 64 by the whole warp.
__global__ void k_count_ascending(uint32_t n, const uint32_t* __restrict__ off, const uint32_t* __restrict__ col,
                                  unsigned long long* cnt) {
  const uint32_t lane = lane_id();
  uint32_t c = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; v0 < n; v0 += stride) {
    const uint32_t v = v0 + lane;
    const uint32_t b = v < n ? off[v] : 0u, e = v < n ? off[v + 1] : 0u;
    const bool heavy = e - b > 64u;
    if (!heavy)
      for (uint32_t i = b; i < e; ++i) c += col[i] > v;
    for (uint32_t hb = __ballot_sync(kFull, heavy); hb; hb &= hb - 1u) {
      const uint32_t l = __ffs(hb) - 1u;
      const uint32_t hv = v0 + l, hb0 = __shfl_sync(kFull, b, l), he = __shfl_sync(kFull, e, l);
      for (uint32_t i = hb0 + lane; i < he; i += 32u) c += col[i] > hv;
    }
  }
  c = __reduce_add_sync(kFull, c);
  if (lane == 0 && c) atomicAdd(cnt, (unsigned long long)c);
}

__global__ void k_and_bits(uint32_t n, const uint32_t* fw, const uint32_t* bw, uint8_t* active) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    active[v] = bit(fw, v) & bit(bw, v);
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

// FW-BW from one pivot before colouring: the active vertex of largest total
// degree (an R-MAT hub, inside the giant SCC) — its SCC is fw ∩ bw of two
// bitmap reach closures restricted to the active vertices, instead of
// several max-colour passes that gather 4 B colours of every vertex.
__global__ void k_pivot(uint32_t n, const uint32_t* __restrict__ aoff, const uint32_t* __restrict__ boff,
                        const uint8_t* active, unsigned long long* best) {
  unsigned long long m = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (active[v]) {
      const unsigned long long d = (unsigned long long)(aoff[v + 1] - aoff[v]) + (boff[v + 1] - boff[v]);
      m = max(m, (d << 32) | v);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, (unsigned long long)__shfl_xor_sync(kFull, m, o));
  if ((threadIdx.x & 31u) == 0 && m) atomicMax(best, m);
}

__global__ void k_and_act(uint32_t n, const uint8_t* active, const uint32_t* fw, uint8_t* out) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    out[v] = active[v] && bit(fw, v);
}

__global__ void k_pivot_scc(uint32_t n, const uint32_t* fw, const uint32_t* bw, const uint8_t* active,
                            uint32_t pivot, uint32_t* inscc, uint32_t* color) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; v0 < n; v0 += stride) {
    const uint32_t v = v0 + lane_id();
    const bool in = v < n && active[v] && bit(fw, v) && bit(bw, v);
    const uint32_t word = __ballot_sync(kFull, in);
    if (lane_id() == 0) inscc[v0 >> 5] = word;
    if (in) color[v] = pivot + 1u;
  }
}

__global__ void k_color_init(uint32_t n, const uint8_t* active, uint32_t* color) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    color[v] = active[v] ? v + 1u : kNoColor;
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

// per root r (colour r+1): size and "has an accepting vertex"; lanes sharing
// a root (one giant SCC on R-MAT) combine before the atomics. The self-loop
// test only matters for singleton SCCs, i.e. the root alone: k_scc_apply
// does it there (one binary search per singleton, not one per vertex).
__global__ void k_scc_stats(uint32_t n, const uint64_t* __restrict__ acc, const uint32_t* inscc,
                            const uint32_t* color, uint32_t* rsize, uint32_t* rflag) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; v0 < n; v0 += stride) {
    const uint32_t v = v0 + lane_id();
    const bool in = v < n && bit(inscc, v);
    const uint32_t r = in ? color[v] - 1u : kNone;
    const uint32_t f = in && accb(acc, v) ? 1u : 0u;
    const uint32_t peers = __match_any_sync(kFull, r);
    const uint32_t fo = __reduce_or_sync(peers, f);
    if (in && (peers & lanemask_lt()) == 0) {  // lowest lane of the group
      atomicAdd(rsize + r, (uint32_t)__popc(peers));
      if (fo) atomicOr(rflag + r, fo);
    }
  }
}

__global__ void k_scc_apply(uint32_t n, const uint32_t* __restrict__ soff, const uint32_t* __restrict__ scol,
                            const uint32_t* color, uint32_t* rsize, uint32_t* rflag, const uint32_t* inscc,
                            uint8_t* active, uint8_t* keep, uint32_t* flag) {
  bool any = false;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (bit(inscc, v)) {
      const uint32_t r = color[v] - 1u;
      const uint32_t sz = rsize[r];
      keep[v] = (rflag[r] & 1u) && (sz >= 2u || has_self_loop(soff, scol, v));
      active[v] = 0;
    }
    any |= active[v] != 0;
  }
  if (any) *flag = 1;
}

// ---- dense pull passes (Gauss-Seidel) with epoch stamps: ep[v] = p when v
// changed in pass p; *cnt += changes. Heavy rows (deg > heavy) are done by the
// *_chunks kernels, one warp per 256-edge chunk.
__device__ __forceinline__ void count_changes(uint32_t c, unsigned long long* cnt) {
  c = __reduce_add_sync(kFull, c);
  if ((threadIdx.x & 31u) == 0 && c) atomicAdd(cnt, (unsigned long long)c);
}

__global__ void k_reach_pull(uint32_t n, const uint32_t* __restrict__ off, const uint32_t* __restrict__ col,
                             uint32_t heavy, uint32_t* mark, uint8_t* ep, uint8_t p, unsigned long long* cnt,
                             const uint8_t* act) {
  uint32_t c = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; w0 < n; w0 += stride) {
    const uint32_t w = w0 + lane_id();
    if (w >= n || bit(mark, w) || (act && !act[w]) || off[w + 1] - off[w] > heavy) continue;
    for (uint32_t i = off[w]; i < off[w + 1]; ++i) {
      if (bit(mark, col[i])) {
        atomicOr(mark + (w >> 5), 1u << (w & 31u));
        ep[w] = p;
        ++c;
        break;
      }
    }
  }
  count_changes(c, cnt);
}

// Colour / same-colour heavy-row chunks (<= kHeavyChunk edges, 4 per lane)
// go two per warp with every load of a stage issued before any use: chunk
// descriptors, the rows' own state, 8 column indices per lane, 8 gathers.
// Config 3: same-colour chunks 3.6 -> 2.6 ms per pass; the colour pass stays
// at 8.4 ms (bound by 32 B random sectors from DRAM, ~2.4 TB/s), and the
// bitmap-only reach chunks were faster in the simple loop (1.2 vs 1.6 ms).
constexpr int kCB = 2;                          // chunks per warp iteration
constexpr int kCR = (int)(kHeavyChunk / 32u);   // column loads per lane per chunk

__device__ __forceinline__ void chunk_cols(const uint4 (&ch)[kCB], const bool (&live)[kCB],
                                           const uint32_t* __restrict__ col, uint32_t (&u)[kCB][kCR]) {
  const uint32_t lane = threadIdx.x & 31u;
#pragma unroll
  for (int b = 0; b < kCB; ++b)
#pragma unroll
    for (int r = 0; r < kCR; ++r) {
      const uint32_t i = ch[b].y + lane + 32u * r;
      u[b][r] = live[b] && i < ch[b].z ? __ldg(col + i) : kNone;
    }
}

__global__ void k_reach_pull_chunks(const uint4* __restrict__ chunks, uint32_t nch,
                                    const uint32_t* __restrict__ col, uint32_t* mark, uint8_t* ep, uint8_t p,
                                    unsigned long long* cnt, const uint8_t* act) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  uint32_t c = 0;
  for (uint32_t k = gw; k < nch; k += nw) {
    const uint4 ch = chunks[k];
    if (bit(mark, ch.x) || (act && !act[ch.x])) continue;
    bool hit = false;
    for (uint32_t i = ch.y + lane; i < ch.z; i += 32u) hit |= bit(mark, col[i]);
    if (__any_sync(kFull, hit) && lane == 0 && test_and_set_bit(mark, ch.x)) {
      ep[ch.x] = p;
      ++c;
    }
  }
  count_changes(c, cnt);
}

__global__ void k_color_pull(uint32_t n, const uint32_t* __restrict__ off, const uint32_t* __restrict__ col,
                             uint32_t heavy, uint32_t* color, uint8_t* ep, uint8_t p, unsigned long long* cnt) {
  uint32_t c = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; w0 < n; w0 += stride) {
    const uint32_t w = w0 + lane_id();
    if (w >= n) continue;
    const uint32_t own = ((volatile uint32_t*)color)[w];
    if (own == kNoColor || off[w + 1] - off[w] > heavy) continue;
    uint32_t best = own;
    for (uint32_t i = off[w]; i < off[w + 1]; ++i) {
      const uint32_t cu = ((volatile uint32_t*)color)[col[i]];
      if (cu != kNoColor) best = max(best, cu);
    }
    if (best > own) {
      atomicMax(color + w, best);
      ep[w] = p;
      ++c;
    }
  }
  count_changes(c, cnt);
}

__global__ void k_color_pull_chunks(const uint4* __restrict__ chunks, uint32_t nch,
                                    const uint32_t* __restrict__ col, uint32_t* color, uint8_t* ep, uint8_t p,
                                    unsigned long long* cnt) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  uint32_t c = 0;
  for (uint32_t k0 = gw * kCB; k0 < nch; k0 += nw * kCB) {
    uint4 ch[kCB];
    uint32_t own[kCB];
    bool live[kCB];
#pragma unroll
    for (int b = 0; b < kCB; ++b) ch[b] = k0 + b < nch ? chunks[k0 + b] : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int b = 0; b < kCB; ++b) own[b] = ch[b].z > ch[b].y ? __ldcg(color + ch[b].x) : kNoColor;
#pragma unroll
    for (int b = 0; b < kCB; ++b) live[b] = own[b] != kNoColor;
    uint32_t u[kCB][kCR];
    chunk_cols(ch, live, col, u);
    uint32_t best[kCB];
#pragma unroll
    for (int b = 0; b < kCB; ++b) {
      best[b] = 0;
#pragma unroll
      for (int r = 0; r < kCR; ++r) {
        const uint32_t cu = u[b][r] != kNone ? __ldcg(color + u[b][r]) : kNoColor;
        if (cu != kNoColor) best[b] = max(best[b], cu);
      }
      for (uint32_t i = ch[b].y + 32u * kCR + lane; live[b] && i < ch[b].z; i += 32u) {
        const uint32_t cu = __ldcg(color + col[i]);
        if (cu != kNoColor) best[b] = max(best[b], cu);
      }
    }
#pragma unroll
    for (int b = 0; b < kCB; ++b) {
      const uint32_t m = __reduce_max_sync(kFull, best[b]);
      if (lane == 0 && live[b] && m > own[b] && atomicMax(color + ch[b].x, m) < m) {
        ep[ch[b].x] = p;
        ++c;
      }
    }
  }
  count_changes(c, cnt);
}

// v joins its root's SCC if a successor (in A) of the same colour has joined
__global__ void k_same_pull(uint32_t n, const uint32_t* __restrict__ off, const uint32_t* __restrict__ col,
                            uint32_t heavy, const uint32_t* color, uint32_t* inscc, uint8_t* ep, uint8_t p,
                            unsigned long long* cnt) {
  uint32_t c = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; v0 < n; v0 += stride) {
    const uint32_t v = v0 + lane_id();
    if (v >= n) continue;
    const uint32_t cv = color[v];
    if (cv == kNoColor || bit(inscc, v) || off[v + 1] - off[v] > heavy) continue;
    for (uint32_t i = off[v]; i < off[v + 1]; ++i) {
      const uint32_t w = col[i];
      if (bit(inscc, w) && color[w] == cv) {
        atomicOr(inscc + (v >> 5), 1u << (v & 31u));
        ep[v] = p;
        ++c;
        break;
      }
    }
  }
  count_changes(c, cnt);
}

__global__ void k_same_pull_chunks(const uint4* __restrict__ chunks, uint32_t nch,
                                   const uint32_t* __restrict__ col, const uint32_t* color, uint32_t* inscc,
                                   uint8_t* ep, uint8_t p, unsigned long long* cnt) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  uint32_t c = 0;
  for (uint32_t k0 = gw * kCB; k0 < nch; k0 += nw * kCB) {
    uint4 ch[kCB];
    uint32_t cv[kCB];
    bool live[kCB];
#pragma unroll
    for (int b = 0; b < kCB; ++b) ch[b] = k0 + b < nch ? chunks[k0 + b] : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int b = 0; b < kCB; ++b) {
      const bool nonempty = ch[b].z > ch[b].y;
      cv[b] = nonempty ? color[ch[b].x] : kNoColor;
      live[b] = nonempty && !bit(inscc, ch[b].x);
    }
#pragma unroll
    for (int b = 0; b < kCB; ++b) live[b] = live[b] && cv[b] != kNoColor;
    uint32_t u[kCB][kCR];
    chunk_cols(ch, live, col, u);
    bool hit[kCB];
#pragma unroll
    for (int b = 0; b < kCB; ++b) {
      hit[b] = false;
#pragma unroll
      for (int r = 0; r < kCR; ++r) hit[b] |= u[b][r] != kNone && bit(inscc, u[b][r]) && color[u[b][r]] == cv[b];
      for (uint32_t i = ch[b].y + 32u * kCR + lane; live[b] && i < ch[b].z; i += 32u) {
        const uint32_t w = col[i];
        hit[b] |= bit(inscc, w) && color[w] == cv[b];
      }
    }
#pragma unroll
    for (int b = 0; b < kCB; ++b)
      if (__any_sync(kFull, hit[b]) && lane == 0 && test_and_set_bit(inscc, ch[b].x)) {
        ep[ch[b].x] = p;
        ++c;
      }
  }
  count_changes(c, cnt);
}

struct SeedEpoch {
  const uint8_t* ep;
  uint8_t p;
  __device__ bool operator()(uint32_t v) const { return ep[v] == p; }
};

__global__ void k_clear_roots(uint32_t n, const uint32_t* color, const uint32_t* inscc, uint32_t* rsize,
                              uint32_t* rflag) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (bit(inscc, v) && color[v] == v + 1u) {
      rsize[v] = 0;
      rflag[v] = 0;
    }
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

// ---- compaction of the kept subgraph. The kept set is a bitmap (n/8 bytes)
// with a per-word exclusive popcount prefix, both L2-resident even at 2^26+
// vertices: keep tests and new ids (prefix + popc) of the random column reads
// hit L2 instead of n-byte / 4n-byte arrays in HBM.
__global__ void k_keep_bits(uint32_t n, const uint8_t* keep, uint32_t* kb, uint32_t* pc) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; v0 < n; v0 += stride) {
    const uint32_t v = v0 + lane_id();
    const uint32_t w = __ballot_sync(kFull, v < n && keep[v]);
    if (lane_id() == 0) {
      kb[v0 >> 5] = w;
      pc[v0 >> 5] = __popc(w);
    }
  }
}

__device__ __forceinline__ bool kbit(const uint32_t* kb, uint32_t v) { return (kb[v >> 5] >> (v & 31u)) & 1u; }
__device__ __forceinline__ uint32_t knew(const uint32_t* kb, const uint32_t* wp, uint32_t v) {
  return wp[v >> 5] + __popc(kb[v >> 5] & ((1u << (v & 31u)) - 1u));
}

// keep bit word and its rank prefix side by side: one 8-byte load (one L2
// sector) per filtered column instead of two (k_filter_fill was bound by
// ~2.3 L2 sectors per column on config 3)
__device__ __forceinline__ uint32_t knew2(uint2 kw, uint32_t v) {
  return kw.y + __popc(kw.x & ((1u << (v & 31u)) - 1u));
}

__global__ void k_interleave(uint32_t words, const uint32_t* kb, const uint32_t* wp, uint2* kw) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < words; i += gridDim.x * blockDim.x)
    kw[i] = make_uint2(kb[i], wp[i]);
}

__global__ void k_kept_list(uint32_t n, const uint32_t* kb, const uint32_t* wp, uint32_t* kept) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (kbit(kb, v)) kept[knew(kb, wp, v)] = v;
}

// One warp per kept row (rows of R-MAT hubs are long): count, then an
// order-preserving ballot compaction of the kept columns.
// Filtering is row-parallel over the kept rows. A warp takes 32 consecutive
// kept rows; rows of <= kFilterLane edges are scanned by their own lane
// (one kept[] -> off[] dependency chain per 32 rows instead of per row),
// rows up to kBigRow by the whole warp, and longer rows (R-MAT hubs: one
// warp on a multi-million-edge row set the whole kernel's time on config 3)
// are cut into kChunkLen-edge chunks, one warp each: the chunk descriptors of
// a row are reserved contiguously and in order, so the output offset of a
// chunk is the row's offset plus an exclusive scan of the chunk counts.
constexpr uint32_t kFilterLane = 48;
constexpr uint32_t kBigRow = 8192;
constexpr uint32_t kChunkLen = 4096;

__device__ __forceinline__ bool filter_row_small(uint32_t b, uint32_t e) { return e - b <= kFilterLane; }
__device__ __forceinline__ bool filter_row_big(uint32_t b, uint32_t e) { return e - b > kBigRow; }

__global__ void k_filter_count(uint32_t k, const uint32_t* kept, const uint32_t* __restrict__ off,
                               const uint32_t* __restrict__ col, const uint32_t* kb, uint32_t* cnt,
                               uint4* desc, uint32_t* nchunks) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t a0 = gw * 32u; a0 < k; a0 += nw * 32u) {
    const uint32_t a = a0 + lane;
    uint32_t b = 0, e = 0;
    if (a < k) {
      const uint32_t v = kept[a];
      b = off[v];
      e = off[v + 1];
    }
    uint32_t c = 0;
    if (filter_row_small(b, e)) {
#pragma unroll 4
      for (uint32_t i = b; i < e; ++i) c += kbit(kb, __ldg(col + i));
    } else if (filter_row_big(b, e)) {  // counted by k_filter_chunk_count
      const uint32_t nc = (e - b + kChunkLen - 1) / kChunkLen;
      const uint32_t j0 = atomicAdd(nchunks, nc);
      for (uint32_t t = 0; t < nc; ++t)
        desc[j0 + t] = make_uint4(a, b + t * kChunkLen, min(e, b + (t + 1) * kChunkLen), j0);
    }
    const bool warp_row = !filter_row_small(b, e) && !filter_row_big(b, e);
    for (uint32_t hb = __ballot_sync(kFull, warp_row); hb; hb &= hb - 1u) {
      const uint32_t l = __ffs(hb) - 1u;
      const uint32_t bb = __shfl_sync(kFull, b, l), ee = __shfl_sync(kFull, e, l);
      uint32_t cc = 0;
      for (uint32_t i = bb + lane; i < ee; i += 32u) cc += kbit(kb, __ldg(col + i));
      cc = __reduce_add_sync(kFull, cc);
      if (lane == l) c = cc;
    }
    if (a < k) cnt[a] = c;
  }
}

__global__ void k_filter_chunk_count(const uint4* __restrict__ desc, const uint32_t* nchunks,
                                     const uint32_t* __restrict__ col, const uint32_t* kb, uint32_t* cch,
                                     uint32_t* cnt) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t C = *nchunks;
  for (uint32_t j = gw; j < C; j += nw) {
    const uint4 d = desc[j];
    uint32_t c = 0;
    for (uint32_t i = d.y + lane; i < d.z; i += 32u) c += kbit(kb, __ldg(col + i));
    c = __reduce_add_sync(kFull, c);
    if (lane == 0) {
      cch[j] = c;
      atomicAdd(cnt + d.x, c);
    }
  }
}

__device__ __forceinline__ void filter_fill_warp(uint32_t b, uint32_t e, uint32_t o, const uint32_t* col,
                                                 const uint2* kw, uint32_t* ncol) {
  const uint32_t lane = threadIdx.x & 31u;
  for (uint32_t i0 = b; i0 < e; i0 += 32u) {
    const uint32_t i = i0 + lane;
    const uint32_t w = i < e ? __ldg(col + i) : 0u;
    const uint2 k2 = i < e ? kw[w >> 5] : make_uint2(0u, 0u);
    const bool in = (k2.x >> (w & 31u)) & 1u;
    const uint32_t bal = __ballot_sync(kFull, in);
    if (in) ncol[o + __popc(bal & lanemask_lt())] = knew2(k2, w);
    o += __popc(bal);
  }
}

__global__ void k_filter_fill(uint32_t k, const uint32_t* kept, const uint32_t* __restrict__ off,
                              const uint32_t* __restrict__ col, const uint2* kw, const uint32_t* noff,
                              uint32_t* ncol) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t a0 = gw * 32u; a0 < k; a0 += nw * 32u) {
    const uint32_t a = a0 + lane;
    uint32_t b = 0, e = 0, o = 0;
    if (a < k) {
      const uint32_t v = kept[a];
      b = off[v];
      e = off[v + 1];
      o = noff[a];
    }
    if (filter_row_small(b, e)) {
#pragma unroll 4
      for (uint32_t i = b; i < e; ++i) {
        const uint32_t w = __ldg(col + i);
        const uint2 k2 = kw[w >> 5];
        if ((k2.x >> (w & 31u)) & 1u) ncol[o++] = knew2(k2, w);
      }
    }
    const bool warp_row = !filter_row_small(b, e) && !filter_row_big(b, e);
    for (uint32_t hb = __ballot_sync(kFull, warp_row); hb; hb &= hb - 1u) {
      const uint32_t l = __ffs(hb) - 1u;
      filter_fill_warp(__shfl_sync(kFull, b, l), __shfl_sync(kFull, e, l), __shfl_sync(kFull, o, l), col, kw,
                       ncol);
    }
  }
}

__global__ void k_filter_chunk_fill(const uint4* __restrict__ desc, uint32_t C, const uint32_t* __restrict__ col,
                                    const uint2* kw, const uint32_t* noff, const uint32_t* __restrict__ pre,
                                    uint32_t* ncol) {
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t j = gw; j < C; j += nw) {
    const uint4 d = desc[j];
    filter_fill_warp(d.y, d.z, noff[d.x] + pre[j] - pre[d.w], col, kw, ncol);
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
    std::fprintf(stderr, "[cyc scc %zx] %-12s passes %5d %9.3f ms\n", (size_t)pthread_self() & 0xFFFFFF, what, passes,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// A closure: Gauss-Seidel pull passes while they change many vertices (cheap
// per edge, no queue traffic; R-MAT converges in a handful), then the
// frontier engine from the vertices the last pass changed (long chains).
constexpr uint32_t kSwitchDiv = 64;  // frontier once a pass changes < n/64
constexpr int kMaxDense = 250;       // epochs are u8

template <class Dense, class Op>
int hybrid_closure(uint32_t n, uint8_t* ep, unsigned long long* dcnt, Dense&& dense, const DevCsr& push,
                   const FrontierBufs& fb, const Op& op, cudaStream_t s) {
  CYC_CUDA(cudaMemsetAsync(ep, 0, n, s));
  unsigned long long prev = ~0ull;
  for (int p = 1;; ++p) {
    unsigned long long c = 0;
    CYC_CUDA(cudaMemsetAsync(dcnt, 0, 8, s));
    dense((uint8_t)p);
    CYC_CUDA(cudaMemcpyAsync(&c, dcnt, 8, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
    if (c == 0) return p;
    // switch once the wave grows slowly or shrinks: a small first pass is
    // often the start of a large wave (config 3's same-colour closure: 6.5 K,
    // 5.9 M, 15 M, ... changes; switching after pass 1 cost 23 ms on the
    // frontier engine, four dense passes 14 ms), while a chain grows by a
    // few vertices per pass (config 4's colouring: 1, 2, 3, 4, 9, ...)
    const bool slow = p == 1 ? c <= 64 : c <= 4 * prev;
    prev = c;
    if ((c < n / kSwitchDiv && slow) || p == kMaxDense) {
      seed_frontier(n, SeedEpoch{ep, (uint8_t)p}, fb, nullptr, s);
      run_frontier(push.o(), push.c(), fb, op, s);
      return -p;  // negative: finished on the frontier engine
    }
  }
}

void filter_csr(const DevCsr& in, const uint32_t* kb, const uint32_t* wp, const uint32_t* kept,
                uint32_t k, cudaStream_t s, DevCsr& out) {
  out.n = k;
  out.off.alloc(((size_t)k + 1) * 4, s);
  DevBuf cnt(((size_t)k + 1) * 4, s), scratch;
  const size_t max_chunks = (size_t)in.m / kChunkLen + in.m / kBigRow + 1;
  DevBuf desc(max_chunks * sizeof(uint4), s), cch((max_chunks + 1) * 4, s), pre((max_chunks + 1) * 4, s);
  DevBuf nch(4, s);
  CYC_CUDA(cudaMemsetAsync(nch.p, 0, 4, s));
  if (k) {
    k_filter_count<<<sm_count() * 8, kT, 0, s>>>(k, kept, in.o(), in.c(), kb, cnt.as<uint32_t>(),
                                                 desc.as<uint4>(), nch.as<uint32_t>());
    CYC_LAUNCHED();
    k_filter_chunk_count<<<sm_count() * 8, kT, 0, s>>>(desc.as<uint4>(), nch.as<uint32_t>(), in.c(), kb,
                                                       cch.as<uint32_t>(), cnt.as<uint32_t>());
    CYC_LAUNCHED();
  }
  exclusive_scan(cnt.as<uint32_t>(), out.off.as<uint32_t>(), k, nullptr, s, scratch);
  uint32_t h[2] = {0, 0};
  CYC_CUDA(cudaMemcpyAsync(&h[0], out.off.as<uint32_t>() + k, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaMemcpyAsync(&h[1], nch.p, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  const uint32_t m = h[0], C = h[1];
  out.m = m;
  out.col.alloc(((size_t)m + 1) * 4, s);
  if (C) exclusive_scan(cch.as<uint32_t>(), pre.as<uint32_t>(), C, nullptr, s, scratch);
  const uint32_t words = (in.n + 31u) / 32u;
  DevBuf kw(((size_t)words + 1) * 8, s);
  if (words) {
    k_interleave<<<grid_for(words, kT, 8), kT, 0, s>>>(words, kb, wp, kw.as<uint2>());
    CYC_LAUNCHED();
  }
  if (k) {
    k_filter_fill<<<sm_count() * 8, kT, 0, s>>>(k, kept, in.o(), in.c(), kw.as<uint2>(), out.off.as<uint32_t>(),
                                                out.col.as<uint32_t>());
    CYC_LAUNCHED();
  }
  if (C) {
    k_filter_chunk_fill<<<grid_for((uint64_t)C * 32, kT, 8), kT, 0, s>>>(
        desc.as<uint4>(), C, in.c(), kw.as<uint2>(), out.off.as<uint32_t>(), pre.as<uint32_t>(),
        out.col.as<uint32_t>());
    CYC_LAUNCHED();
  }
}

}  // namespace

void scc_keep_mask(const DevCsr& snap_in, const DevCsr& gath_in, const uint64_t* acc, cudaStream_t s,
                   uint8_t* keep) {
  const uint32_t n = snap_in.n;
  CYC_CUDA(cudaMemsetAsync(keep, 0, (size_t)n + 1, s));
  if (!n) return;
  SccLog lg;
  const uint32_t grid = grid_for(n, kT, 8);
  DevBuf flag(32, s);
  uint32_t* f = flag.as<uint32_t>();
  // 0. colours flow along A, the relation with mostly ascending edges
  unsigned long long asc = 0;
  CYC_CUDA(cudaMemsetAsync(f, 0, 8, s));
  k_count_ascending<<<grid, kT, 0, s>>>(n, snap_in.o(), snap_in.c(), (unsigned long long*)f);
  CYC_LAUNCHED();
  CYC_CUDA(cudaMemcpyAsync(&asc, f, 8, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  const bool flip = 2 * asc < (unsigned long long)snap_in.m;
  const DevCsr& A = flip ? gath_in : snap_in;  // row u = successors of u in A
  const DevCsr& B = flip ? snap_in : gath_in;  // reverse of A
  const size_t words = (size_t)n / 32 + 2;
  DevBuf fw(words * 4, s), bw(words * 4, s), inscc(words * 4, s), active((size_t)n + 1, s);
  DevBuf color(((size_t)n + 1) * 4, s), stamp(((size_t)n + 1) * 4, s);
  DevBuf rsize(((size_t)n + 1) * 4, s), rflag(((size_t)n + 1) * 4, s);
  FrontierWs ws;
  const FrontierBufs fb = ws.bufs(n, (uint64_t)snap_in.m, s);
  lg.mark(flip ? "orient-rev" : "orient-fwd", 1);
  // 1. reach from F along A and along B (seeds: F, marked)
  CYC_CUDA(cudaMemsetAsync(fw.p, 0, words * 4, s));
  CYC_CUDA(cudaMemsetAsync(bw.p, 0, words * 4, s));
  CYC_CUDA(cudaMemcpyAsync(fw.p, acc, ((size_t)n + 63) / 64 * 8, cudaMemcpyDeviceToDevice, s));
  CYC_CUDA(cudaMemcpyAsync(bw.p, acc, ((size_t)n + 63) / 64 * 8, cudaMemcpyDeviceToDevice, s));
  DevBuf ep((size_t)n + 1, s);
  unsigned long long* dc = reinterpret_cast<unsigned long long*>(f + 4);
  const uint32_t cg = sm_count() * 8;
  auto hv = [](const DevCsr& g) { return g.n_heavy_chunks ? g.heavy_deg : kNone; };
  auto reach = [&](const DevCsr& push, const DevCsr& pull, DevBuf& mark, const uint8_t* act) {
    return hybrid_closure(n, ep.as<uint8_t>(), dc, [&](uint8_t p) {
      k_reach_pull<<<grid, kT, 0, s>>>(n, pull.o(), pull.c(), hv(pull), mark.as<uint32_t>(), ep.as<uint8_t>(), p, dc,
                                       act);
      CYC_LAUNCHED();
      if (pull.n_heavy_chunks) {
        k_reach_pull_chunks<<<cg, kT, 0, s>>>(pull.heavy.as<uint4>(), pull.n_heavy_chunks, pull.c(),
                                              mark.as<uint32_t>(), ep.as<uint8_t>(), p, dc, act);
        CYC_LAUNCHED();
      }
    }, push, fb, OpReach{mark.as<uint32_t>(), act}, s);
  };
  int np = reach(A, B, fw, nullptr);
  lg.mark("reach-A", np);
  np = reach(B, A, bw, nullptr);
  lg.mark("reach-B", np);
  k_and_bits<<<grid, kT, 0, s>>>(n, fw.as<uint32_t>(), bw.as<uint32_t>(), active.as<uint8_t>());
  CYC_LAUNCHED();
  for (int round = 0;; ++round) {
    np = until_stable(f, s, [&] {
      k_trim<<<grid, kT, 0, s>>>(n, A.o(), A.c(), B.o(), B.c(), active.as<uint8_t>(), f);
      CYC_LAUNCHED();
    });
    lg.mark("trim", np);
    if (round == 0) {
      unsigned long long* best = reinterpret_cast<unsigned long long*>(f + 6);
      unsigned long long hb = 0;
      CYC_CUDA(cudaMemsetAsync(best, 0, 8, s));
      k_pivot<<<grid, kT, 0, s>>>(n, A.o(), B.o(), active.as<uint8_t>(), best);
      CYC_LAUNCHED();
      CYC_CUDA(cudaMemcpyAsync(&hb, best, 8, cudaMemcpyDeviceToHost, s));
      CYC_CUDA(cudaStreamSynchronize(s));
      if (hb) {  // some vertex is active
        const uint32_t pivot = (uint32_t)hb, word = 1u << (pivot & 31u);
        CYC_CUDA(cudaMemsetAsync(fw.p, 0, words * 4, s));
        CYC_CUDA(cudaMemsetAsync(bw.p, 0, words * 4, s));
        CYC_CUDA(cudaMemcpyAsync(fw.as<uint32_t>() + (pivot >> 5), &word, 4, cudaMemcpyHostToDevice, s));
        CYC_CUDA(cudaMemcpyAsync(bw.as<uint32_t>() + (pivot >> 5), &word, 4, cudaMemcpyHostToDevice, s));
        np = reach(A, B, fw, active.as<uint8_t>());
        lg.mark("pivot-fw", np);
        // the pivot's SCC lies inside its forward set: the backward closure
        // only explores fw (config 2's pivot is a DAG connector: 63 backward
        // passes over the whole graph otherwise)
        uint8_t* act2 = stamp.as<uint8_t>();  // scratch until the colour closure
        k_and_act<<<grid, kT, 0, s>>>(n, active.as<uint8_t>(), fw.as<uint32_t>(), act2);
        CYC_LAUNCHED();
        np = reach(B, A, bw, act2);
        lg.mark("pivot-bw", np);
        k_pivot_scc<<<grid, kT, 0, s>>>(n, fw.as<uint32_t>(), bw.as<uint32_t>(), active.as<uint8_t>(), pivot,
                                        inscc.as<uint32_t>(), color.as<uint32_t>());
        CYC_LAUNCHED();
        k_clear_roots<<<grid, kT, 0, s>>>(n, color.as<uint32_t>(), inscc.as<uint32_t>(), rsize.as<uint32_t>(),
                                          rflag.as<uint32_t>());
        CYC_LAUNCHED();
        k_scc_stats<<<grid, kT, 0, s>>>(n, acc, inscc.as<uint32_t>(), color.as<uint32_t>(), rsize.as<uint32_t>(),
                                        rflag.as<uint32_t>());
        CYC_LAUNCHED();
        uint32_t any = 0;
        CYC_CUDA(cudaMemsetAsync(f, 0, 4, s));
        k_scc_apply<<<grid, kT, 0, s>>>(n, A.o(), A.c(), color.as<uint32_t>(), rsize.as<uint32_t>(),
                                        rflag.as<uint32_t>(), inscc.as<uint32_t>(), active.as<uint8_t>(), keep, f);
        CYC_LAUNCHED();
        CYC_CUDA(cudaMemcpyAsync(&any, f, 4, cudaMemcpyDeviceToHost, s));
        CYC_CUDA(cudaStreamSynchronize(s));
        lg.mark("pivot-apply", 1);
        if (lg.on) {
          unsigned long long cnt_scc = 0;
          std::vector<uint32_t> hw(words);
          CYC_CUDA(cudaMemcpyAsync(hw.data(), inscc.p, words * 4, cudaMemcpyDeviceToHost, s));
          CYC_CUDA(cudaStreamSynchronize(s));
          for (uint32_t x : hw) cnt_scc += __builtin_popcount(x);
          std::fprintf(stderr, "[cyc scc]   pivot %u deg %llu scc %llu (n %u, m %u)\n", pivot, hb >> 32, cnt_scc, n,
                       snap_in.m);
        }
        if (!any) break;
        continue;  // trim what the pivot's SCC leaves, then colour it
      }
    }
    k_color_init<<<grid, kT, 0, s>>>(n, active.as<uint8_t>(), color.as<uint32_t>());
    CYC_LAUNCHED();
    CYC_CUDA(cudaMemsetAsync(stamp.p, 0, (size_t)n * 4, s));
    np = hybrid_closure(n, ep.as<uint8_t>(), dc, [&](uint8_t p) {
      k_color_pull<<<grid, kT, 0, s>>>(n, B.o(), B.c(), hv(B), color.as<uint32_t>(), ep.as<uint8_t>(), p, dc);
      CYC_LAUNCHED();
      if (B.n_heavy_chunks) {
        k_color_pull_chunks<<<cg, kT, 0, s>>>(B.heavy.as<uint4>(), B.n_heavy_chunks, B.c(), color.as<uint32_t>(),
                                              ep.as<uint8_t>(), p, dc);
        CYC_LAUNCHED();
      }
    }, A, fb, OpColor{color.as<uint32_t>(), stamp.as<uint32_t>()}, s);
    lg.mark("color", np);
    CYC_CUDA(cudaMemsetAsync(inscc.p, 0, words * 4, s));
    seed_frontier(n, SeedRoots{color.as<uint32_t>()}, fb, inscc.as<uint32_t>(), s);
    np = hybrid_closure(n, ep.as<uint8_t>(), dc, [&](uint8_t p) {
      k_same_pull<<<grid, kT, 0, s>>>(n, A.o(), A.c(), hv(A), color.as<uint32_t>(), inscc.as<uint32_t>(),
                                      ep.as<uint8_t>(), p, dc);
      CYC_LAUNCHED();
      if (A.n_heavy_chunks) {
        k_same_pull_chunks<<<cg, kT, 0, s>>>(A.heavy.as<uint4>(), A.n_heavy_chunks, A.c(), color.as<uint32_t>(),
                                             inscc.as<uint32_t>(), ep.as<uint8_t>(), p, dc);
        CYC_LAUNCHED();
      }
    }, B, fb, OpSameColor{color.as<uint32_t>(), inscc.as<uint32_t>()}, s);
    lg.mark("same-color", np);
    k_clear_roots<<<grid, kT, 0, s>>>(n, color.as<uint32_t>(), inscc.as<uint32_t>(), rsize.as<uint32_t>(),
                                      rflag.as<uint32_t>());
    CYC_LAUNCHED();
    k_scc_stats<<<grid, kT, 0, s>>>(n, acc, inscc.as<uint32_t>(), color.as<uint32_t>(), rsize.as<uint32_t>(),
                                    rflag.as<uint32_t>());
    CYC_LAUNCHED();
    uint32_t any = 0;
    CYC_CUDA(cudaMemsetAsync(f, 0, 4, s));
    k_scc_apply<<<grid, kT, 0, s>>>(n, A.o(), A.c(), color.as<uint32_t>(), rsize.as<uint32_t>(), rflag.as<uint32_t>(),
                                    inscc.as<uint32_t>(), active.as<uint8_t>(), keep, f);
    CYC_LAUNCHED();
    CYC_CUDA(cudaMemcpyAsync(&any, f, 4, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
    lg.mark("apply", round + 1);
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
  const size_t nwd = (size_t)n / 32 + 2;
  DevBuf keep((size_t)n + 1, s), kb(nwd * 4, s), pc(nwd * 4, s), wp((nwd + 1) * 4, s), scratch;
  scc_keep_mask(snap, gath, acc, s, keep.as<uint8_t>());
  SccLog lg;
  CYC_CUDA(cudaMemsetAsync(kb.p, 0, nwd * 4, s));
  CYC_CUDA(cudaMemsetAsync(pc.p, 0, nwd * 4, s));
  if (n) {
    k_keep_bits<<<grid_for(n, kT, 8), kT, 0, s>>>(n, keep.as<uint8_t>(), kb.as<uint32_t>(), pc.as<uint32_t>());
    CYC_LAUNCHED();
  }
  const uint32_t nw = (uint32_t)((n + 31) / 32);
  exclusive_scan(pc.as<uint32_t>(), wp.as<uint32_t>(), nw, nullptr, s, scratch);
  uint32_t k = 0;
  CYC_CUDA(cudaMemcpyAsync(&k, wp.as<uint32_t>() + nw, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  out_kept.alloc(((size_t)k + 1) * 4, s);
  if (n) {
    k_kept_list<<<grid_for(n, kT, 8), kT, 0, s>>>(n, kb.as<uint32_t>(), wp.as<uint32_t>(), out_kept.as<uint32_t>());
    CYC_LAUNCHED();
  }
  lg.mark("kept-list", 1);
  filter_csr(snap, kb.as<uint32_t>(), wp.as<uint32_t>(), out_kept.as<uint32_t>(), k, s, out_snap);
  lg.mark("filter-snap", 1);
  filter_csr(gath, kb.as<uint32_t>(), wp.as<uint32_t>(), out_kept.as<uint32_t>(), k, s, out_gath);
  lg.mark("filter-gath", 1);
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
