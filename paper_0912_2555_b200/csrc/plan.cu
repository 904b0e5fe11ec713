// plan.cu — degree-ordered storage for the MAP loop (see plan.cuh).
//
// Build, all on the device, deterministic:
//   1. bucket key per vertex from its snapshot-row length (= how many gather
//      rows contain it), descending; log-linear buckets above 512.
//   2. stable counting sort of the vertices by key: per-warp ranges, a
//      [bucket x warp] count table scanned bucket-major, then each warp places
//      its vertices in sequence order (match_any ranks) -> orig[] and perm[].
//      Ties (equally gathered vertices, so equally hot in L2) are broken by
//      gather-row length through a first stable pass (LSD), which makes the
//      sliced ELL's 32-row slices near uniform (config 3 family: 2.2x -> 1.01x
//      padding of the light rows).
//   3. both CSRs re-laid out in storage order with columns mapped through
//      perm[]: rows <= kHeavyDeg as 32-row warp groups walking their
//      concatenated edges, longer rows from the graph's heavy-chunk lists.
// Row contents keep their (sorted-by-id) order; the loop never relies on
// column order, only on the set.
#include <chrono>
#include <cstdlib>
#include <vector>

#include "plan.cuh"

namespace cyc {

namespace {

constexpr uint32_t kBuckets = 1024;
constexpr int kPlanWarps = 8;  // warps per CTA in the sort kernels
// tie-break classes: gather-row lengths 0..64 exact, longer (heavy-slab) rows
// share one class, so the 32-row slices of the sliced ELL are near uniform
constexpr uint32_t kTieClamp = 65;

__device__ __forceinline__ uint32_t lane_of() { return threadIdx.x & 31u; }

// monotone non-decreasing in d; exact below 512, 64 sub-buckets per octave above
__device__ __forceinline__ uint32_t deg_bucket(uint32_t d) {
  if (d < 512u) return d;
  const uint32_t lg = 31u - __clz(d);
  const uint32_t b = 512u + (lg - 9u) * 64u + ((d >> (lg - 6u)) & 63u);
  return b < kBuckets ? b : kBuckets - 1u;
}

// descending degree first (degrees above `clamp` share one bucket)
__device__ __forceinline__ uint32_t sort_key(const uint32_t* __restrict__ off, uint32_t v, uint32_t clamp) {
  return kBuckets - 1u - min(deg_bucket(__ldg(off + v + 1) - __ldg(off + v)), clamp);
}

// i-th vertex of the sequence being sorted (ids, or a previous pass's order)
__device__ __forceinline__ uint32_t seq_at(const uint32_t* __restrict__ src, uint64_t i) {
  return src ? __ldg(src + i) : (uint32_t)i;
}

// T[key * nw + w] = vertices of warp range w with that key
__global__ void k_plan_hist(uint32_t n, uint32_t per_warp, const uint32_t* __restrict__ soff,
                            const uint32_t* __restrict__ src, uint32_t clamp, uint32_t* __restrict__ T,
                            uint32_t nw) {
  __shared__ uint32_t h[kPlanWarps][kBuckets];
  const uint32_t wl = threadIdx.x >> 5, lane = lane_of();
  const uint32_t gw = blockIdx.x * kPlanWarps + wl;
  for (uint32_t k = lane; k < kBuckets; k += 32u) h[wl][k] = 0u;
  __syncwarp();
  if (gw < nw) {
    const uint64_t lo = (uint64_t)gw * per_warp;
    const uint64_t hi = lo + per_warp < n ? lo + per_warp : n;
    for (uint64_t v = lo + lane; v < hi; v += 32u) atomicAdd(&h[wl][sort_key(soff, seq_at(src, v), clamp)], 1u);
    __syncwarp();
    for (uint32_t k = lane; k < kBuckets; k += 32u) T[(size_t)k * nw + gw] = h[wl][k];
  }
}

// per-bucket totals (the decision input), one thread per bucket
__global__ void k_plan_totals(const uint32_t* __restrict__ T, uint32_t nw, unsigned long long* tot) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= kBuckets) return;
  unsigned long long s = 0;
  for (uint32_t w = 0; w < nw; ++w) s += T[(size_t)k * nw + w];
  tot[k] = s;
}

__global__ void k_plan_place(uint32_t n, uint32_t per_warp, const uint32_t* __restrict__ soff,
                             const uint32_t* __restrict__ src, uint32_t clamp, const uint32_t* __restrict__ base, uint32_t nw, uint32_t* __restrict__ orig,
                             uint32_t* __restrict__ perm) {
  __shared__ uint32_t cur[kPlanWarps][kBuckets];
  const uint32_t wl = threadIdx.x >> 5, lane = lane_of();
  const uint32_t gw = blockIdx.x * kPlanWarps + wl;
  if (gw >= nw) return;
  for (uint32_t k = lane; k < kBuckets; k += 32u) cur[wl][k] = base[(size_t)k * nw + gw];
  __syncwarp();
  const uint64_t lo = (uint64_t)gw * per_warp;
  const uint64_t hi = lo + per_warp < n ? lo + per_warp : n;
  const uint32_t below = (1u << lane) - 1u;
  for (uint64_t i0 = lo; i0 < hi; i0 += 32u) {
    const uint64_t i = i0 + lane;
    const bool ok = i < hi;
    const uint32_t v = ok ? seq_at(src, i) : 0u;
    const uint32_t key = ok ? sort_key(soff, v, clamp) : kBuckets + lane;  // unmatched sentinel
    const uint32_t peers = __match_any_sync(kFull, key);
    if (ok) {
      const uint32_t pos = cur[wl][key] + __popc(peers & below);
      orig[pos] = v;
      if (perm) perm[v] = pos;
    }
    __syncwarp();
    if (ok && (__ffs(peers) - 1u) == lane) cur[wl][key] += __popc(peers);
    __syncwarp();
  }
}

__global__ void k_plan_pad(uint32_t n, uint32_t np1, uint32_t* orig) {
  for (uint32_t p = n + blockIdx.x * blockDim.x + threadIdx.x; p < np1; p += gridDim.x * blockDim.x) orig[p] = p;
}

// storage row lengths
__global__ void k_plan_degs(uint32_t n, const uint32_t* __restrict__ orig, const uint32_t* __restrict__ off,
                            uint32_t* __restrict__ deg) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const uint32_t v = __ldg(orig + p);
    deg[p] = __ldg(off + v + 1) - __ldg(off + v);
  }
}

// Rows of at most `heavy` edges: a warp takes 32 storage rows and walks their
// concatenated edges (owner lane by a 5-step shuffle search), so a warp's
// output is one contiguous range and its reads 32 short sequential runs.
__global__ void k_plan_light(uint32_t n, uint32_t heavy, const uint32_t* __restrict__ orig,
                             const uint32_t* __restrict__ off, const uint32_t* __restrict__ col,
                             const uint32_t* __restrict__ perm, const uint32_t* __restrict__ noff,
                             uint32_t* __restrict__ ncol) {
  const uint32_t lane = lane_of();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t p0 = gw * 32u; p0 < n; p0 += nw * 32u) {
    const uint32_t p = p0 + lane;
    uint32_t b = 0, d = 0, o = 0;
    if (p < n) {
      const uint32_t v = __ldg(orig + p);
      b = __ldg(off + v);
      d = __ldg(off + v + 1) - b;
      o = __ldg(noff + p);
      if (d > heavy) d = 0;  // chunk pass
    }
    uint32_t incl = d;  // inclusive prefix over lanes
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, k);
      if (lane >= (uint32_t)k) incl += t;
    }
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    const uint32_t excl = incl - d;
    // 4 rounds of 32 edges at a time: all column and perm loads in flight
    for (uint32_t e0 = 0; e0 < total; e0 += 128u) {
      uint32_t src[4], dst[4], u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t e = e0 + 32u * q + lane;
        // owner r: largest lane with excl[r] <= e (d[r] > 0 guaranteed for it)
        uint32_t r = 0;
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
          const uint32_t probe = __shfl_sync(kFull, excl, r + s);
          if (probe <= e) r += s;
        }
        const uint32_t rb = __shfl_sync(kFull, b, r), ro = __shfl_sync(kFull, o, r),
                       rx = __shfl_sync(kFull, excl, r);
        src[q] = e < total ? rb + (e - rx) : kNone;
        dst[q] = ro + (e - rx);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) u[q] = src[q] != kNone ? __ldg(col + src[q]) : 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q) u[q] = src[q] != kNone ? __ldg(perm + u[q]) : 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (src[q] != kNone) ncol[dst[q]] = u[q];
    }
  }
}

// Heavy rows from the graph's chunk list {row, beg, end, 0}: one warp per chunk.
__global__ void k_plan_chunks(const uint4* __restrict__ chunks, uint32_t nch, const uint32_t* __restrict__ off,
                              const uint32_t* __restrict__ col, const uint32_t* __restrict__ perm,
                              const uint32_t* __restrict__ noff, uint32_t* __restrict__ ncol) {
  const uint32_t lane = lane_of();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t c = gw; c < nch; c += nw) {
    const uint4 ch = chunks[c];
    const uint32_t dst = __ldg(noff + __ldg(perm + ch.x)) + (ch.y - __ldg(off + ch.x));
    for (uint32_t i0 = ch.y; i0 < ch.z; i0 += 128u) {  // all loads of 4 rounds in flight
      uint32_t u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t i = i0 + 32u * q + lane;
        u[q] = i < ch.z ? __ldg(col + i) : 0u;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) u[q] = i0 + 32u * q + lane < ch.z ? __ldg(perm + u[q]) : 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t i = i0 + 32u * q + lane;
        if (i < ch.z) ncol[dst + (i - ch.y)] = u[q];
      }
    }
  }
}

// per slice of 32 rows: widest light row and the mask of heavy rows
__global__ void k_sell_width(uint32_t n, uint32_t row0, uint32_t nsl, const uint32_t* __restrict__ off,
                             uint32_t heavy, uint32_t* __restrict__ width, uint32_t* __restrict__ hmask) {
  const uint32_t lane = lane_of();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t sI = gw; sI < nsl; sI += nw) {
    const uint32_t v = row0 + sI * 32u + lane;
    const uint32_t d = v < n ? __ldg(off + v + 1) - __ldg(off + v) : 0u;
    const bool hv = d > heavy;
    const uint32_t w = __reduce_max_sync(kFull, hv ? 0u : d);
    const uint32_t hm = __ballot_sync(kFull, hv);
    if (lane == 0) {
      width[sI] = w;
      hmask[sI] = hm;
    }
  }
}

__global__ void k_sell_fill(uint32_t n, uint32_t row0, uint32_t nsl, uint32_t np, const uint32_t* __restrict__ off,
                            const uint32_t* __restrict__ col, const uint32_t* __restrict__ width,
                            const uint32_t* __restrict__ soff, const uint32_t* __restrict__ hmask,
                            uint32_t* __restrict__ sell, uint4* __restrict__ sdesc) {
  const uint32_t lane = lane_of();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t sI = gw; sI < nsl; sI += nw) {
    const uint32_t v = row0 + sI * 32u + lane;
    const uint32_t hm = hmask[sI], w = width[sI], o = soff[sI];
    uint32_t b = 0, d = 0;
    if (v < n && !((hm >> lane) & 1u)) {
      b = __ldg(off + v);
      d = __ldg(off + v + 1) - b;
    }
    for (uint32_t j = 0; j < w; ++j) sell[((size_t)o + j) * 32u + lane] = j < d ? __ldg(col + b + j) : np;
    if (lane == 0) sdesc[sI] = make_uint4(o, w, hm, 0u);
  }
}

// heavy chunk c {row, beg, end} -> padded column block and its row
__global__ void k_hslab_fill(const uint4* __restrict__ chunks, uint32_t nch, const uint32_t* __restrict__ col,
                             uint32_t np, uint32_t* __restrict__ hcol, uint32_t* __restrict__ hrow) {
  const uint32_t lane = lane_of();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t c = gw; c < nch; c += nw) {
    const uint4 ch = chunks[c];
    for (uint32_t j = lane; j < kHeavyChunk; j += 32u)
      hcol[(size_t)c * kHeavyChunk + j] = ch.y + j < ch.z ? __ldg(col + ch.y + j) : np;
    if (lane == 0) hrow[c] = ch.x;
  }
}

// ---- heavy rows' columns in storage order ----------------------------------
// Sorted by storage position, a hub row's hot sources (low positions) sit in
// the same chunk rounds, so a warp's gathers touch fewer distinct lines
// (scale-23 model: 15 % fewer over all heavy rows, 48 % above 16 K edges;
// measured on config 3: 0.9 % of run_map — the hot words were mostly L1/L2
// hits already).
// Rows up to kSortSmall columns: bitonic sort in shared memory, a CTA per row;
// longer ones: their columns below kHotBits through a shared bitmap (emitted
// in order), the rest (cold: one per line anyway) after them in their order.
constexpr uint32_t kSortSmall = 4096;
constexpr uint32_t kHotBits = 1u << 20;  // 128 KB bitmap

__global__ void k_heavy_rowlist(const uint4* __restrict__ chunks, uint32_t nch, const uint32_t* __restrict__ off,
                                uint32_t* __restrict__ small, uint32_t* __restrict__ big, uint32_t* cnt) {
  const uint32_t lane = lane_of();
  const uint32_t t0 = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (uint32_t c0 = t0 - lane; c0 < nch; c0 += nt) {
    const uint32_t c = c0 + lane;
    bool first = false, sm = false;
    uint32_t row = 0;
    if (c < nch) {
      const uint4 ch = chunks[c];
      row = ch.x;
      first = ch.y == __ldg(off + row);
      sm = __ldg(off + row + 1) - ch.y <= kSortSmall;
    }
    const uint32_t ms = __ballot_sync(kFull, first && sm), mb = __ballot_sync(kFull, first && !sm);
    uint32_t bs = 0, bb = 0;
    if (lane == 0) {
      if (ms) bs = atomicAdd(cnt, __popc(ms));
      if (mb) bb = atomicAdd(cnt + 1, __popc(mb));
    }
    bs = __shfl_sync(kFull, bs, 0);
    bb = __shfl_sync(kFull, bb, 0);
    const uint32_t below = (1u << lane) - 1u;
    if (first && sm) small[bs + __popc(ms & below)] = row;
    if (first && !sm) big[bb + __popc(mb & below)] = row;
  }
}

__global__ void __launch_bounds__(512) k_sort_small(const uint32_t* __restrict__ rows, const uint32_t* cnt,
                                                    const uint32_t* __restrict__ off,
                                                    const uint32_t* __restrict__ src, uint32_t* __restrict__ dst) {
  __shared__ uint32_t k[kSortSmall];
  const uint32_t nr = cnt[0];
  for (uint32_t i = blockIdx.x; i < nr; i += gridDim.x) {
    const uint32_t r = rows[i], b = __ldg(off + r), d = __ldg(off + r + 1) - b;
    uint32_t N = 128;
    while (N < d) N <<= 1;
    for (uint32_t j = threadIdx.x; j < N; j += blockDim.x) k[j] = j < d ? __ldg(src + b + j) : 0xFFFFFFFFu;
    __syncthreads();
    for (uint32_t kk = 2; kk <= N; kk <<= 1)
      for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
        for (uint32_t x = threadIdx.x; x < N; x += blockDim.x) {
          const uint32_t y = x ^ jj;
          if (y > x) {
            const uint32_t p = k[x], q = k[y];
            if ((p > q) == ((x & kk) == 0u)) {
              k[x] = q;
              k[y] = p;
            }
          }
        }
        __syncthreads();
      }
    for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) dst[b + j] = k[j];
    __syncthreads();
  }
}

// exclusive scan over the CTA; *tot = the total (valid after the call)
__device__ __forceinline__ uint32_t cta_scan(uint32_t x, uint32_t* ws, uint32_t* tot) {
  const uint32_t lane = lane_of(), w = threadIdx.x >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, inc, o);
    if (lane >= (uint32_t)o) inc += y;
  }
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t v = lane < (blockDim.x >> 5) ? ws[lane] : 0u;
    uint32_t vi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, vi, o);
      if (lane >= (uint32_t)o) vi += y;
    }
    ws[lane] = vi - v;
    if (lane == 31) *tot = vi;
  }
  __syncthreads();
  const uint32_t r = ws[w] + inc - x;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(1024, 1) k_sort_hub(const uint32_t* __restrict__ rows, const uint32_t* cnt,
                                                      const uint32_t* __restrict__ off, uint32_t np,
                                                      const uint32_t* __restrict__ src, uint32_t* __restrict__ dst) {
  extern __shared__ uint32_t bm[];
  __shared__ uint32_t ws[32], tot;
  const uint32_t nr = cnt[1];
  const uint32_t hot = np < kHotBits ? np : kHotBits, nwd = (hot + 31u) / 32u;
  for (uint32_t i = blockIdx.x; i < nr; i += gridDim.x) {
    const uint32_t r = rows[i], b = __ldg(off + r), e = __ldg(off + r + 1);
    for (uint32_t j = threadIdx.x; j < nwd; j += blockDim.x) bm[j] = 0u;
    __syncthreads();
    uint32_t cold = 0;
    for (uint32_t j = b + threadIdx.x; j < e; j += blockDim.x) {
      const uint32_t c = __ldg(src + j);
      if (c < hot) atomicOr(bm + (c >> 5), 1u << (c & 31u));
      else ++cold;
    }
    cta_scan(cold, ws, &tot);
    uint32_t cbase = e - tot;
    for (uint32_t j0 = b; j0 < e; j0 += blockDim.x) {
      const uint32_t j = j0 + threadIdx.x;
      const uint32_t c = j < e ? __ldg(src + j) : 0u;
      const uint32_t f = j < e && c >= hot;
      const uint32_t pos = cta_scan(f, ws, &tot);
      if (f) dst[cbase + pos] = c;
      cbase += tot;
      __syncthreads();
    }
    const uint32_t per = (nwd + blockDim.x - 1u) / blockDim.x;
    const uint32_t w0 = min(threadIdx.x * per, nwd), w1 = min(w0 + per, nwd);
    uint32_t hc = 0;
    for (uint32_t w = w0; w < w1; ++w) hc += __popc(bm[w]);
    uint32_t o = b + cta_scan(hc, ws, &tot);
    for (uint32_t w = w0; w < w1; ++w) {
      uint32_t m = bm[w];
      while (m) {
        dst[o++] = w * 32u + (__ffs(m) - 1u);
        m &= m - 1u;
      }
    }
    __syncthreads();
  }
}

void sort_heavy_rows(DevCsr& g, uint32_t np, cudaStream_t s) {
  if (!g.n_heavy_chunks) return;
  DevBuf lists(((size_t)g.n_heavy_chunks * 2 + 2) * 4, s), cnt(8, s), out((size_t)g.m * 4 + 4, s);
  uint32_t* small = lists.as<uint32_t>();
  uint32_t* big = small + g.n_heavy_chunks + 1;
  CYC_CUDA(cudaMemsetAsync(cnt.p, 0, 8, s));
  CYC_CUDA(cudaMemcpyAsync(out.p, g.col.p, (size_t)g.m * 4, cudaMemcpyDeviceToDevice, s));  // light rows
  k_heavy_rowlist<<<grid_for(g.n_heavy_chunks, 256, 8), 256, 0, s>>>(g.heavy.as<uint4>(), g.n_heavy_chunks, g.o(),
                                                                    small, big, cnt.as<uint32_t>());
  CYC_LAUNCHED();
  k_sort_small<<<sm_count() * 4, 512, 0, s>>>(small, cnt.as<uint32_t>(), g.o(), g.c(), out.as<uint32_t>());
  CYC_LAUNCHED();
  static const bool attr = [] {
    CYC_CUDA(cudaFuncSetAttribute(k_sort_hub, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kHotBits / 8)));
    return true;
  }();
  (void)attr;
  k_sort_hub<<<sm_count(), 1024, kHotBits / 8, s>>>(big, cnt.as<uint32_t>(), g.o(), np, g.c(), out.as<uint32_t>());
  CYC_LAUNCHED();
  g.col = std::move(out);
}

__global__ void k_permute_bits(const uint32_t* __restrict__ src, const uint32_t* __restrict__ orig, uint32_t n,
                               uint32_t* __restrict__ dst) {
  const uint32_t lane = lane_of();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t words = (n + 31u) / 32u;
  for (uint32_t wi = gw; wi < words; wi += nw) {
    const uint32_t p = wi * 32u + lane;
    bool bit = false;
    if (p < n) {
      const uint32_t v = __ldg(orig + p);
      bit = (__ldg(src + (v >> 5)) >> (v & 31u)) & 1u;
    }
    const uint32_t w = __ballot_sync(kFull, bit);
    if (lane == 0) dst[wi] = w;
  }
}

}  // namespace

// One CSR in storage order (rows and columns relabelled); rows longer than
// in.heavy_deg come from in's heavy-chunk list.
void relayout(const DevCsr& in, const uint32_t* orig, const uint32_t* perm, DevCsr& out, DevBuf& scratch,
              cudaStream_t s) {
  const uint32_t n = in.n;
  out.n = n;
  out.m = in.m;
  out.off.alloc(((size_t)n + 1) * 4, s);
  out.col.alloc((in.m ? in.m : 1) * 4ull, s);
  DevBuf deg(((size_t)n + 1) * 4, s);
  k_plan_degs<<<grid_for(n, 256, 8), 256, 0, s>>>(n, orig, in.o(), deg.as<uint32_t>());
  CYC_LAUNCHED();
  exclusive_scan(deg.as<uint32_t>(), out.off.as<uint32_t>(), n, nullptr, s, scratch);
  const uint32_t heavy = in.n_heavy_chunks ? in.heavy_deg : 0xFFFFFFFFu;
  k_plan_light<<<grid_for((uint64_t)n, 256, 8), 256, 0, s>>>(n, heavy, orig, in.o(), in.c(), perm, out.o(),
                                                             out.col.as<uint32_t>());
  CYC_LAUNCHED();
  if (in.n_heavy_chunks) {
    k_plan_chunks<<<grid_for((uint64_t)in.n_heavy_chunks * 32, 256, 8), 256, 0, s>>>(
        in.heavy.as<uint4>(), in.n_heavy_chunks, in.o(), in.c(), perm, out.o(), out.col.as<uint32_t>());
    CYC_LAUNCHED();
  }
}

void degree_order(const uint32_t* key_off, const uint32_t* tie_off, uint32_t n, uint32_t* orig, uint32_t* perm,
                  cudaStream_t s) {
  const uint32_t nw = (uint32_t)sm_count() * kPlanWarps;
  const uint32_t per_warp = div_up(div_up(n, nw), 32) * 32;
  const uint32_t blocks = div_up(nw, kPlanWarps);
  const uint32_t np = (uint32_t)(((uint64_t)n + kRowPad - 1) / kRowPad * kRowPad);
  DevBuf T((size_t)kBuckets * nw * 4, s), base((size_t)kBuckets * nw * 4 + 4, s), scratch, seq;
  // LSD: the tie-break pass first (stable sorts), then the primary key over its order
  auto pass = [&](const uint32_t* off, const uint32_t* src, uint32_t clamp, uint32_t* out, uint32_t* pm) {
    k_plan_hist<<<blocks, kPlanWarps * 32, 0, s>>>(n, per_warp, off, src, clamp, T.as<uint32_t>(), nw);
    CYC_LAUNCHED();
    exclusive_scan(T.as<uint32_t>(), base.as<uint32_t>(), kBuckets * nw, nullptr, s, scratch);
    k_plan_place<<<blocks, kPlanWarps * 32, 0, s>>>(n, per_warp, off, src, clamp, base.as<uint32_t>(), nw, out, pm);
    CYC_LAUNCHED();
  };
  const char* tb = std::getenv("CYC_PLAN_TIE");
  if (tie_off && !(tb && tb[0] == '0')) {
    seq.alloc((size_t)n * 4, s);
    pass(tie_off, nullptr, kTieClamp, seq.as<uint32_t>(), nullptr);
    pass(key_off, seq.as<uint32_t>(), kBuckets - 1u, orig, perm);
  } else {
    pass(key_off, nullptr, kBuckets - 1u, orig, perm);
  }
  k_plan_pad<<<grid_for(np + 1 - n, 256, 1), 256, 0, s>>>(n, np + 1, orig);
  CYC_LAUNCHED();
}

void build_hslab(DevCsr& g, uint32_t np, DevBuf& hcol, DevBuf& hrow, uint32_t& n_hchunks, cudaStream_t s) {
  build_heavy(g, kHeavyDeg, kHeavyChunk, s, 1u);
  // rows sorted by position: ~0.9 % on config 3's run_map (11.55 -> 11.45 ms,
  // alternating A/B, scripts/gpu_ab_sort.sh) for ~20 ms of plan build;
  // CYC_SORT_HEAVY=0 keeps the id order
  const char* sh = std::getenv("CYC_SORT_HEAVY");
  if (!(sh && sh[0] == '0')) sort_heavy_rows(g, np, s);
  n_hchunks = g.n_heavy_chunks;
  hcol.alloc(((size_t)n_hchunks * kHeavyChunk + 1) * 4, s);
  hrow.alloc(((size_t)n_hchunks + 1) * 4, s);
  if (n_hchunks) {
    k_hslab_fill<<<grid_for((uint64_t)n_hchunks * 32, 256, 8), 256, 0, s>>>(
        g.heavy.as<uint4>(), n_hchunks, g.c(), np, hcol.as<uint32_t>(), hrow.as<uint32_t>());
    CYC_LAUNCHED();
  }
}

uint64_t build_sell(const DevCsr& g, uint32_t row_lo, uint32_t row_hi, uint32_t np, DevBuf& sell, DevBuf& sdesc,
                    cudaStream_t s) {
  const uint32_t nsl = (row_hi - row_lo) / 32u;
  DevBuf width(((size_t)nsl + 1) * 4, s), soff(((size_t)nsl + 1) * 4, s), hmask(((size_t)nsl + 1) * 4, s), scratch;
  k_sell_width<<<grid_for((uint64_t)nsl * 32, 256, 8), 256, 0, s>>>(g.n, row_lo, nsl, g.o(), kHeavyDeg,
                                                                   width.as<uint32_t>(), hmask.as<uint32_t>());
  CYC_LAUNCHED();
  exclusive_scan(width.as<uint32_t>(), soff.as<uint32_t>(), nsl, nullptr, s, scratch);
  uint32_t tot = 0;
  CYC_CUDA(cudaMemcpyAsync(&tot, soff.as<uint32_t>() + nsl, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  const uint64_t words = (uint64_t)tot * 32u;
  sell.alloc((words ? words : 1) * 4, s);
  sdesc.alloc(((size_t)nsl + 1) * sizeof(uint4), s);
  k_sell_fill<<<grid_for((uint64_t)nsl * 32, 256, 8), 256, 0, s>>>(g.n, row_lo, nsl, np, g.o(), g.c(),
                                                                  width.as<uint32_t>(), soff.as<uint32_t>(),
                                                                  hmask.as<uint32_t>(), sell.as<uint32_t>(),
                                                                  sdesc.as<uint4>());
  CYC_LAUNCHED();
  return words;
}

void permute_bits(const uint32_t* src, const uint32_t* orig, uint32_t n, uint32_t* dst, cudaStream_t s) {
  if (!n) return;
  k_permute_bits<<<grid_for((uint64_t)n, 256, 8), 256, 0, s>>>(src, orig, n, dst);
  CYC_LAUNCHED();
}

bool build_plan(const DevCsr& snap, const DevCsr& gath, int layout, MapPlan& plan, cudaStream_t s) {
  if (const char* e = std::getenv("CYC_LAYOUT")) layout = std::atoi(e);
  if (plan.decided && plan.layout == layout) return false;
  const auto t0 = std::chrono::steady_clock::now();
  const bool dbg = std::getenv("CYC_DEBUG_TIMING") != nullptr;
  auto tm = t0;
  auto mark = [&](const char* what) {  // CYC_DEBUG_TIMING=1: host-observed phase times
    if (!dbg) return;
    CYC_CUDA(cudaStreamSynchronize(s));
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[cyc plan] %-10s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - tm).count());
    tm = now;
  };
  plan = MapPlan();
  plan.decided = true;
  plan.layout = layout;
  const uint32_t n = gath.n;
  if (layout == kLayoutIdentity || n < 64) return true;
  // a map buffer within ~1/3 of L2 stays resident in id order
  if (layout == kLayoutAuto && (uint64_t)n * 4 <= (40ull << 20)) return true;
  const uint32_t nw = (uint32_t)sm_count() * kPlanWarps;
  const uint32_t per_warp = div_up(div_up(n, nw), 32) * 32;
  DevBuf T((size_t)kBuckets * nw * 4, s), base((size_t)kBuckets * nw * 4 + 4, s), tot(kBuckets * 8, s);
  const uint32_t blocks = div_up(nw, kPlanWarps);
  k_plan_hist<<<blocks, kPlanWarps * 32, 0, s>>>(n, per_warp, snap.o(), nullptr, kBuckets - 1u, T.as<uint32_t>(), nw);
  CYC_LAUNCHED();
  k_plan_totals<<<kBuckets / 256, 256, 0, s>>>(T.as<uint32_t>(), nw, tot.as<unsigned long long>());
  CYC_LAUNCHED();
  std::vector<unsigned long long> ht(kBuckets);
  CYC_CUDA(cudaMemcpyAsync(ht.data(), tot.p, kBuckets * 8, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  // gathers taken by the n/8 most-gathered vertices (bucket lower bounds)
  auto lower = [](uint32_t b) -> double {
    if (b < 512) return b;
    const uint32_t lg = 9 + (b - 512) / 64, sub = (b - 512) % 64;
    return (double)(1ull << lg) * (1.0 + sub / 64.0);
  };
  double hot = 0, room = n / 8.0;
  for (uint32_t k = 0; k < kBuckets && room > 0; ++k) {
    const double take = std::min<double>(room, (double)ht[k]);
    hot += take * lower(kBuckets - 1 - k);
    room -= take;
  }
  mark("hist");
  plan.hot_share = gath.m ? std::min(1.0, hot / (double)gath.m) : 0.0;
  if (layout == kLayoutAuto && plan.hot_share < 0.5) return true;
  plan.relabel = true;
  const uint32_t np = (uint32_t)(((uint64_t)n + kRowPad - 1) / kRowPad * kRowPad);
  plan.orig.alloc(((size_t)np + 1) * 4, s);
  plan.perm.alloc((size_t)n * 4, s);
  DevBuf scratch;
  degree_order(snap.o(), gath.o(), n, plan.orig.as<uint32_t>(), plan.perm.as<uint32_t>(), s);
  mark("place");
  relayout(gath, plan.orig.as<uint32_t>(), plan.perm.as<uint32_t>(), plan.gath, scratch, s);
  mark("gath");
  relayout(snap, plan.orig.as<uint32_t>(), plan.perm.as<uint32_t>(), plan.snap, scratch, s);
  mark("snap");
  build_hslab(plan.gath, np, plan.hcol, plan.hrow, plan.n_hchunks, s);
  mark("heavy");
  plan.sell_words = build_sell(plan.gath, 0, np, np, plan.sell, plan.sdesc, s);  // map_run.cu pull_sell
  mark("sell");
  CYC_CUDA(cudaStreamSynchronize(s));
  plan.build_ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (dbg) {  // gathers covered by the first K storage positions (= prefix of the storage snapshot offsets)
    for (uint32_t k : {4096u, 16384u, 32768u, 65536u, 1u << 20, 1u << 23}) {
      if (k > n) break;
      uint32_t o = 0;
      CYC_CUDA(cudaMemcpy(&o, plan.snap.o() + k, 4, cudaMemcpyDeviceToHost));
      std::fprintf(stderr, "[cyc plan] first %8u positions take %.4f of the gathers\n", k, gath.m ? (double)o / gath.m : 0.0);
    }
  }
  if (dbg)
    std::fprintf(stderr, "[cyc plan] relabel n=%u m=%u hot_share=%.3f sell_words=%llu heavy_chunks=%u %.3f ms\n", n,
                 gath.m, plan.hot_share, (unsigned long long)plan.sell_words, plan.gath.n_heavy_chunks, plan.build_ms);
  return true;
}

}  // namespace cyc
