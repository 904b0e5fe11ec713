// build.cu — K1: device CSR construction from an edge log.
//
// Replaces build_snapshot (reference graph.cpp:63-105) and the gather-index
// construction of MaxPropagation (map_engine.cpp:9-19). Both are
// single-threaded counting sorts on the CPU; here the phases run as
// HBM-bound kernels over the whole log:
//   1. bucket histogram (2^14 rows per bucket, shared-memory counters; also
//      counts bucket runs in log order)
//   2. MSD partition log -> buckets in sub-chunks held in registers
//      (contiguous runs per bin): one pass for a bucket-local log, 4-bit
//      digits per pass for a scattered one
//   3. one CTA per bucket counting-sorts its rows in shared memory
//   4. per-row sort+dedup by length: registers (<=16), one warp in registers
//      (<=512), longer rows by an MSD split into ~256-value sub-buckets sorted
//      by warps (CTA fallback for overfull ones)
//   5. scan of unique counts, warp-flattened compaction into the final CSR.
// (n > 2^28: a flat atomic counting sort replaces 1-3.)
// Row offsets are u32 (snapshot edges < 2^32; checked by the caller).
#include <algorithm>
#include <chrono>
#include <vector>
#include <cstdio>
#include <cstdlib>

#include "build.cuh"

namespace cyc {

namespace {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr uint32_t kScanTile = kScanThreads * kScanItems;
constexpr uint32_t kSmallRow = 16;
constexpr uint32_t kWarpRow = 512;
constexpr uint32_t kMedRow = 4096;
constexpr int kMedThreads = 256;
constexpr uint32_t kBigTile = 4096;
constexpr int kBigThreads = 1024;

template <int THREADS>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* total) {
  __shared__ uint32_t warp_sums[THREADS / 32];
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  uint32_t incl = warp_incl_scan(x);
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint32_t s = lane < THREADS / 32 ? warp_sums[lane] : 0u;
    s = warp_incl_scan(s);
    if (lane < THREADS / 32) warp_sums[lane] = s;
  }
  __syncthreads();
  uint32_t base = wid ? warp_sums[wid - 1] : 0u;
  *total = warp_sums[THREADS / 32 - 1];
  __syncthreads();
  return base + incl - x;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t* __restrict__ in,
                                                               uint32_t n, uint32_t per_block,
                                                               uint32_t* __restrict__ bsum) {
  uint64_t lo = (uint64_t)blockIdx.x * per_block;
  uint64_t hi = lo + per_block < n ? lo + per_block : n;
  uint32_t s = 0;
  for (uint64_t i = lo + threadIdx.x; i < hi; i += kScanThreads) s += in[i];
  s = __reduce_add_sync(kFull, s);
  __shared__ uint32_t ws[kScanThreads / 32];
  if ((threadIdx.x & 31u) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t t = threadIdx.x < kScanThreads / 32 ? ws[threadIdx.x] : 0u;
    t = __reduce_add_sync(kFull, t);
    if (threadIdx.x == 0) bsum[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) k_scan_blocks(uint32_t* bsum, uint32_t nb, uint32_t* total) {
  uint32_t x = threadIdx.x < nb ? bsum[threadIdx.x] : 0u;
  uint32_t tot;
  uint32_t ex = block_excl_scan<1024>(x, &tot);
  if (threadIdx.x < nb) bsum[threadIdx.x] = ex;
  if (threadIdx.x == 0 && total) *total = tot;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_down(const uint32_t* in, uint32_t* out,
                                                             uint32_t n, uint32_t per_block,
                                                             const uint32_t* __restrict__ bsum) {
  uint64_t lo = (uint64_t)blockIdx.x * per_block;
  uint64_t hi = lo + per_block < n ? lo + per_block : n;
  uint32_t run = bsum[blockIdx.x];
  for (uint64_t t0 = lo; t0 < hi; t0 += kScanTile) {
    uint32_t v[kScanItems];
    uint64_t base = t0 + (uint64_t)threadIdx.x * kScanItems;
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      v[k] = base + k < hi ? in[base + k] : 0u;
      s += v[k];
    }
    uint32_t tot;
    uint32_t ex = block_excl_scan<kScanThreads>(s, &tot) + run;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      if (base + k < hi) out[base + k] = ex;
      ex += v[k];
    }
    run += tot;
  }
}

// ---------------------------------------------------------------- histogram
__global__ void k_hist(const uint2* __restrict__ edges, uint64_t m, uint32_t n, int key_dst,
                       uint32_t* __restrict__ cnt, uint32_t* __restrict__ err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < m; i0 += stride) {
    uint64_t i = i0 + threadIdx.x;
    uint32_t row = kNone;
    if (i < m) {
      uint2 e = edges[i];
      if (e.x >= n || e.y >= n) {
        *err = 1u;
      } else {
        row = key_dst ? e.y : e.x;
      }
    }
    uint32_t peers = __match_any_sync(kFull, row);
    if (row != kNone && (__ffs(peers) - 1) == (int)lane_id()) atomicAdd(cnt + row, __popc(peers));
  }
}

// Counting-down cursors: cnt[row] starts at the row length.
__global__ void k_scatter(const uint2* __restrict__ edges, uint64_t m, uint32_t n, int key_dst,
                          const uint32_t* __restrict__ roff, uint32_t* __restrict__ cnt,
                          uint32_t* __restrict__ raw) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < m; i0 += stride) {
    uint64_t i = i0 + threadIdx.x;
    uint32_t row = kNone, other = 0;
    if (i < m) {
      uint2 e = edges[i];
      if (e.x < n && e.y < n) {
        row = key_dst ? e.y : e.x;
        other = key_dst ? e.x : e.y;
      }
    }
    uint32_t peers = __match_any_sync(kFull, row);
    if (row != kNone) {
      int leader = __ffs(peers) - 1;
      uint32_t base = 0;
      if (leader == (int)lane_id()) base = atomicSub(cnt + row, (uint32_t)__popc(peers));
      base = __shfl_sync(peers, base, leader);
      uint32_t rank = __popc(peers & lanemask_lt());
      raw[roff[row] + base - 1u - rank] = other;
    }
  }
}

// ------------------------------------------------------------ small rows
template <int N>
__device__ __forceinline__ void sort_net(uint32_t (&a)[N]) {
  // bitonic network, ascending (N power of two)
#pragma unroll
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        int p = i ^ j;
        if (p > i) {
          bool up = (i & k) == 0;
          uint32_t x = a[i], y = a[p];
          if ((x > y) == up) {
            a[i] = y;
            a[p] = x;
          }
        }
      }
    }
  }
}

template <int N>
__device__ __forceinline__ uint32_t sort_small_row(uint32_t* __restrict__ seg, uint32_t d) {
  uint32_t a[N];
#pragma unroll
  for (int i = 0; i < N; ++i) a[i] = (uint32_t)i < d ? seg[i] : kNone;
  sort_net<N>(a);
  uint32_t k = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    if ((uint32_t)i < d && (i == 0 || a[i] != a[i - 1])) seg[k++] = a[i];
  }
  return k;
}

__global__ void k_sort_small(uint32_t n, const uint32_t* __restrict__ roff,
                             uint32_t* __restrict__ raw, uint32_t* __restrict__ ucnt,
                             uint32_t* __restrict__ med, uint32_t* __restrict__ big,
                             uint32_t* __restrict__ wrows,
                             uint32_t* __restrict__ counts /* [0]=med [1]=big [2]=warp */) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    uint32_t b = roff[v], d = roff[v + 1] - b;
    uint32_t* seg = raw + b;
    if (d <= 1) {
      ucnt[v] = d;
    } else if (d == 2) {
      uint32_t x = seg[0], y = seg[1];
      if (x == y) {
        ucnt[v] = 1;
      } else {
        seg[0] = min(x, y);
        seg[1] = max(x, y);
        ucnt[v] = 2;
      }
    } else if (d <= 4) {
      ucnt[v] = sort_small_row<4>(seg, d);
    } else if (d <= 8) {
      ucnt[v] = sort_small_row<8>(seg, d);
    } else if (d <= kSmallRow) {
      ucnt[v] = sort_small_row<16>(seg, d);
    } else if (d <= kWarpRow) {
      wrows[atomicAdd(counts + 2, 1u)] = v;
    } else {
      med[atomicAdd(counts + 0, 1u)] = v;  // long rows: split sort (sort_long_rows)
    }
  }
}

// Block-wide dedup of a sorted shared-memory array s[0..d) into seg, returns
// unique count (all threads).
template <int THREADS>
__device__ uint32_t block_unique_store(const uint32_t* s, uint32_t d, uint32_t prev_last,
                                       bool has_prev, uint32_t* seg_out) {
  // each thread handles a contiguous run of items
  const uint32_t per = (d + THREADS - 1) / THREADS;
  const uint32_t lo = threadIdx.x * per;
  const uint32_t hi = min(d, lo + per);
  uint32_t c = 0;
  for (uint32_t i = lo; i < hi; ++i) {
    bool first = i == 0 ? !has_prev || s[0] != prev_last : s[i] != s[i - 1];
    c += first;
  }
  uint32_t tot;
  uint32_t pos = block_excl_scan<THREADS>(c, &tot);
  for (uint32_t i = lo; i < hi; ++i) {
    bool first = i == 0 ? !has_prev || s[0] != prev_last : s[i] != s[i - 1];
    if (first) seg_out[pos++] = s[i];
  }
  return tot;
}

__device__ __forceinline__ void smem_bitonic(uint32_t* s, uint32_t P, int nthreads) {
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < P; i += nthreads) {
        uint32_t p = (j == (k >> 1)) ? (i ^ (k - 1)) : (i ^ j);
        if (p > i) {
          uint32_t x = s[i], y = s[p];
          if (x > y) {
            s[i] = y;
            s[p] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Hub rows: bitonic network (all-ascending "flip" formulation, so virtual
// +inf padding beyond d never moves) with every stage whose partner distance
// is below kBigTile run inside a shared-memory tile.
__device__ void big_tile_stages(uint32_t* s, uint32_t* g, uint32_t d, uint32_t t0, uint32_t kmax,
                                bool from_start) {
  // load tile
  for (uint32_t i = threadIdx.x; i < kBigTile; i += kBigThreads)
    s[i] = t0 + i < d ? g[t0 + i] : kNone;
  __syncthreads();
  if (from_start) {
    smem_bitonic(s, kBigTile, kBigThreads);
  } else {
    // only the half-cleaner tail j = kBigTile/2 .. 1 of merge size kmax
    (void)kmax;
    for (uint32_t j = kBigTile >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < kBigTile; i += kBigThreads) {
        uint32_t p = i ^ j;
        if (p > i) {
          uint32_t x = s[i], y = s[p];
          if (x > y) {
            s[i] = y;
            s[p] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t i = threadIdx.x; i < kBigTile; i += kBigThreads)
    if (t0 + i < d) g[t0 + i] = s[i];
  __syncthreads();
}

// Sorts and deduplicates g[0..d) in place with one 1024-thread CTA (bitonic
// in shared-memory tiles plus global merge stages); returns the unique count.
__device__ uint32_t cta_sort_unique_global(uint32_t* s, uint32_t* g, uint32_t d) {
  __shared__ uint32_t carry;
  uint32_t P = kBigTile;
  while (P < d) P <<= 1;
  for (uint32_t t0 = 0; t0 < d; t0 += kBigTile) big_tile_stages(s, g, d, t0, kBigTile, true);
  for (uint32_t k = kBigTile << 1; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j >= kBigTile; j >>= 1) {
      const bool flip = j == (k >> 1);
      for (uint32_t i = threadIdx.x; i < d; i += kBigThreads) {
        uint32_t p = flip ? (i ^ (k - 1)) : (i ^ j);
        if (p > i && p < d) {
          uint32_t x = g[i], y = g[p];
          if (x > y) {
            g[i] = y;
            g[p] = x;
          }
        }
      }
      __syncthreads();
    }
    for (uint32_t t0 = 0; t0 < d; t0 += kBigTile) big_tile_stages(s, g, d, t0, k, false);
  }
  // dedup tile by tile (writes never overtake reads: output index <= input index)
  uint32_t written = 0;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t t0 = 0; t0 < d; t0 += kBigTile) {
    uint32_t len = min(kBigTile, d - t0);
    for (uint32_t i = threadIdx.x; i < len; i += kBigThreads) s[i] = g[t0 + i];
    __syncthreads();
    uint32_t prev = carry;
    __syncthreads();
    uint32_t u = block_unique_store<kBigThreads>(s, len, prev, t0 > 0, g + written);
    if (threadIdx.x == 0) carry = s[len - 1];
    written += u;
    __syncthreads();
  }
  return written;
}

// ------------------------------------------------------------------ compact
// Rows of raw degree <= kWarpRow: one warp per 32 consecutive rows walks the
// concatenation of their unique prefixes 32 values per round, so the writes
// (a contiguous range of col) and the reads are coalesced.
__global__ void k_compact_rows(uint32_t n, const uint32_t* __restrict__ roff, const uint32_t* __restrict__ off,
                               const uint32_t* __restrict__ raw, uint32_t* __restrict__ col) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; v0 < n; v0 += stride) {
    const uint32_t v = v0 + lane;
    uint32_t src = 0, dst = 0, u = 0;
    if (v < n && roff[v + 1] - roff[v] <= kWarpRow) {  // longer rows: k_compact_list
      src = roff[v];
      dst = off[v];
      u = off[v + 1] - dst;
    }
    const uint32_t incl = warp_incl_scan(u);
    const uint32_t excl = incl - u;
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    for (uint32_t r = 0; r < total; r += 32u) {
      const uint32_t e = r + lane;
      uint32_t owner = 0;
#pragma unroll
      for (uint32_t step = 16; step >= 1; step >>= 1) {
        const uint32_t cand = owner + step;
        const uint32_t ex = __shfl_sync(kFull, excl, cand & 31u);
        if (cand < 32u && ex <= e) owner = cand;
      }
      const uint32_t os = __shfl_sync(kFull, src, owner);
      const uint32_t od = __shfl_sync(kFull, dst, owner);
      const uint32_t oe = __shfl_sync(kFull, excl, owner);
      if (e < total) col[od + (e - oe)] = raw[os + (e - oe)];
    }
  }
}

__global__ void k_compact_list(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ cnt,
                               const uint32_t* __restrict__ roff, const uint32_t* __restrict__ off,
                               const uint32_t* __restrict__ raw, uint32_t* __restrict__ col) {
  // one warp per long row (a CTA per row spent its time on the per-row
  // offset loads of short-ish rows)
  const uint32_t nrows = *cnt;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = gw; r < nrows; r += nw) {
    const uint32_t v = rows[r];
    const uint32_t b = roff[v], o = off[v], u = off[v + 1] - o;
#pragma unroll 4
    for (uint32_t i = lane; i < u; i += 32u) col[o + i] = __ldg(raw + b + i);
  }
}

__global__ void k_heavy_chunks(uint32_t n, const uint32_t* __restrict__ off, uint32_t heavy,
                               uint32_t chunk, uint4* __restrict__ out, uint32_t* __restrict__ cnt) {
  // warp-aggregated reservation, descriptors written by the whole warp (a hub
  // row has thousands of chunks)
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; v0 < n; v0 += stride) {
    const uint32_t v = v0 + lane;
    uint32_t b = 0, e = 0;
    if (v < n) {
      b = off[v];
      e = off[v + 1];
    }
    const uint32_t nc = v < n && e - b > heavy ? (e - b + chunk - 1) / chunk : 0u;
    const uint32_t incl = warp_incl_scan(nc);
    const uint32_t tot = __shfl_sync(kFull, incl, 31);
    if (!tot) continue;
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(cnt, tot);
    base = __shfl_sync(kFull, base, 0) + incl - nc;
    for (uint32_t hb = __ballot_sync(kFull, nc != 0); hb; hb &= hb - 1u) {
      const uint32_t l = __ffs(hb) - 1u;
      const uint32_t lb = __shfl_sync(kFull, b, l), le = __shfl_sync(kFull, e, l);
      const uint32_t ln = __shfl_sync(kFull, nc, l), lbase = __shfl_sync(kFull, base, l);
      for (uint32_t c = lane; c < ln; c += 32u) {
        const uint32_t cb = lb + c * chunk;
        out[lbase + c] = make_uint4(v0 + l, cb, min(le, cb + chunk), 0u);
      }
    }
  }
}

// Heavy rows split at column-block boundaries (cols are sorted, so each
// block's part of a row is one range), chunks grouped by column block: the
// pull pass walks the list in order, so at any time all warps gather from one
// L2-sized slice of the map vector (config 3: 268 MB vector, 126 MB L2).
__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* p, uint32_t len, uint32_t x) {
  uint32_t lo = 0, hi = len;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (p[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_heavy_blocks(uint32_t n, const uint32_t* __restrict__ off, const uint32_t* __restrict__ col,
                               uint32_t heavy, uint32_t chunk, uint32_t ncb, uint32_t width,
                               uint32_t* __restrict__ bcount, uint32_t* __restrict__ bcur, uint4* __restrict__ out) {
  // warp-aggregated per-block reservations (one atomic per warp and column
  // block instead of one per heavy row), descriptors written by the warp
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; v0 < n; v0 += stride) {
    const uint32_t v = v0 + lane;
    uint32_t b = 0, e = 0;
    if (v < n) {
      b = off[v];
      e = off[v + 1];
    }
    const bool hv = v < n && e - b > heavy;
    if (!__any_sync(kFull, hv)) continue;
    uint32_t lo = 0;
    for (uint32_t j = 0; j < ncb; ++j) {
      uint32_t hi = 0, nc = 0;
      if (hv) {
        const uint64_t bound = (uint64_t)(j + 1) * width;
        hi = j + 1 == ncb || bound > 0xFFFFFFFFull
                 ? e - b
                 : lo + lower_bound_u32(col + b + lo, e - b - lo, (uint32_t)bound);
        nc = (hi - lo + chunk - 1) / chunk;
      }
      const uint32_t incl = warp_incl_scan(nc);
      const uint32_t tot = __shfl_sync(kFull, incl, 31);
      if (tot) {
        if (!out) {
          if (lane == 0) atomicAdd(bcount + j, tot);
        } else {
          uint32_t base = 0;
          if (lane == 0) base = atomicAdd(bcur + j, tot);
          base = __shfl_sync(kFull, base, 0) + incl - nc;
          for (uint32_t hb = __ballot_sync(kFull, nc != 0); hb; hb &= hb - 1u) {
            const uint32_t l = __ffs(hb) - 1u;
            const uint32_t lb = __shfl_sync(kFull, b + lo, l), le = __shfl_sync(kFull, b + hi, l);
            const uint32_t ln = __shfl_sync(kFull, nc, l), lbase = __shfl_sync(kFull, base, l);
            for (uint32_t c = lane; c < ln; c += 32u) {
              const uint32_t cb = lb + c * chunk;
              out[lbase + c] = make_uint4(v0 + l, cb, min(le, cb + chunk), 0u);
            }
          }
        }
      }
      lo = hi;
    }
  }
}

__global__ void k_max_degree(uint32_t n, const uint32_t* __restrict__ off, uint32_t* out) {
  uint32_t mx = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride)
    mx = max(mx, off[v + 1] - off[v]);
  mx = __reduce_max_sync(kFull, mx);
  if ((threadIdx.x & 31u) == 0) atomicMax(out, mx);
}

// ------------------------------------------------- MSD bucket partition
// Counting sort by row done as two levels so no atomic or write ever lands in
// an n-sized random array: (1) bucket = row >> sh histogram in shared memory,
// (2) partition of the log into buckets, (3) one CTA per bucket counting-sorts
// its <= 2^sh rows in shared memory and emits the row offsets.
constexpr int kPartThreads = 1024;
constexpr uint32_t kBucketLog = 14;  // rows per bucket (pass 3 counters in smem)

__global__ void __launch_bounds__(kPartThreads) k_bucket_hist(const uint2* __restrict__ edges, uint64_t m,
                                                              uint32_t n, int key_dst, uint32_t sh,
                                                              uint32_t nb, uint64_t per_block,
                                                              uint32_t* __restrict__ bcnt,
                                                              uint32_t* __restrict__ err,
                                                              unsigned long long* __restrict__ changes) {
  // also counts log positions whose bucket differs from the previous one
  // (adjacent lanes), i.e. how many bucket runs the log order has
  extern __shared__ uint32_t h[];
  __shared__ uint32_t sh_changes;
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) h[b] = 0;
  if (threadIdx.x == 0) sh_changes = 0;
  __syncthreads();
  const uint64_t lo = blockIdx.x * per_block, hi = min(m, lo + per_block);
  uint32_t my_changes = 0;
  for (uint64_t i0 = lo; i0 < hi; i0 += blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    uint32_t bk = 0xFFFFFFFFu;
    if (i < hi) {
      const uint2 e = edges[i];
      if (e.x >= n || e.y >= n) {
        *err = 1u;
      } else {
        bk = (key_dst ? e.y : e.x) >> sh;
        atomicAdd(&h[bk], 1u);
      }
    }
    const uint32_t prev = __shfl_up_sync(kFull, bk, 1);
    my_changes += __popc(__ballot_sync(kFull, (threadIdx.x & 31u) && bk != prev && i < hi));
  }
  if ((threadIdx.x & 31u) == 0 && my_changes) atomicAdd(&sh_changes, my_changes);
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x)
    if (h[b]) atomicAdd(bcnt + b, h[b]);
  if (threadIdx.x == 0 && sh_changes) atomicAdd(changes, (unsigned long long)sh_changes);
}

// Multi-pass MSD partition of the log into bucket order, kDigit bits of the
// bucket id per pass (the first pass takes the remainder). Measured on
// config 3 (1.07 G pairs, 4096 buckets): a pass costs ~5-6 ms at fan-out 16
// but 8-21 ms at fan-out 64 and ~28 ms at 1024 (more concurrently open
// output regions spread over the array); a single pass at fan-out 4096 wrote
// L2 lines half-filled and paid ~3x the payload in DRAM traffic. Each block
// works on kSubChunk-element sub-chunks (histogram, one reservation per bin,
// scatter) so the second read of a sub-chunk hits L2 and every bin receives a
// contiguous run.
constexpr uint32_t kDigitDefault = 4;
static uint32_t part_digit() {
  static const uint32_t v = [] {
    const char* e = getenv("CYC_PART_DIGIT");  // tuning knob
    const uint32_t d = e ? (uint32_t)atoi(e) : kDigitDefault;
    return d >= 1 && d <= 14 ? d : kDigitDefault;
  }();
  return v;
}
constexpr uint32_t kSubChunk = 16384;

template <bool FROM_EDGES>
__global__ void __launch_bounds__(kPartThreads) k_part(const void* __restrict__ in, uint64_t m, uint32_t n,
                                                       int key_dst, uint32_t shift, uint32_t nbins,
                                                       uint32_t* __restrict__ cursor,
                                                       unsigned long long* __restrict__ out, uint32_t slog) {
  // each thread keeps its kPer elements of the sub-chunk in registers between
  // the histogram and the scatter (16 independent loads in flight, one read)
  constexpr uint32_t kPer = kSubChunk / kPartThreads;
  extern __shared__ uint32_t h[];
  const uint64_t nsub = (m + kSubChunk - 1) / kSubChunk;
  for (uint64_t c = blockIdx.x; c < nsub; c += gridDim.x) {
    const uint64_t lo = c * kSubChunk, hi = min(m, lo + kSubChunk);
    // later passes: the input is sorted by bin >> slog, so only the bins of
    // the groups between the sub-chunk's first and last element can occur
    uint32_t b0 = 0, b1 = nbins;
    if (!FROM_EDGES) {
      const unsigned long long* t = reinterpret_cast<const unsigned long long*>(in);
      b0 = (((uint32_t)(t[lo] >> 32) >> shift) >> slog) << slog;
      b1 = min(nbins, ((((uint32_t)(t[hi - 1] >> 32) >> shift) >> slog) + 1) << slog);
    }
    for (uint32_t b = b0 + threadIdx.x; b < b1; b += blockDim.x) h[b - b0] = 0;
    // all kPer loads are issued before any is used (a use between loads made
    // the compiler wait on each one in turn); edges are validated afterwards
    const unsigned long long* raw = reinterpret_cast<const unsigned long long*>(in);
    unsigned long long v[kPer];
#pragma unroll
    for (uint32_t k = 0; k < kPer; ++k) {
      const uint64_t i = lo + k * kPartThreads + threadIdx.x;
      v[k] = i < hi ? __ldg(raw + i) : ~0ull;
    }
    if (FROM_EDGES) {
#pragma unroll
      for (uint32_t k = 0; k < kPer; ++k) {
        if (v[k] == ~0ull) continue;
        const uint32_t x = (uint32_t)v[k], y = (uint32_t)(v[k] >> 32);  // uint2 {src, dst}
        const uint32_t row = key_dst ? y : x, other = key_dst ? x : y;
        v[k] = (x < n && y < n) ? ((unsigned long long)row << 32) | other : ~0ull;
      }
    }
    __syncthreads();
#pragma unroll
    for (uint32_t k = 0; k < kPer; ++k)
      if (v[k] != ~0ull) atomicAdd(&h[((uint32_t)(v[k] >> 32) >> shift) - b0], 1u);
    __syncthreads();
    for (uint32_t b = b0 + threadIdx.x; b < b1; b += blockDim.x) {
      const uint32_t x = h[b - b0];
      h[b - b0] = x ? atomicAdd(cursor + b, x) : 0u;
    }
    __syncthreads();
    // reserve every slot first, then store: the stores no longer wait on
    // each shared-memory atomic in turn
    constexpr uint32_t kBatch = 8;
#pragma unroll
    for (uint32_t k0 = 0; k0 < kPer; k0 += kBatch) {
      uint32_t pos[kBatch];
#pragma unroll
      for (uint32_t k = 0; k < kBatch; ++k)
        pos[k] = v[k0 + k] != ~0ull ? atomicAdd(&h[((uint32_t)(v[k0 + k] >> 32) >> shift) - b0], 1u) : 0u;
#pragma unroll
      for (uint32_t k = 0; k < kBatch; ++k)
        if (v[k0 + k] != ~0ull) out[pos[k]] = v[k0 + k];
    }
    __syncthreads();
  }
}

// cursor of bin x at (bucket shift + slog) = start of its first bucket
__global__ void k_super_cursors(const uint32_t* __restrict__ bbase, uint32_t nb, uint32_t ns, uint32_t* cur,
                                uint32_t slog) {
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += gridDim.x * blockDim.x)
    cur[s] = bbase[min(nb, s << slog)];
}

__global__ void __launch_bounds__(kPartThreads) k_bucket_rows(const unsigned long long* __restrict__ tmp,
                                                              const uint32_t* __restrict__ bbase,
                                                              uint32_t n, uint32_t sh, uint32_t nb,
                                                              uint32_t* __restrict__ roff,
                                                              uint32_t* __restrict__ raw) {
  extern __shared__ uint32_t cnt[];  // 2^sh row counters, then row cursors
  __shared__ uint32_t warp_sums[kPartThreads / 32];
  const uint32_t rows_per = 1u << sh;
  const uint32_t per_thread = rows_per / kPartThreads;
  for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const uint32_t r0 = b << sh;
    const uint32_t nr = min(rows_per, n - r0);
    const uint32_t lo = bbase[b], hi = bbase[b + 1];
    for (uint32_t j = threadIdx.x; j < rows_per; j += blockDim.x) cnt[j] = 0;
    __syncthreads();
    // 4 independent loads per thread per iteration (one load in flight per
    // thread left the bucket latency-bound)
    constexpr uint32_t kU = 4;
    for (uint32_t i0 = lo + threadIdx.x; i0 < hi; i0 += kU * blockDim.x) {
      unsigned long long t[kU];
#pragma unroll
      for (uint32_t u = 0; u < kU; ++u) {
        const uint32_t i = i0 + u * blockDim.x;
        t[u] = i < hi ? __ldg(tmp + i) : ~0ull;
      }
#pragma unroll
      for (uint32_t u = 0; u < kU; ++u)
        if (t[u] != ~0ull) atomicAdd(&cnt[(uint32_t)(t[u] >> 32) - r0], 1u);
    }
    __syncthreads();
    // exclusive scan of cnt: each thread owns per_thread consecutive rows
    uint32_t run = 0;
    const uint32_t j0 = threadIdx.x * per_thread;
    for (uint32_t k = 0; k < per_thread; ++k) run += cnt[j0 + k];
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    uint32_t incl = warp_incl_scan(run);
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      uint32_t w = warp_sums[lane];
      w = warp_incl_scan(w);
      warp_sums[lane] = w;
    }
    __syncthreads();
    uint32_t pre = (wid ? warp_sums[wid - 1] : 0u) + incl - run;
    for (uint32_t k = 0; k < per_thread; ++k) {
      const uint32_t c = cnt[j0 + k];
      cnt[j0 + k] = lo + pre;
      if (j0 + k < nr) roff[r0 + j0 + k] = lo + pre;
      pre += c;
    }
    __syncthreads();
    for (uint32_t i0 = lo + threadIdx.x; i0 < hi; i0 += kU * blockDim.x) {
      unsigned long long t[kU];
      uint32_t pos[kU];
#pragma unroll
      for (uint32_t u = 0; u < kU; ++u) {
        const uint32_t i = i0 + u * blockDim.x;
        t[u] = i < hi ? __ldg(tmp + i) : ~0ull;
      }
#pragma unroll
      for (uint32_t u = 0; u < kU; ++u)
        pos[u] = t[u] != ~0ull ? atomicAdd(&cnt[(uint32_t)(t[u] >> 32) - r0], 1u) : 0u;
#pragma unroll
      for (uint32_t u = 0; u < kU; ++u)
        if (t[u] != ~0ull) raw[pos[u]] = (uint32_t)t[u];
    }
    if (b == nb - 1 && threadIdx.x == 0) roff[n] = hi;
    __syncthreads();
  }
}

// ------------------------------------------------- warp sort (17..256 / row)
// Bitonic network over 32*E register slots of one warp (slot i = r*32 + lane,
// +inf padding), then in-register dedup; the warp writes the unique values
// back to the front of its row segment.
template <int E>
__device__ uint32_t warp_sort_row(uint32_t* seg, uint32_t d) {
  constexpr uint32_t N = 32u * E;
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t a[E];
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const uint32_t i = r * 32u + lane;
    a[r] = i < d ? seg[i] : kNone;
  }
#pragma unroll
  for (uint32_t k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int rj = (int)(j >> 5);
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int rp = r ^ rj;
          if (rp > r) {
            const uint32_t i = r * 32u + lane;
            const bool up = (i & k) == 0;
            const uint32_t x = a[r], y = a[rp];
            if ((x > y) == up) {
              a[r] = y;
              a[rp] = x;
            }
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const uint32_t i = r * 32u + lane;
          const bool up = (i & k) == 0;
          const bool lower = (lane & j) == 0;
          const uint32_t y = __shfl_xor_sync(kFull, a[r], j);
          a[r] = (lower == up) ? min(a[r], y) : max(a[r], y);
        }
      }
    }
  }
  uint32_t written = 0;
  uint32_t prev_last = kNone;  // last element of the previous register row (slot r*32-1)
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const uint32_t i = r * 32u + lane;
    uint32_t prev = __shfl_up_sync(kFull, a[r], 1);
    if (lane == 0) prev = prev_last;
    const bool first = i < d && (i == 0 || a[r] != prev);
    const uint32_t bal = __ballot_sync(kFull, first);
    if (first) seg[written + __popc(bal & lanemask_lt())] = a[r];
    written += __popc(bal);
    prev_last = __shfl_sync(kFull, a[r], 31);
  }
  return written;
}

__global__ void k_sort_warp(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ counts,
                            const uint32_t* __restrict__ roff, uint32_t* __restrict__ raw,
                            uint32_t* __restrict__ ucnt) {
  const uint32_t nrows = counts[2];
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = gw; r < nrows; r += nw) {
    const uint32_t v = rows[r];
    const uint32_t b = roff[v], d = roff[v + 1] - b;
    uint32_t u;
    if (d <= 64) u = warp_sort_row<2>(raw + b, d);
    else if (d <= 128) u = warp_sort_row<4>(raw + b, d);
    else if (d <= 256) u = warp_sort_row<8>(raw + b, d);
    else u = warp_sort_row<16>(raw + b, d);
    if ((threadIdx.x & 31u) == 0) ucnt[v] = u;
  }
}

// ---------------------------------------------------- long rows: MSD split
// Rows longer than kWarpRow (R-MAT hubs reach millions of columns) are split
// by the high bits of (col - row_min) into a power-of-two number of
// sub-buckets of ~kSubTarget values; each sub-bucket is then sorted and
// deduplicated by one warp in registers (warp_sort_row), the rare overfull
// ones by a CTA. Sub-buckets cover disjoint, ordered value ranges, so their
// concatenation is the sorted unique row. Every pass is spread over all SMs
// (kSplitChunk-element chunks), where a per-row sort put one hub on one CTA.
constexpr uint32_t kSubTarget = 256;
constexpr uint32_t kSplitChunk = 4096;
constexpr uint32_t kSplitThreads = 1024;
constexpr uint32_t kSplitBins = 8192;  // shared-memory histogram bins per chunk

__device__ __forceinline__ uint32_t ceil_log2(uint64_t x) {  // smallest b with 2^b >= x
  return x <= 1 ? 0u : 64u - __clzll(x - 1);
}

// per long row r: chunk count (SoA: rw[0..n) degrees, rw[n..2n) chunks)
__global__ void k_split_setup(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ cts,
                              const uint32_t* __restrict__ roff, uint32_t* nch, uint32_t* rmin, uint32_t* rmax) {
  const uint32_t nr = cts[0];
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += gridDim.x * blockDim.x) {
    const uint32_t v = rows[r];
    const uint32_t d = roff[v + 1] - roff[v];
    nch[r] = (d + kSplitChunk - 1) / kSplitChunk;
    rmin[r] = kNone;
    rmax[r] = 0;
  }
}

__global__ void k_split_desc(const uint32_t* __restrict__ cts, const uint32_t* __restrict__ chbase,
                             uint2* desc) {
  const uint32_t nr = cts[0];
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += gridDim.x * blockDim.x)
    for (uint32_t c = chbase[r]; c < chbase[r + 1]; ++c) desc[c] = make_uint2(r, c - chbase[r]);
}

__global__ void __launch_bounds__(kSplitThreads) k_split_minmax(const uint2* __restrict__ desc, uint32_t nchunks,
                                                                const uint32_t* __restrict__ rows,
                                                                const uint32_t* __restrict__ roff,
                                                                const uint32_t* __restrict__ raw, uint32_t* rmin,
                                                                uint32_t* rmax) {
  for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint2 dc = desc[c];
    const uint32_t v = rows[dc.x];
    const uint32_t b = roff[v] + dc.y * kSplitChunk, e = min(roff[v + 1], b + kSplitChunk);
    uint32_t lo = kNone, hi = 0;
    for (uint32_t i = b + threadIdx.x; i < e; i += blockDim.x) {
      lo = min(lo, raw[i]);
      hi = max(hi, raw[i]);
    }
    lo = __reduce_min_sync(kFull, lo);
    hi = __reduce_max_sync(kFull, hi);
    if ((threadIdx.x & 31u) == 0) {
      atomicMin(rmin + dc.x, lo);
      atomicMax(rmax + dc.x, hi);
    }
  }
}

// nsub = next power of two of ceil(d / kSubTarget), capped by the value range
__global__ void k_split_nsub(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ cts,
                             const uint32_t* __restrict__ roff, const uint32_t* __restrict__ rmin,
                             const uint32_t* __restrict__ rmax, uint32_t* nsub, uint32_t* shift) {
  const uint32_t nr = cts[0];
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += gridDim.x * blockDim.x) {
    const uint32_t v = rows[r];
    const uint32_t d = roff[v + 1] - roff[v];
    const uint32_t rb = ceil_log2((uint64_t)(rmax[r] - rmin[r]) + 1);  // value-range bits
    uint32_t sb = ceil_log2((d + kSubTarget - 1) / kSubTarget);
    if (sb > rb) sb = rb;
    nsub[r] = 1u << sb;
    shift[r] = rb - sb;
  }
}

template <bool SCATTER>
__global__ void __launch_bounds__(kSplitThreads) k_split_bins(const uint2* __restrict__ desc, uint32_t nchunks,
                                                              const uint32_t* __restrict__ rows,
                                                              const uint32_t* __restrict__ roff,
                                                              const uint32_t* __restrict__ raw,
                                                              const uint32_t* __restrict__ rmin,
                                                              const uint32_t* __restrict__ shift,
                                                              const uint32_t* __restrict__ nsub,
                                                              const uint32_t* __restrict__ subbase,
                                                              uint32_t* cnt_or_cur, uint32_t* tmp) {
  __shared__ uint32_t h[kSplitBins];
  for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint2 dc = desc[c];
    const uint32_t r = dc.x, v = rows[r];
    const uint32_t b = roff[v] + dc.y * kSplitChunk, e = min(roff[v + 1], b + kSplitChunk);
    const uint32_t lo = rmin[r], sh = shift[r], ns = nsub[r], sb = subbase[r];
    if (ns > kSplitBins) {  // very long rows: few elements per bin, global atomics
      for (uint32_t i = b + threadIdx.x; i < e; i += blockDim.x) {
        const uint32_t x = raw[i];
        const uint32_t bin = (x - lo) >> sh;
        if (SCATTER) tmp[atomicAdd(cnt_or_cur + sb + bin, 1u)] = x;
        else atomicAdd(cnt_or_cur + sb + bin, 1u);
      }
      continue;
    }
    for (uint32_t k = threadIdx.x; k < ns; k += blockDim.x) h[k] = 0;
    __syncthreads();
    for (uint32_t i = b + threadIdx.x; i < e; i += blockDim.x) atomicAdd(&h[(raw[i] - lo) >> sh], 1u);
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < ns; k += blockDim.x) {
      const uint32_t x = h[k];
      if (SCATTER) h[k] = x ? atomicAdd(cnt_or_cur + sb + k, x) : 0u;  // reserve: h becomes the base
      else if (x) atomicAdd(cnt_or_cur + sb + k, x);
    }
    __syncthreads();
    if (SCATTER) {
      for (uint32_t i = b + threadIdx.x; i < e; i += blockDim.x) {
        const uint32_t x = raw[i];
        tmp[atomicAdd(&h[(x - lo) >> sh], 1u)] = x;
      }
    }
    __syncthreads();  // h is reused by the next chunk
  }
}

// one warp per sub-bucket: sort + dedup in place; overfull ones are listed
__global__ void k_split_sort(uint32_t S, const uint32_t* __restrict__ soff, uint32_t* tmp, uint32_t* usub,
                             uint32_t* over, uint32_t* nover) {
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t sI = gw; sI < S; sI += nw) {
    const uint32_t b = soff[sI], d = soff[sI + 1] - b;
    uint32_t u;
    if (d <= 1) u = d;
    else if (d <= 64) u = warp_sort_row<2>(tmp + b, d);
    else if (d <= 128) u = warp_sort_row<4>(tmp + b, d);
    else if (d <= 256) u = warp_sort_row<8>(tmp + b, d);
    else if (d <= kWarpRow) u = warp_sort_row<16>(tmp + b, d);
    else {
      if ((threadIdx.x & 31u) == 0) over[atomicAdd(nover, 1u)] = sI;
      continue;
    }
    if ((threadIdx.x & 31u) == 0) usub[sI] = u;
  }
}

__global__ void __launch_bounds__(kBigThreads) k_split_sort_over(const uint32_t* __restrict__ over,
                                                                 const uint32_t* __restrict__ nover,
                                                                 const uint32_t* __restrict__ soff, uint32_t* tmp,
                                                                 uint32_t* usub) {
  __shared__ uint32_t s[kBigTile];
  const uint32_t no = *nover;
  for (uint32_t k = blockIdx.x; k < no; k += gridDim.x) {
    const uint32_t sI = over[k];
    const uint32_t b = soff[sI], d = soff[sI + 1] - b;
    uint32_t u;
    if (d <= kBigTile) {
      uint32_t P = 1;
      while (P < d) P <<= 1;
      for (uint32_t i = threadIdx.x; i < P; i += kBigThreads) s[i] = i < d ? tmp[b + i] : kNone;
      __syncthreads();
      smem_bitonic(s, P, kBigThreads);
      u = block_unique_store<kBigThreads>(s, d, 0, false, tmp + b);
    } else {
      u = cta_sort_unique_global(s, tmp + b, d);
    }
    if (threadIdx.x == 0) usub[sI] = u;
    __syncthreads();
  }
}

// one warp per sub-bucket: unique values to their place in the row
__global__ void k_split_write(uint32_t S, uint32_t nr, const uint32_t* __restrict__ rows,
                              const uint32_t* __restrict__ roff, const uint32_t* __restrict__ subbase,
                              const uint32_t* __restrict__ soff, const uint32_t* __restrict__ uoff,
                              const uint32_t* __restrict__ tmp, uint32_t* raw, uint32_t* ucnt) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t sI = gw; sI < S; sI += nw) {
    uint32_t lo = 0, hi = nr;  // row r: subbase[r] <= sI < subbase[r+1]
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (subbase[mid] <= sI) lo = mid; else hi = mid;
    }
    const uint32_t v = rows[lo];
    const uint32_t first = uoff[subbase[lo]];
    const uint32_t u = uoff[sI + 1] - uoff[sI];
    uint32_t* dst = raw + roff[v] + (uoff[sI] - first);
    const uint32_t* src = tmp + soff[sI];
    for (uint32_t i = lane; i < u; i += 32u) dst[i] = src[i];
    if (sI == subbase[lo] && lane == 0) ucnt[v] = uoff[subbase[lo + 1]] - first;
  }
}


// per K in {1,2,4,8}: rows longer than K and the edges beyond K
__global__ void k_ell_hist(uint32_t n, const uint32_t* __restrict__ off,
                           unsigned long long* __restrict__ out /* [8] */) {
  unsigned long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    const uint32_t d = off[v + 1] - off[v];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t k = 1u << i;
      if (d > k) {
        acc[2 * i] += 1;
        acc[2 * i + 1] += d - k;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    unsigned long long x = acc[i];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
    if ((threadIdx.x & 31u) == 0 && x) atomicAdd(out + i, x);
  }
}

// Column-major slab of the first K columns of every row (rows padded to np,
// sentinel np for absent entries); heavy rows get only sentinels (a separate
// chunk pass owns them) and, like rows longer than K, their ovf bit.
__global__ void k_ell_fill(uint32_t n, uint32_t np, const uint32_t* __restrict__ off,
                           const uint32_t* __restrict__ col, uint32_t K, uint32_t heavy,
                           uint32_t* __restrict__ ell, uint32_t* __restrict__ ovf) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; v0 < np; v0 += stride) {
    const uint32_t v = v0 + lane;
    bool over = false;
    uint32_t b = 0, d = 0;
    if (v < n) {
      b = off[v];
      d = off[v + 1] - b;
      over = d > K;
      if (d > heavy) d = 0;
    }
    for (uint32_t k = 0; k < K; ++k) ell[(size_t)k * np + v] = k < d ? col[b + k] : np;
    const uint32_t w = __ballot_sync(kFull, over);
    if (lane == 0) ovf[v0 >> 5] = w;
  }
}

}  // namespace

void build_ell(DevCsr& g, cudaStream_t s) {
  g.ell_k = 0;
  g.ell_n = 0;
  if (!g.n) return;
  DevBuf h(64, s);
  CYC_CUDA(cudaMemsetAsync(h.p, 0, 64, s));
  k_ell_hist<<<grid_for(g.n, 256, 8), 256, 0, s>>>(g.n, g.o(), h.as<unsigned long long>());
  CYC_LAUNCHED();
  unsigned long long hh[8];
  CYC_CUDA(cudaMemcpyAsync(hh, h.p, 64, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  // bytes per dense step: slab reads 4Kn; overflow rows add offsets (8 B) and
  // their remaining columns (4 B each)
  uint32_t best_k = 1;
  double best = 1e300;
  for (int i = 0; i < 4; ++i) {
    const double cost = 4.0 * (1u << i) * g.n + 8.0 * (double)hh[2 * i] + 4.0 * (double)hh[2 * i + 1];
    if (cost < best * 0.97) {  // prefer narrower slabs on near-ties
      best = cost;
      best_k = 1u << i;
    }
  }
  g.ell_k = best_k;
  const uint32_t np = (uint32_t)(((uint64_t)g.n + kRowPad - 1) / kRowPad * kRowPad);
  g.ell_n = np;
  g.ell.alloc((size_t)best_k * np * 4, s);
  const size_t words = (size_t)np / 32 + 1;
  g.ovf.alloc(words * 4, s);
  CYC_CUDA(cudaMemsetAsync(g.ovf.p, 0, words * 4, s));
  k_ell_fill<<<grid_for(np, 256, 8), 256, 0, s>>>(g.n, np, g.o(), g.c(), best_k,
                                                  g.heavy_deg ? g.heavy_deg : 0xFFFFFFFFu,
                                                  g.ell.as<uint32_t>(), g.ovf.as<uint32_t>());
  CYC_LAUNCHED();
}

int sm_count() {
  static int c = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return c;
}

uint32_t grid_for(uint64_t items, int threads, int per_sm) {
  uint64_t want = (items + threads - 1) / threads;
  uint64_t cap = (uint64_t)sm_count() * per_sm;
  if (want > cap) want = cap;
  return want ? (uint32_t)want : 1u;
}

void exclusive_scan(const uint32_t* in, uint32_t* out, uint32_t n, uint32_t* total,
                    cudaStream_t s, DevBuf& scratch) {
  // out has n+1 entries; out[n] = total (also written to *total if non-null, device ptr)
  uint32_t nb = div_up(n ? n : 1, kScanTile);
  if (nb > 1024) nb = 1024;
  uint32_t per_block = div_up(div_up(n ? n : 1, nb), kScanTile) * kScanTile;
  nb = div_up(n ? n : 1, per_block);
  if (scratch.bytes < (nb + 1) * sizeof(uint32_t)) scratch.alloc((nb + 1) * sizeof(uint32_t), s);
  uint32_t* bsum = scratch.as<uint32_t>();
  k_scan_reduce<<<nb, kScanThreads, 0, s>>>(in, n, per_block, bsum);
  CYC_LAUNCHED();
  k_scan_blocks<<<1, 1024, 0, s>>>(bsum, nb, out + n);
  CYC_LAUNCHED();
  k_scan_down<<<nb, kScanThreads, 0, s>>>(in, out, n, per_block, bsum);
  CYC_LAUNCHED();
  if (total) CYC_CUDA(cudaMemcpyAsync(total, out + n, 4, cudaMemcpyDeviceToDevice, s));
}

// Builds a deduplicated, row-sorted CSR keyed by one half of each logged pair.
// Row offsets (roff, n+1) and the bucketed log (raw) of the counting sort.
static void count_sort_rows(const uint2* e2, uint64_t m_log, uint32_t n, int key_dst, cudaStream_t s,
                            uint32_t* roff, uint32_t* raw, uint32_t* d_err, BuildArena& ar) {
  DevBuf& scratch = ar.scratch;
  if (n <= (1u << 28) && m_log > 0) {
    const uint32_t sh = kBucketLog;
    const uint32_t nb = (uint32_t)(((uint64_t)n + (1u << sh) - 1) >> sh);
    static const bool attr = [] {  // thread-safe one-time init
      CYC_CUDA(cudaFuncSetAttribute(k_bucket_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
      CYC_CUDA(cudaFuncSetAttribute(k_part<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
      CYC_CUDA(cudaFuncSetAttribute(k_part<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
      CYC_CUDA(cudaFuncSetAttribute(k_bucket_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
      return true;
    }();
    (void)attr;
    uint32_t* bcnt = ar.get<uint32_t>(ar.bcnt, ((size_t)nb + 4) * 4, s);
    unsigned long long* changes = reinterpret_cast<unsigned long long*>(bcnt + ((nb + 2) & ~1u));
    uint32_t* bbase = ar.get<uint32_t>(ar.bbase, ((size_t)nb + 2) * 4, s);
    uint32_t* bcur = ar.get<uint32_t>(ar.bcur, ((size_t)nb + 1) * 4, s);
    unsigned long long* tmp = ar.get<unsigned long long>(ar.tmp, m_log * 8, s);
    CYC_CUDA(cudaMemsetAsync(bcnt, 0, ((size_t)nb + 4) * 4, s));
    const uint32_t blocks = (uint32_t)std::min<uint64_t>((uint64_t)sm_count() * 2, (m_log + 4095) / 4096);
    const uint64_t per_block = (m_log + blocks - 1) / blocks;
    k_bucket_hist<<<blocks, kPartThreads, nb * 4, s>>>(e2, m_log, n, key_dst, sh, nb, per_block,
                                                       bcnt, d_err, changes);
    CYC_LAUNCHED();
    exclusive_scan(bcnt, bbase, nb, nullptr, s, scratch);
    uint32_t m_ok = 0;  // valid logged edges (invalid ones were counted nowhere)
    unsigned long long runs = 0;
    CYC_CUDA(cudaMemcpyAsync(&m_ok, bbase + nb, 4, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaMemcpyAsync(&runs, changes, 8, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
    // partition passes: after pass j the elements are sorted by
    // row >> (sh + rem_j), rem_j = bucket-id bits still unsorted; the last
    // pass lands in tmp
    // A log whose order is already bucket-local (config 4's BFS-ordered
    // product log: few bucket runs per sub-chunk) partitions in one pass at
    // full fan-out (41 vs 61 ms on config 4); a scattered one (RMAT) takes
    // kDigit-bit passes; logs of <= 256 MB at most two passes (config 2:
    // 1.5 ms vs 1.7 for one or three).
    uint32_t bits = 0;
    while ((1u << bits) < nb) ++bits;
    const bool local = (double)runs * kSubChunk <= 64.0 * (double)m_log;
    const bool small = m_log * 8 <= (256ull << 20);
    const uint32_t D = local ? 32u : small ? std::max(6u, (bits + 1) / 2) : part_digit();
    const uint32_t passes = bits ? (bits + D - 1) / D : 1;
    if (getenv("CYC_PART_DEBUG"))
      fprintf(stderr, "partition: m %llu nb %u runs %llu (%.1f per sub-chunk) passes %u\n",
              (unsigned long long)m_log, nb, runs, (double)runs * kSubChunk / (double)(m_log ? m_log : 1), passes);
    unsigned long long* tmp2 = ar.get<unsigned long long>(ar.tmp2, passes > 1 ? m_log * 8 : 8, s);
    const uint32_t pblocks = (uint32_t)std::min<uint64_t>((uint64_t)sm_count() * 2, (m_log + kSubChunk - 1) / kSubChunk);
    const void* src = e2;
    uint64_t m_in = m_log;
    uint32_t rem = bits;
    for (uint32_t j = 0; j < passes; ++j) {
      const uint32_t take = j == 0 ? bits - D * (passes - 1) : D;
      const uint32_t rem_in = rem;
      rem -= std::min(rem, take);
      const uint32_t nbins = (nb + (1u << rem) - 1) >> rem;
      unsigned long long* dst = ((passes - 1 - j) & 1) ? tmp2 : tmp;
      if (rem) {
        k_super_cursors<<<grid_for(nbins, 256, 4), 256, 0, s>>>(bbase, nb, nbins, bcur, rem);
        CYC_LAUNCHED();
      } else {
        CYC_CUDA(cudaMemcpyAsync(bcur, bbase, (size_t)nb * 4, cudaMemcpyDeviceToDevice, s));
      }
      if (j == 0) {
        k_part<true><<<pblocks, kPartThreads, nbins * 4, s>>>(src, m_in, n, key_dst, sh + rem, nbins, bcur, dst, 0);
        CYC_LAUNCHED();
        m_in = m_ok;
      } else {
        k_part<false><<<pblocks, kPartThreads, nbins * 4, s>>>(src, m_in, n, key_dst, sh + rem, nbins, bcur, dst,
                                                               rem_in - rem);
        CYC_LAUNCHED();
      }
      src = dst;
    }
    k_bucket_rows<<<std::min<uint32_t>(nb, sm_count() * 2), kPartThreads, (1u << sh) * 4, s>>>(
        tmp, bbase, n, sh, nb, roff, raw);
    CYC_LAUNCHED();
    return;
  }
  uint32_t* c = ar.get<uint32_t>(ar.bcnt, ((size_t)n + 1) * 4, s);
  CYC_CUDA(cudaMemsetAsync(c, 0, ((size_t)n + 1) * 4, s));
  if (m_log) {
    k_hist<<<grid_for(m_log, 256, 16), 256, 0, s>>>(e2, m_log, n, key_dst, c, d_err);
    CYC_LAUNCHED();
  }
  exclusive_scan(c, roff, n, nullptr, s, scratch);
  if (m_log) {
    k_scatter<<<grid_for(m_log, 256, 16), 256, 0, s>>>(e2, m_log, n, key_dst, roff, c, raw);
    CYC_LAUNCHED();
  }
}

// A borrowed arena buffer with DevBuf's accessor.
struct View {
  uint32_t* p;
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

// CYC_DEBUG_TIMING=1 prints host-observed phase times of the build (stderr).
struct PhaseTimer {
  bool on;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t;
  explicit PhaseTimer(cudaStream_t st) : on(std::getenv("CYC_DEBUG_TIMING") != nullptr), s(st) {
    t = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[cyc build] %-14s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Long rows (list `rows`, count cts[0]): the MSD split sort above.
static void sort_long_rows(const uint32_t* rows, const uint32_t* cts, const uint32_t* roff, uint32_t* raw,
                           uint32_t* ucnt, cudaStream_t s, BuildArena& ar) {
  uint32_t nr = 0;
  CYC_CUDA(cudaMemcpyAsync(&nr, cts, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  if (!nr) return;
  DevBuf& scratch = ar.scratch;
  // per-row arrays: nch, chbase, rmin, rmax, nsub, shift, subbase, (misc)
  uint32_t* rw = ar.get<uint32_t>(ar.sp_row, ((size_t)nr + 2) * 4 * 8, s);
  const size_t R = (size_t)nr + 2;
  uint32_t *nch = rw, *chbase = rw + R, *rmin = rw + 2 * R, *rmax = rw + 3 * R, *nsub = rw + 4 * R,
           *shift = rw + 5 * R, *subbase = rw + 6 * R, *misc = rw + 7 * R;
  const uint32_t g = grid_for(nr, 256, 8);
  k_split_setup<<<g, 256, 0, s>>>(rows, cts, roff, nch, rmin, rmax);
  CYC_LAUNCHED();
  exclusive_scan(nch, chbase, nr, nullptr, s, scratch);
  uint32_t hdr[2] = {0, 0};  // chunks, elements
  CYC_CUDA(cudaMemcpyAsync(&hdr[0], chbase + nr, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  const uint32_t C = hdr[0];
  uint2* desc = ar.get<uint2>(ar.sp_desc, ((size_t)C + 1) * 8, s);
  k_split_desc<<<g, 256, 0, s>>>(cts, chbase, desc);
  CYC_LAUNCHED();
  const uint32_t gc = std::min<uint32_t>(C, sm_count() * 2);
  k_split_minmax<<<gc, kSplitThreads, 0, s>>>(desc, C, rows, roff, raw, rmin, rmax);
  CYC_LAUNCHED();
  k_split_nsub<<<g, 256, 0, s>>>(rows, cts, roff, rmin, rmax, nsub, shift);
  CYC_LAUNCHED();
  exclusive_scan(nsub, subbase, nr, nullptr, s, scratch);
  uint32_t S = 0;
  CYC_CUDA(cudaMemcpyAsync(&S, subbase + nr, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  // per-sub arrays: cnt/cursor, soff, usub, uoff, over list
  uint32_t* sw = ar.get<uint32_t>(ar.sp_sub, ((size_t)S + 2) * 4 * 5, s);
  const size_t SS = (size_t)S + 2;
  uint32_t *cnt = sw, *soff = sw + SS, *usub = sw + 2 * SS, *uoff = sw + 3 * SS, *over = sw + 4 * SS;
  CYC_CUDA(cudaMemsetAsync(cnt, 0, SS * 4, s));
  CYC_CUDA(cudaMemsetAsync(misc, 0, 8, s));
  k_split_bins<false><<<gc, kSplitThreads, 0, s>>>(desc, C, rows, roff, raw, rmin, shift, nsub, subbase, cnt,
                                                   nullptr);
  CYC_LAUNCHED();
  exclusive_scan(cnt, soff, S, nullptr, s, scratch);
  uint32_t E = 0;
  CYC_CUDA(cudaMemcpyAsync(&E, soff + S, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaMemcpyAsync(cnt, soff, (size_t)S * 4, cudaMemcpyDeviceToDevice, s));  // cursors
  CYC_CUDA(cudaStreamSynchronize(s));
  uint32_t* tmp = ar.get<uint32_t>(ar.sp_tmp, ((size_t)E + 1) * 4, s);
  k_split_bins<true><<<gc, kSplitThreads, 0, s>>>(desc, C, rows, roff, raw, rmin, shift, nsub, subbase, cnt, tmp);
  CYC_LAUNCHED();
  k_split_sort<<<grid_for((uint64_t)S * 32, 256, 8), 256, 0, s>>>(S, soff, tmp, usub, over, misc);
  CYC_LAUNCHED();
  k_split_sort_over<<<sm_count(), kBigThreads, 0, s>>>(over, misc, soff, tmp, usub);
  CYC_LAUNCHED();
  exclusive_scan(usub, uoff, S, nullptr, s, scratch);
  k_split_write<<<grid_for((uint64_t)S * 32, 256, 8), 256, 0, s>>>(S, nr, rows, roff, subbase, soff, uoff, tmp,
                                                                   raw, ucnt);
  CYC_LAUNCHED();
}

void build_csr(const uint32_t* d_edges, uint64_t m_log, uint32_t n, int key_dst, cudaStream_t s,
               DevCsr& out, uint32_t* d_err, BuildArena& ar) {
  PhaseTimer pt(s);
  out.n = n;
  out.off.alloc(((size_t)n + 1) * 4, s);
  View roff{ar.get<uint32_t>(ar.roff, ((size_t)n + 1) * 4, s)};
  View raw{ar.get<uint32_t>(ar.raw, (m_log ? m_log : 1) * 4, s)};
  View ucnt{ar.get<uint32_t>(ar.ucnt, ((size_t)n + 1) * 4, s)};
  View lists{ar.get<uint32_t>(ar.lists, ((size_t)n + 1) * 4 * 3, s)};
  View counts{ar.get<uint32_t>(ar.counts, 16, s)};
  DevBuf& scratch = ar.scratch;
  CYC_CUDA(cudaMemsetAsync(counts.p, 0, 16, s));
  CYC_CUDA(cudaMemsetAsync(roff.p, 0, ((size_t)n + 1) * 4, s));
  const uint2* e2 = reinterpret_cast<const uint2*>(d_edges);
  pt.mark("alloc");
  count_sort_rows(e2, m_log, n, key_dst, s, roff.p, raw.p, d_err, ar);
  pt.mark("count_sort");
  uint32_t* med = lists.as<uint32_t>();
  uint32_t* big = med + n + 1;
  uint32_t* wrows = big + n + 1;
  uint32_t* cts = counts.as<uint32_t>();
  if (n) {
    k_sort_small<<<grid_for(n, 256, 16), 256, 0, s>>>(n, roff.as<uint32_t>(), raw.as<uint32_t>(),
                                                       ucnt.as<uint32_t>(), med, big, wrows, cts);
    CYC_LAUNCHED();
    k_sort_warp<<<sm_count() * 8, 256, 0, s>>>(wrows, cts, roff.as<uint32_t>(), raw.as<uint32_t>(),
                                               ucnt.as<uint32_t>());
    CYC_LAUNCHED();
    sort_long_rows(med, cts, roff.as<uint32_t>(), raw.as<uint32_t>(), ucnt.as<uint32_t>(), s, ar);
  }
  pt.mark("row_sort");
  exclusive_scan(ucnt.as<uint32_t>(), out.off.as<uint32_t>(), n, nullptr, s, scratch);
  uint32_t m = 0;
  CYC_CUDA(cudaMemcpyAsync(&m, out.off.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  out.m = m;
  out.col.alloc((m ? m : 1) * 4ull, s);
  if (n) {
    k_compact_rows<<<grid_for(n, 256, 16), 256, 0, s>>>(n, roff.as<uint32_t>(), out.off.as<uint32_t>(),
                                                        raw.as<uint32_t>(), out.col.as<uint32_t>());
    CYC_LAUNCHED();
    k_compact_list<<<sm_count() * 4, 256, 0, s>>>(med, cts, roff.as<uint32_t>(), out.off.as<uint32_t>(),
                                                  raw.as<uint32_t>(), out.col.as<uint32_t>());
    CYC_LAUNCHED();
  }
  pt.mark("compact");
}

void build_heavy(DevCsr& g, uint32_t heavy, uint32_t chunk, cudaStream_t s, uint32_t col_blocks) {
  const uint32_t ncb = col_blocks ? col_blocks : 1;
  uint64_t cap = g.m / chunk + (g.m / (heavy ? heavy : 1) + 1) * ncb + 2;
  g.heavy.alloc(cap * sizeof(uint4), s);
  DevBuf cnt(8, s);
  CYC_CUDA(cudaMemsetAsync(cnt.p, 0, 8, s));
  if (g.n && ncb == 1) {
    k_heavy_chunks<<<grid_for(g.n, 256, 16), 256, 0, s>>>(g.n, g.off.as<uint32_t>(), heavy, chunk,
                                                          g.heavy.as<uint4>(), cnt.as<uint32_t>());
    CYC_LAUNCHED();
  } else if (g.n) {
    const uint32_t width = (uint32_t)(((uint64_t)g.n + ncb - 1) / ncb);
    DevBuf bc((size_t)(2 * ncb + 2) * 4, s);
    CYC_CUDA(cudaMemsetAsync(bc.p, 0, (size_t)(2 * ncb + 2) * 4, s));
    uint32_t* bcount = bc.as<uint32_t>();
    uint32_t* bcur = bcount + ncb + 1;
    k_heavy_blocks<<<grid_for(g.n, 256, 16), 256, 0, s>>>(g.n, g.o(), g.c(), heavy, chunk, ncb, width, bcount,
                                                          nullptr, nullptr);
    CYC_LAUNCHED();
    std::vector<uint32_t> hc(ncb), hb(ncb + 1, 0);
    CYC_CUDA(cudaMemcpyAsync(hc.data(), bcount, ncb * 4, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
    for (uint32_t j = 0; j < ncb; ++j) hb[j + 1] = hb[j] + hc[j];
    CYC_CUDA(cudaMemcpyAsync(bcur, hb.data(), ncb * 4, cudaMemcpyHostToDevice, s));
    CYC_CUDA(cudaMemcpyAsync(cnt.p, &hb[ncb], 4, cudaMemcpyHostToDevice, s));
    k_heavy_blocks<<<grid_for(g.n, 256, 16), 256, 0, s>>>(g.n, g.o(), g.c(), heavy, chunk, ncb, width, nullptr,
                                                          bcur, g.heavy.as<uint4>());
    CYC_LAUNCHED();
  }
  if (g.n) {
    k_max_degree<<<grid_for(g.n, 256, 8), 256, 0, s>>>(g.n, g.off.as<uint32_t>(),
                                                       cnt.as<uint32_t>() + 1);
    CYC_LAUNCHED();
  }
  uint32_t h[2] = {0, 0};
  CYC_CUDA(cudaMemcpyAsync(h, cnt.p, 8, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  g.n_heavy_chunks = h[0];
  g.max_degree = h[1];
  g.heavy_deg = heavy;
}

uint32_t pull_col_blocks(uint32_t n) {
  // keep each column block's slice of the map vector (4 B per vertex) within
  // ~96 MB of the 126 MB L2 (measured on config 3: 3 blocks 69 ms per 8
  // steps, 6 blocks 77, 12 blocks 145, none 97 — more blocks cut rows into
  // more, shorter chunks)
  const uint64_t bytes = (uint64_t)n * 4;
  const uint64_t budget = 96ull << 20;
  return bytes <= 2 * budget ? 1u : (uint32_t)((bytes + budget - 1) / budget);
}

}  // namespace cyc
