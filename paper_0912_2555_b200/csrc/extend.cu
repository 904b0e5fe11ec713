// extend.cu — incremental snapshots. The explorer's detector
// rebuilds the snapshot of a growing log prefix every round (explore.cpp:
// 71-124, graph.cpp:63-105: counting sort + per-row sort + dedup of ALL
// logged edges). Rows of a CSR snapshot are sorted and duplicate-free, so the
// snapshot of prefix (m1, n1) is the row-wise sorted union of the snapshot of
// prefix (m0, n0) and the snapshot of the new edges [m0, m1): only the new
// edges are sorted, the old rows are merged in one streaming pass.
//
// merge_csr: per row, |out| = |a| + |b| - |a ∩ b|; rows with |a|+|b| <= 64
// merge on one thread (two-pointer), longer rows on a warp: an element x = a[i]
// lands at i + lower_bound(b, x) - (elements of a before i that are in b); an
// element y = b[j] not in a at lower_bound(a, y) + j - (elements of b before j
// that are in a).
#include "extend.cuh"

namespace cyc {

namespace {

constexpr int kT = 256;
constexpr uint32_t kThreadMerge = 64;

__device__ __forceinline__ uint32_t lower_bound(const uint32_t* p, uint32_t len, uint32_t x) {
  uint32_t lo = 0, hi = len;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (p[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

struct Rows {
  const uint32_t* aoff;
  const uint32_t* acol;
  uint32_t an;
  const uint32_t* boff;
  const uint32_t* bcol;
  __device__ void get(uint32_t v, const uint32_t*& a, uint32_t& da, const uint32_t*& b, uint32_t& db) const {
    if (v < an) {
      a = acol + aoff[v];
      da = aoff[v + 1] - aoff[v];
    } else {
      a = acol;
      da = 0;
    }
    b = bcol + boff[v];
    db = boff[v + 1] - boff[v];
  }
};

// thread two-pointer merge; out == nullptr counts only
__device__ __forceinline__ uint32_t merge_thread(const uint32_t* a, uint32_t da, const uint32_t* b, uint32_t db,
                                                 uint32_t* out) {
  uint32_t i = 0, j = 0, k = 0;
  while (i < da || j < db) {
    uint32_t x;
    if (j >= db || (i < da && a[i] < b[j])) {
      x = a[i++];
    } else if (i >= da || b[j] < a[i]) {
      x = b[j++];
    } else {
      x = a[i++];
      ++j;
    }
    if (out) out[k] = x;
    ++k;
  }
  return k;
}

// warp merge of one row (all lanes); returns the merged length
__device__ uint32_t merge_warp(const uint32_t* a, uint32_t da, const uint32_t* b, uint32_t db, uint32_t* out) {
  const uint32_t lane = lane_id();
  if (out) {
    uint32_t common = 0;  // elements of a before i that are also in b
    for (uint32_t i0 = 0; i0 < da; i0 += 32u) {
      const uint32_t i = i0 + lane;
      bool in_b = false;
      uint32_t lb = 0, x = 0;
      if (i < da) {
        x = a[i];
        lb = lower_bound(b, db, x);
        in_b = lb < db && b[lb] == x;
      }
      const uint32_t bal = __ballot_sync(kFull, in_b);
      if (i < da) out[i + lb - (common + __popc(bal & lanemask_lt()))] = x;
      common += __popc(bal);
    }
  }
  uint32_t dups = 0;
  for (uint32_t j0 = 0; j0 < db; j0 += 32u) {
    const uint32_t j = j0 + lane;
    bool in_a = false;
    uint32_t lb = 0, y = 0;
    if (j < db) {
      y = b[j];
      lb = lower_bound(a, da, y);
      in_a = lb < da && a[lb] == y;
    }
    const uint32_t bal = __ballot_sync(kFull, in_a);
    if (out && j < db && !in_a) out[lb + j - (dups + __popc(bal & lanemask_lt()))] = y;
    dups += __popc(bal);
  }
  return da + db - dups;
}

__global__ void k_merge_count(uint32_t n, Rows r, uint32_t* cnt) {
  const uint32_t lane = lane_id();
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; v0 < n; v0 += stride) {
    const uint32_t v = v0 + lane;
    const uint32_t *a = nullptr, *b = nullptr;
    uint32_t da = 0, db = 0;
    if (v < n) r.get(v, a, da, b, db);
    const bool big = da + db > kThreadMerge;
    if (v < n && !big) cnt[v] = merge_thread(a, da, b, db, nullptr);
    for (uint32_t hb = __ballot_sync(kFull, big); hb; hb &= hb - 1u) {
      const uint32_t l = __ffs(hb) - 1u;
      const uint32_t* ra;
      const uint32_t* rb;
      uint32_t xa, xb;
      r.get(v0 + l, ra, xa, rb, xb);
      const uint32_t k = merge_warp(ra, xa, rb, xb, nullptr);
      if (lane == 0) cnt[v0 + l] = k;
    }
  }
}

__global__ void k_merge_fill(uint32_t n, Rows r, const uint32_t* __restrict__ ooff, uint32_t* __restrict__ ocol) {
  const uint32_t lane = lane_id();
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; v0 < n; v0 += stride) {
    const uint32_t v = v0 + lane;
    const uint32_t *a = nullptr, *b = nullptr;
    uint32_t da = 0, db = 0;
    if (v < n) r.get(v, a, da, b, db);
    const bool big = da + db > kThreadMerge;
    if (v < n && !big) merge_thread(a, da, b, db, ocol + ooff[v]);
    for (uint32_t hb = __ballot_sync(kFull, big); hb; hb &= hb - 1u) {
      const uint32_t l = __ffs(hb) - 1u;
      const uint32_t* ra;
      const uint32_t* rb;
      uint32_t xa, xb;
      r.get(v0 + l, ra, xa, rb, xb);
      merge_warp(ra, xa, rb, xb, ocol + ooff[v0 + l]);
    }
  }
}

}  // namespace

void merge_csr(const DevCsr& a, const DevCsr& b, uint32_t n, cudaStream_t s, DevCsr& out) {
  out.n = n;
  out.off.alloc(((size_t)n + 1) * 4, s);
  DevBuf cnt(((size_t)n + 1) * 4, s), scratch;
  Rows r{a.o(), a.c(), a.n, b.o(), b.c()};
  if (n) {
    k_merge_count<<<grid_for(n, kT, 8), kT, 0, s>>>(n, r, cnt.as<uint32_t>());
    CYC_LAUNCHED();
  }
  exclusive_scan(cnt.as<uint32_t>(), out.off.as<uint32_t>(), n, nullptr, s, scratch);
  uint32_t m = 0;
  CYC_CUDA(cudaMemcpyAsync(&m, out.off.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  out.m = m;
  out.col.alloc((m ? m : 1) * 4ull, s);
  if (n) {
    k_merge_fill<<<grid_for(n, kT, 8), kT, 0, s>>>(n, r, out.off.as<uint32_t>(), out.col.as<uint32_t>());
    CYC_LAUNCHED();
  }
}

}  // namespace cyc
