// frontier.cuh — level-synchronous frontier propagation in ONE persistent
// cooperative kernel, for the closures of K2 (reachability, max-colour,
// same-colour backward reach) and OWCTY's reach.
//
// Dense passes cost O(n + m) each and need as many passes as the graph is
// deep along the id order: 16.5 K passes (1.2 s) on config 5's chain. Here a
// level only touches the rows of vertices that changed in the previous level
// and levels are separated by a grid barrier (~1.2 us), not a host round trip.
//
// Level L pops queue q[L&1] and pushes into q[(L+1)&1]. A warp takes 32
// queued vertices and walks the concatenation of their rows 32 edges per
// round (owner lane found by a shuffle binary search over the degree scan),
// so lanes stay converged and enqueueing is one atomicAdd per warp round.
// Rows longer than kBigDeg go, as kBigChunk-edge chunks, to a side list that
// all warps share after the level's barrier (R-MAT hubs would otherwise pin
// one warp for the whole level). Counters rotate over three slots so each is reset
// exactly one level before it is reused, with one barrier per level.
//
// An Op supplies
//   uint32_t token(u)            value carried by popped vertex u
//   bool relax(u, token, w, L)   apply edge u -> w at level L; true iff w is
//                                newly queued for level L+1
// and must queue each vertex at most once per level (it owns the dedup).
#pragma once

#include <cooperative_groups.h>

#include "build.cuh"

namespace cyc {

constexpr int kFrontierThreads = 512;
constexpr uint32_t kBigDeg = 256;
constexpr uint32_t kBigChunk = 1024;

struct FrontierBufs {
  uint32_t* q[2] = {nullptr, nullptr};    // capacity cap each
  uint2* big[2] = {nullptr, nullptr};     // {row, chunk} entries, capacity bigcap each
  uint32_t* cnt = nullptr;  // [0..2] queue lengths, [3..5] big counts, [6] levels, [7] solo exit level
  uint32_t cap = 0;
  uint32_t bigcap = 0;
};

__device__ __forceinline__ bool test_and_set_bit(uint32_t* bits, uint32_t v) {
  const uint32_t m = 1u << (v & 31u);
  if (__ldcg(bits + (v >> 5)) & m) return false;
  return !(atomicOr(bits + (v >> 5), m) & m);
}

__device__ __forceinline__ void frontier_push(bool push, uint32_t w, uint32_t* q, uint32_t* qcnt) {
  const uint32_t bal = __ballot_sync(kFull, push);
  if (!bal) return;
  uint32_t base = 0;
  if (lane_id() == 0) base = atomicAdd(qcnt, (uint32_t)__popc(bal));
  base = __shfl_sync(kFull, base, 0);
  if (push) q[base + __popc(bal & lanemask_lt())] = w;
}

// One warp walks the rows of its (up to) 32 vertices, 32 edges per round;
// rows with d > big_deg are handed to big(u, d) instead. push(ok, w) is
// called converged once per round.
template <class Op, class Push, class Big>
__device__ __forceinline__ void warp_rows(bool has, uint32_t u, const uint32_t* __restrict__ off,
                                          const uint32_t* __restrict__ col, const Op& op, uint32_t L,
                                          uint32_t big_deg, Push&& push, Big&& big) {
  const uint32_t lane = lane_id();
  const uint32_t tok = has ? op.token(u) : 0u;
  uint32_t b = 0, d = 0;
  if (has) {
    b = off[u];
    d = off[u + 1] - b;
    if (d > big_deg) {
      big(u, d);
      d = 0;
    }
  }
  const uint32_t incl = warp_incl_scan(d);
  const uint32_t excl = incl - d;
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
    const uint32_t ob = __shfl_sync(kFull, b, owner);
    const uint32_t oe = __shfl_sync(kFull, excl, owner);
    const uint32_t ot = __shfl_sync(kFull, tok, owner);
    const uint32_t ou = __shfl_sync(kFull, u, owner);
    bool ok = false;
    uint32_t w = 0;
    if (e < total) {
      w = col[ob + (e - oe)];
      ok = op.relax(ou, ot, w, L);
    }
    push(ok, w);
  }
}

// Solo mode: while levels stay small, CTA 0 runs them alone from shared-memory
// queues with __syncthreads() between levels (a level then costs its memory
// round trips, not a grid barrier); the other CTAs wait at the grid barrier.
// On exit it leaves the global queue and counters as level `L` of the normal
// mode expects them and publishes L in cnt[7]: queue q[L&1] with cnt[L%3]
// entries, every other counter zero.
constexpr uint32_t kSoloCap = 2048;     // shared queue entries per level
constexpr uint32_t kSoloMaxDeg = 4096;  // a longer row sends the level back to the grid
constexpr uint32_t kSoloEnter = 512;    // one 32-vertex group per warp of the CTA

template <class Op>
__device__ void solo_levels(const uint32_t* __restrict__ off, const uint32_t* __restrict__ col,
                            const FrontierBufs& fb, const Op& op, uint32_t L, uint32_t len) {
  __shared__ uint32_t sq[2][kSoloCap];
  __shared__ uint32_t scnt[2];
  __shared__ uint32_t sbig;
  const uint32_t lane = lane_id();
  const uint32_t wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  {
    const uint32_t* qc = (L & 1u) ? fb.q[1] : fb.q[0];
    for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) sq[0][i] = __ldcg(qc + i);
  }
  if (threadIdx.x == 0) {
    scnt[0] = len;
    scnt[1] = 0;
    sbig = 0;
  }
  __syncthreads();
  int cur = 0;
  for (;;) {
    const uint32_t n0 = scnt[cur];
    // a long row in this level: hand the level back to the grid
    for (uint32_t i = threadIdx.x; i < n0; i += blockDim.x) {
      const uint32_t u = sq[cur][i];
      if (off[u + 1] - off[u] > kSoloMaxDeg) sbig = 1;
    }
    __syncthreads();
    if (sbig) {
      uint32_t* qg = (L & 1u) ? fb.q[1] : fb.q[0];
      for (uint32_t i = threadIdx.x; i < n0; i += blockDim.x) qg[i] = sq[cur][i];
      if (threadIdx.x == 0) {
        for (int k = 0; k < 6; ++k) fb.cnt[k] = 0;
        fb.cnt[L % 3u] = n0;
        fb.cnt[7] = L;
      }
      return;
    }
    uint32_t* qn_glob = (L & 1u) ? fb.q[0] : fb.q[1];  // overflow target = level L+1's queue
    uint32_t* sn = sq[cur ^ 1];
    uint32_t* snc = &scnt[cur ^ 1];
    auto push = [&](bool ok, uint32_t w) {
      const uint32_t bal = __ballot_sync(kFull, ok);
      if (!bal) return;
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(snc, (uint32_t)__popc(bal));
      base = __shfl_sync(kFull, base, 0);
      if (ok) {
        const uint32_t idx = base + __popc(bal & lanemask_lt());
        if (idx < kSoloCap) sn[idx] = w; else qn_glob[idx] = w;
      }
    };
    auto nobig = [](uint32_t, uint32_t) {};
    for (uint32_t base = wid * 32u; base < n0; base += nwarps * 32u) {
      const uint32_t i = base + lane;
      const bool has = i < n0;
      warp_rows(has, has ? sq[cur][i] : 0u, off, col, op, L, 0xFFFFFFFFu, push, nobig);
    }
    __syncthreads();
    const uint32_t nn = *snc;
    ++L;
    if (nn == 0 || nn > kSoloCap) {  // done, or back to the grid with level L
      for (uint32_t i = threadIdx.x; i < nn && i < kSoloCap; i += blockDim.x) qn_glob[i] = sn[i];
      if (threadIdx.x == 0) {
        for (int k = 0; k < 6; ++k) fb.cnt[k] = 0;
        fb.cnt[L % 3u] = nn;
        fb.cnt[7] = L;
      }
      return;
    }
    if (threadIdx.x == 0) scnt[cur] = 0;
    cur ^= 1;
    __syncthreads();
  }
}

template <class Op>
__global__ void __launch_bounds__(kFrontierThreads) k_frontier(const uint32_t* __restrict__ off,
                                                                const uint32_t* __restrict__ col,
                                                                FrontierBufs fb, Op op) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const uint32_t lane = lane_id();
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t gw = gtid >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  bool solo_ok = true;  // no solo right after leaving it for a long row
  for (uint32_t L = 0;;) {
    const uint32_t len = __ldcg(fb.cnt + L % 3u);
    if (len == 0) {
      if (gtid == 0) fb.cnt[6] = L;
      return;
    }
    if (len <= kSoloEnter && solo_ok) {
      // every block has read this level's length before CTA 0 rewrites the
      // counters: without this barrier a block still on its way here could
      // read the count solo left behind (a later level's, same slot mod 3)
      // and take the grid branch alone — the intermittent hang of round 1
      // (~1 in 1800 restrictions; dropin_test, test_gpu_concurrency)
      grid.sync();
      if (blockIdx.x == 0) solo_levels(off, col, fb, op, L, len);
      grid.sync();
      const uint32_t L2 = __ldcg(fb.cnt + 7);
      solo_ok = L2 != L;  // solo handed back the level it started with: run it on the grid
      L = L2;
      continue;
    }
    solo_ok = true;
    const bool odd = L & 1u;
    const uint32_t* __restrict__ qc = odd ? fb.q[1] : fb.q[0];
    uint32_t* qn = odd ? fb.q[0] : fb.q[1];
    uint32_t* ncnt = fb.cnt + (L + 1u) % 3u;
    uint2* bl = odd ? fb.big[1] : fb.big[0];
    uint32_t* bcnt = fb.cnt + 3u + L % 3u;
    if (gtid == 0) {
      fb.cnt[(L + 2u) % 3u] = 0;       // read at level L-1, written at level L+1
      fb.cnt[3u + (L + 2u) % 3u] = 0;
    }
    // phase A: rows of the queued vertices, 32 vertices per warp
    auto push = [&](bool ok, uint32_t w) { frontier_push(ok, w, qn, ncnt); };
    auto big = [&](uint32_t u, uint32_t d) {
      const uint32_t nc = (d + kBigChunk - 1u) / kBigChunk;
      const uint32_t at = atomicAdd(bcnt, nc);
      for (uint32_t c = 0; c < nc; ++c) bl[at + c] = make_uint2(u, c);
    };
    for (uint32_t base = gw * 32u; base < len; base += nw * 32u) {
      const uint32_t i = base + lane;
      const bool has = i < len;
      warp_rows(has, has ? __ldcg(qc + i) : 0u, off, col, op, L, kBigDeg, push, big);
    }
    grid.sync();
    // phase B: chunks of long rows, one warp per chunk
    const uint32_t nb = __ldcg(bcnt);
    if (nb) {
      for (uint32_t k = gw; k < nb; k += nw) {
        const uint2 ch = __ldcg(bl + k);
        const uint32_t u = ch.x;
        const uint32_t tok = op.token(u);
        const uint32_t e = off[u + 1];
        const uint32_t b = off[u] + ch.y * kBigChunk;
        const uint32_t end = min(e, b + kBigChunk);
        for (uint32_t i0 = b; i0 < end; i0 += 32u) {
          const uint32_t i = i0 + lane;
          bool ok = false;
          uint32_t w = 0;
          if (i < end) {
            w = col[i];
            ok = op.relax(u, tok, w, L);
          }
          frontier_push(ok, w, qn, ncnt);
        }
      }
      grid.sync();
    }
    ++L;
  }
}

// Seeds q with {v < n : pred(v)} (any order) and adds their count to *cnt;
// bits (nullable) receives the predicate as a bitmap.
template <class Pred>
__global__ void k_seed(uint32_t n, Pred pred, uint32_t* q, uint32_t* cnt, uint32_t* bits) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; v0 < n; v0 += stride) {
    const uint32_t v = v0 + lane_id();
    const bool s = v < n && pred(v);
    if (bits) {
      const uint32_t w = __ballot_sync(kFull, s);
      if (lane_id() == 0) bits[v0 >> 5] = w;
    }
    frontier_push(s, v, q, cnt);
  }
}

// Scratch for run_frontier, grown on demand and reusable across calls.
struct FrontierWs {
  DevBuf q0, q1, b0, b1, cnt;
  // big chunks per level <= sum over rows with d > kBigDeg of ceil(d / kBigChunk) <= m / kBigDeg
  FrontierBufs bufs(uint32_t n, uint64_t m, cudaStream_t s) {
    const size_t bytes = ((size_t)n + 64) * 4;
    for (DevBuf* b : {&q0, &q1})
      if (b->bytes < bytes) b->alloc(bytes, s);
    const size_t bigcap = m / kBigDeg + 64;
    for (DevBuf* b : {&b0, &b1})
      if (b->bytes < bigcap * 8) b->alloc(bigcap * 8, s);
    if (!cnt.p) cnt.alloc(64, s);
    FrontierBufs f;
    f.q[0] = q0.as<uint32_t>();
    f.q[1] = q1.as<uint32_t>();
    f.big[0] = b0.as<uint2>();
    f.big[1] = b1.as<uint2>();
    f.cnt = cnt.as<uint32_t>();
    f.cap = n;
    f.bigcap = (uint32_t)(bigcap < 0xFFFFFFFFull ? bigcap : 0xFFFFFFFFull);
    return f;
  }
};

// Zeroes the counters and seeds level 0 with {v : pred(v)}.
template <class Pred>
void seed_frontier(uint32_t n, const Pred& pred, const FrontierBufs& fb, uint32_t* bits, cudaStream_t s) {
  CYC_CUDA(cudaMemsetAsync(fb.cnt, 0, 8 * sizeof(uint32_t), s));
  if (!n) return;
  k_seed<Pred><<<grid_for(n, 256, 8), 256, 0, s>>>(n, pred, fb.q[0], fb.cnt, bits);
  CYC_LAUNCHED();
}

// Runs levels until the queue empties (level 0 = the seeded queue). The level
// count lands in cnt[6].
template <class Op>
void run_frontier(const uint32_t* off, const uint32_t* col, const FrontierBufs& fb, const Op& op,
                  cudaStream_t s) {
  static int grid = [] {
    int b = 0;
    CYC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_frontier<Op>, kFrontierThreads, 0));
    return (b > 2 ? 2 : (b < 1 ? 1 : b)) * sm_count();
  }();
  FrontierBufs f = fb;
  Op o = op;
  const uint32_t* a0 = off;
  const uint32_t* a1 = col;
  void* args[] = {(void*)&a0, (void*)&a1, (void*)&f, (void*)&o};
  coop_launch((const void*)k_frontier<Op>, dim3(grid), dim3(kFrontierThreads), args, 0, s);
  CYC_LAUNCHED();
}

}  // namespace cyc
