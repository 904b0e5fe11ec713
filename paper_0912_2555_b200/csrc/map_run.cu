// map_run.cu — K3 (propagation step), K4 (witness + demotion), K5 (device
// loop) of the MAP engine as ONE persistent cooperative kernel.
//
// Replaces run_map / fixpoint / MaxPropagation::step / demote of the
// reference (map_engine.cpp:21-162). The host launches once per run_map and
// reads back {verdict, witness, MapStats}; every step, every convergence
// test and every demotion round happens on the device, separated by grid
// barriers. No per-step host synchronisation.
//
// Jacobi semantics are kept exactly (map_engine.cpp:56-66):
// after k steps x[v] = max{u in F : path u -> v of length 1..k}. Two step
// kinds compute the same Jacobi step:
//   pull  dense over all rows of the gather index, reading P[cur] and
//         writing P[cur^1] (double buffer); the north_star SpMV in the
//         (max, vertex-id) semiring. Each lane walks kRows rows in lock-step
//         so it keeps several independent gathers in flight.
//   push  only vertices raised in the previous step scatter their frozen
//         previous-step value with atomicMax into P[cur] in place. A vertex
//         that did not change cannot change anyone's max, so this equals
//         the dense step. The frozen value of a raised vertex is the maximum
//         raise it received in that step, kept per step parity in T[] as
//         (tag << 32 | value); tags grow monotonically, so T never needs
//         clearing and "first raise in this step" is a 64-bit atomicMax whose
//         previous tag is older. The frontier itself is a bitmap per step
//         parity (no list, no contended counter); vertices of push degree
//         > kBigDeg go to a short list of kChunk-edge chunks instead.
// The step kind is chosen on the device from the previous frontier's edge
// count (push when edges * alpha < m): direction-optimising traversal.
//
// Self-witness (map_engine.cpp:66): exact per row in pull; in push the
// raises to exactly v+1 of accepting v are candidates, confirmed after the
// barrier when T shows v+1 is that step's maximum raise.
#include <cstring>

#include "../../include/cyc_gen.h"
#include "map_run.cuh"

namespace cyc {

namespace {

constexpr int kRunThreads = 1024;
constexpr int kModePull = 1, kModePush = 2;
constexpr int kRows = 4;         // rows per lane in a pull step
constexpr int kBatch = 4;        // frontier vertices per lane in a push step
constexpr int kHeavyPerLane = 8;  // pull heavy chunk = 256 edges
constexpr uint32_t kTileWords = 8;  // bitmap words per warp tile (256 vertices)

__device__ __forceinline__ bool f_bit(const uint32_t* F, uint32_t v) {
  return (__ldcg(F + (v >> 5)) >> (v & 31u)) & 1u;
}

__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

__device__ __forceinline__ uint32_t cand_of(uint32_t w, uint32_t u) {
  return (w & kFlag) ? max(w & kCode, u + 1u) : w;
}

// ---------------------------------------------------------- block helpers
struct BlockSh {
  unsigned long long w[32];
  unsigned long long bcast[2];
  uint32_t wmin[33];
  uint32_t q[kRunThreads / 32][kTileWords * 32];  // per-warp push queues
};

// Sum over the CTA, result in every thread.
__device__ unsigned long long block_sum(unsigned long long x, BlockSh* sh) {
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  x = warp_sum64(x);
  if (lane == 0) sh->w[wid] = x;
  __syncthreads();
  if (wid == 0) {
    unsigned long long y = lane < nw ? sh->w[lane] : 0ull;
    y = warp_sum64(y);
    if (lane == 0) sh->bcast[0] = y;
  }
  __syncthreads();
  const unsigned long long r = sh->bcast[0];
  __syncthreads();
  return r;
}

__device__ uint32_t block_min(uint32_t x, BlockSh* sh) {
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  x = __reduce_min_sync(kFull, x);
  if (lane == 0) sh->wmin[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t y = lane < nw ? sh->wmin[lane] : kNone;
    y = __reduce_min_sync(kFull, y);
    if (lane == 0) sh->wmin[32] = y;
  }
  __syncthreads();
  const uint32_t r = sh->wmin[32];
  __syncthreads();
  return r;
}

// Per-thread step counters, reduced once per CTA per step.
struct StepAcc {
  unsigned long long raised = 0;  // successful raises (any > 0 => changed)
  unsigned long long first = 0;   // distinct vertices raised
  unsigned long long fedges = 0;  // push degrees of the next frontier
};

__device__ void step_flags(const StepAcc& acc, RunCtl* ctl, uint32_t slot, BlockSh* sh) {
  const unsigned long long r = block_sum(acc.raised, sh);
  const unsigned long long c = block_sum(acc.first, sh);
  const unsigned long long e = block_sum(acc.fedges, sh);
  if (threadIdx.x == 0) {
    if (r) *(volatile unsigned int*)&ctl->changed[slot] = 1u;
    if (c) atomicAdd(&ctl->nraised[slot], (unsigned)c);
    if (e) atomicAdd(&ctl->fedges[slot], e);
  }
}

// Frontier bookkeeping of a vertex v first raised in step `slot`: a bit in
// the step's bitmap, or kChunk-edge chunks for a big push degree.
__device__ __forceinline__ void enlist(const RunArgs& a, uint32_t v, uint32_t b, uint32_t e,
                                       uint32_t* fb, uint4* bc, unsigned int* nchunk) {
  const uint32_t deg = e - b;
  if (deg == 0) return;
  if (deg <= kBigDeg) {
    atomicOr(fb + (v >> 5), 1u << (v & 31u));
  } else {
    const uint32_t nc = (deg + kChunk - 1) / kChunk;
    const uint32_t base = atomicAdd(nchunk, nc);
    for (uint32_t c = 0; c < nc && base + c < a.chunk_cap; ++c)
      bc[base + c] = make_uint4(v, b + c * kChunk, min(e, b + (c + 1) * kChunk), 0u);
  }
}

// Batched atomicMax raise of P[tgt[r]] to val[r] (Jacobi push). Written as
// predicated stages (load, raise, tag, degree, enlist) so the R independent
// chains overlap instead of running one dependent chain after another. The
// first raise of a target in step g enlists it in the next frontier.
template <int R>
__device__ __forceinline__ void raise_batch(const RunArgs& a, uint32_t* P, unsigned long long* Tc,
                                            uint32_t g, const uint32_t (&tgt)[R],
                                            const uint32_t (&val)[R], uint32_t* fb, uint4* bc,
                                            unsigned int* nchunk, uint32_t* Cn, unsigned int* ccnt,
                                            StepAcc& acc) {
  uint32_t old[R], prev[R];
  bool go[R];
#pragma unroll
  for (int r = 0; r < R; ++r) old[r] = tgt[r] != kNone ? __ldcg(P + tgt[r]) : kCode;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    go[r] = tgt[r] != kNone && val[r] > (old[r] & kCode);
    prev[r] = go[r] ? atomicMax(P + tgt[r], (old[r] & kFlag) | val[r]) : kCode;
  }
  unsigned long long pt[R];
  const unsigned long long tag = (unsigned long long)g << 32;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    go[r] = go[r] && (prev[r] & kCode) < val[r];
    pt[r] = go[r] ? atomicMax(Tc + tgt[r], tag | val[r]) : tag;
  }
  uint32_t b[R], e[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    acc.raised += go[r];
    const bool first = go[r] && (uint32_t)(pt[r] >> 32) < g;
    b[r] = first ? __ldg(a.poff + tgt[r]) : 0u;
    e[r] = first ? __ldg(a.poff + tgt[r] + 1) : 0u;
    acc.first += first;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (e[r] > b[r]) {
      acc.fedges += e[r] - b[r];
      enlist(a, tgt[r], b[r], e[r], fb, bc, nchunk);
    }
    if (go[r] && (old[r] & kFlag) && val[r] == tgt[r] + 1u) Cn[atomicAdd(ccnt, 1u)] = tgt[r];
  }
}

// ------------------------------------------------------------------ pull
__device__ void pull_step(const RunArgs& a, uint32_t g, int cur, bool clear_prev, BlockSh* sh) {
  const uint32_t slot = g % 3u;
  const uint32_t* __restrict__ P = a.P[cur];
  uint32_t* __restrict__ Q = a.P[cur ^ 1];
  unsigned long long* Tc = a.T[g & 1u];
  uint32_t* Cn = a.C[g & 1u];
  RunCtl* ctl = a.ctl;
  const uint32_t lane = lane_id();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  StepAcc acc;
  if (clear_prev) {  // keep the bitmap invariant: FB[(g+1)&1] is zero when step g+1 starts
    uint32_t* fb = a.FB[(g - 1u) & 1u];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.nwords; i += gridDim.x * blockDim.x)
      fb[i] = 0u;
  }
  // heavy rows first (they are the long poles): one warp per chunk of at
  // most 32*kHeavyPerLane edges, every lane issuing all its loads at once;
  // combined with atomicMax into Q (Q holds an earlier, never larger, value
  // of the same fixpoint)
  for (uint32_t c = gw; c < a.n_heavy; c += nw) {
    const uint4 ch = a.heavy[c];
    const uint32_t v = ch.x;
    uint32_t u[kHeavyPerLane];
#pragma unroll
    for (int r = 0; r < kHeavyPerLane; ++r) {
      const uint32_t i = ch.y + lane + 32u * r;
      u[r] = i < ch.z ? __ldg(a.gcol + i) : kNone;
    }
    uint32_t best = 0;
#pragma unroll
    for (int r = 0; r < kHeavyPerLane; ++r)
      if (u[r] != kNone) best = max(best, cand_of(__ldcg(P + u[r]), u[r]));
    best = __reduce_max_sync(kFull, best);
    if (lane == 0) {
      const uint32_t own = __ldcg(P + v);
      best = max(best, own & kCode);
      atomicMax(Q + v, (own & kFlag) | best);
      if (best > (own & kCode)) {
        ++acc.raised;
        const unsigned long long pt = atomicMax(Tc + v, ((unsigned long long)g << 32) | best);
        acc.first += (uint32_t)(pt >> 32) < g;
        if ((own & kFlag) && best == v + 1u) Cn[atomicAdd(&ctl->cand_cnt[slot], 1u)] = v;
      }
    }
  }
  // light rows: each lane owns kRows rows (32*kRows consecutive rows per warp)
  // and walks their edge lists in lock-step, so every lane keeps up to
  // 2*kRows independent col/gather loads in flight (latency hiding by ILP).
  for (uint32_t base = gw * (32u * kRows); base < a.n; base += nw * (32u * kRows)) {
    uint32_t b[kRows], e[kRows], own[kRows], best[kRows];
    uint32_t skip = 0;  // bit k: row k is past n or heavy (chunk pass below)
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
      const uint32_t v = base + 32u * k + lane;
      b[k] = e[k] = 0;
      if (v < a.n) {
        b[k] = __ldg(a.goff + v);
        e[k] = __ldg(a.goff + v + 1);
        if (e[k] - b[k] > a.heavy_deg) {
          e[k] = b[k];
          skip |= 1u << k;
        }
      } else {
        skip |= 1u << k;
      }
    }
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
      const uint32_t v = base + 32u * k + lane;
      own[k] = v < a.n ? __ldcg(P + v) : 0u;
      best[k] = own[k] & kCode;
    }
    for (uint32_t j = 0;; j += 2) {
      uint32_t u0[kRows], u1[kRows];
      bool any = false;
#pragma unroll
      for (int k = 0; k < kRows; ++k) {
        u0[k] = b[k] + j < e[k] ? __ldg(a.gcol + b[k] + j) : kNone;
        u1[k] = b[k] + j + 1 < e[k] ? __ldg(a.gcol + b[k] + j + 1) : kNone;
        any |= b[k] + j < e[k];
      }
      if (!any) break;
#pragma unroll
      for (int k = 0; k < kRows; ++k) {
        if (u0[k] != kNone) best[k] = max(best[k], cand_of(__ldcg(P + u0[k]), u0[k]));
        if (u1[k] != kNone) best[k] = max(best[k], cand_of(__ldcg(P + u1[k]), u1[k]));
      }
    }
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
      const uint32_t v = base + 32u * k + lane;
      if (!((skip >> k) & 1u)) {
        Q[v] = (own[k] & kFlag) | best[k];
        const bool up = best[k] > (own[k] & kCode);
        acc.raised += up;
        acc.first += up;
        if ((own[k] & kFlag) && best[k] == v + 1u) atomicMin(&ctl->wit[slot], v);
      }
    }
  }
  step_flags(acc, ctl, slot, sh);
}

// After a pull step (tag gp), rebuild that step's frontier from the two
// buffers so a push step can follow: T values, bitmap words, big chunks.
__device__ void transition_pass(const RunArgs& a, uint32_t gp, int cur, BlockSh* sh) {
  const uint32_t* P = a.P[cur];
  const uint32_t* Q = a.P[cur ^ 1];
  unsigned long long* Tp = a.T[gp & 1u];
  uint32_t* fb = a.FB[gp & 1u];
  uint4* bc = a.BC[gp & 1u];
  unsigned int* nchunk = &a.ctl->nchunk[gp % 3u];
  const uint32_t lane = lane_id();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  StepAcc acc;
  for (uint32_t wi = gw; wi < a.nwords; wi += nw) {
    const uint32_t v = wi * 32u + lane;
    bool small = false;
    if (v < a.n) {
      const uint32_t xb = __ldcg(P + v) & kCode, xa = __ldcg(Q + v) & kCode;
      if (xb != xa) {
        Tp[v] = ((unsigned long long)gp << 32) | xb;
        const uint32_t b = __ldg(a.poff + v), e = __ldg(a.poff + v + 1);
        acc.fedges += e - b;
        small = e > b && e - b <= kBigDeg;
        if (e - b > kBigDeg) enlist(a, v, b, e, fb, bc, nchunk);
      }
    }
    const uint32_t word = __ballot_sync(kFull, small);
    if (lane == 0) fb[wi] = word;
  }
  const unsigned long long fe = block_sum(acc.fedges, sh);
  if (threadIdx.x == 0 && fe) atomicAdd(&a.ctl->fedges[gp % 3u], fe);
}

// ------------------------------------------------------------------ push
__device__ void push_step(const RunArgs& a, uint32_t g, int cur, BlockSh* sh) {
  const uint32_t slot = g % 3u, pslot = (g - 1u) % 3u;
  RunCtl* ctl = a.ctl;
  uint32_t* fp = a.FB[(g - 1u) & 1u];
  const uint4* bp = a.BC[(g - 1u) & 1u];
  const unsigned long long* Tp = a.T[(g - 1u) & 1u];
  unsigned long long* Tc = a.T[g & 1u];
  uint32_t* fb = a.FB[g & 1u];
  uint4* bc = a.BC[g & 1u];
  unsigned int* nchunk = &ctl->nchunk[slot];
  unsigned int* ccnt = &ctl->cand_cnt[slot];
  uint32_t* Cn = a.C[g & 1u];
  uint32_t* P = a.P[cur];
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  uint32_t* q = sh->q[wid];
  StepAcc acc;
  // big frontier vertices first: one warp per kChunk-edge chunk, each lane
  // raising kChunk/32 targets as one batch
  const uint32_t nch = min(__ldcg(&ctl->nchunk[pslot]), a.chunk_cap);
  for (uint32_t c = gw; c < nch; c += nw) {
    const uint4 ch = bp[c];
    const uint32_t v = ch.x;
    uint32_t vv = (uint32_t)__ldcg(Tp + v);
    if (f_bit(a.F, v)) vv = max(vv, v + 1u);
    uint32_t t[kChunk / 32], val[kChunk / 32];
#pragma unroll
    for (int r = 0; r < (int)(kChunk / 32); ++r) {
      const uint32_t i = ch.y + lane + 32u * r;
      t[r] = i < ch.z ? __ldg(a.pcol + i) : kNone;
      val[r] = vv;
    }
    raise_batch(a, P, Tc, g, t, val, fb, bc, nchunk, Cn, ccnt, acc);
  }
  // small frontier vertices, from the bitmap (each word read once and cleared)
  for (uint32_t wb = gw * kTileWords; wb < a.nwords; wb += nw * kTileWords) {
    uint32_t word = 0;
    const uint32_t wi = wb + lane;
    if (lane < kTileWords && wi < a.nwords) {
      word = __ldcg(fp + wi);
      if (word) fp[wi] = 0u;
    }
    const uint32_t c = __popc(word);
    const uint32_t incl = warp_incl_scan(c);
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    if (total == 0) continue;
    uint32_t pos = incl - c;
    while (word) {
      q[pos++] = wi * 32u + (uint32_t)(__ffs(word) - 1);
      word &= word - 1u;
    }
    __syncwarp();
    for (uint32_t k0 = 0; k0 < total; k0 += 32u * kBatch) {
      uint32_t v[kBatch], b[kBatch], e[kBatch], val[kBatch];
#pragma unroll
      for (int r = 0; r < kBatch; ++r) {
        const uint32_t k = k0 + 32u * r + lane;
        v[r] = k < total ? q[k] : kNone;
        b[r] = v[r] != kNone ? __ldg(a.poff + v[r]) : 0u;
        e[r] = v[r] != kNone ? __ldg(a.poff + v[r] + 1) : 0u;
      }
#pragma unroll
      for (int r = 0; r < kBatch; ++r) {
        val[r] = v[r] != kNone ? (uint32_t)__ldcg(Tp + v[r]) : 0u;
        if (v[r] != kNone && f_bit(a.F, v[r])) val[r] = max(val[r], v[r] + 1u);
      }
      for (uint32_t j = 0;; ++j) {
        uint32_t t[kBatch];
        bool any = false;
#pragma unroll
        for (int r = 0; r < kBatch; ++r) {
          t[r] = b[r] + j < e[r] ? __ldg(a.pcol + b[r] + j) : kNone;
          any |= t[r] != kNone;
        }
        if (!any) break;
        raise_batch(a, P, Tc, g, t, val, fb, bc, nchunk, Cn, ccnt, acc);
      }
    }
    __syncwarp();
  }
  step_flags(acc, ctl, slot, sh);
}

// ------------------------------------------------------- iteration passes
// Dense pass over the fixpoint vector: iteration hash, full self-witness (for
// early_exit = false, map_engine.cpp:108-112) and the "used" bitmap of demote
// (map_engine.cpp:124-126).
__device__ void finish_pass(const RunArgs& a, int cur, uint64_t t, bool mark_used, BlockSh* sh) {
  const uint32_t* P = a.P[cur];
  RunCtl* ctl = a.ctl;
  const uint32_t lane = lane_id();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  unsigned long long h = 0;
  uint32_t fw = kNone;
  for (uint32_t base = gw * 32u; base < a.n; base += nw * 32u) {
    const uint32_t v = base + lane;
    uint32_t code = 0;
    if (v < a.n) {
      const uint32_t x = __ldcg(P + v);
      code = x & kCode;
      h += cyc_splitmix64(((unsigned long long)v << 32) | code);
      if ((x & kFlag) && code == v + 1u) fw = min(fw, v);
    }
    if (mark_used) {
      const uint32_t peers = __match_any_sync(kFull, code);
      if (code && (__ffs(peers) - 1) == (int)lane) {
        const uint32_t u = code - 1u, bit = 1u << (u & 31u);
        if (!(__ldcg(a.used + (u >> 5)) & bit)) atomicOr(a.used + (u >> 5), bit);
      }
    }
  }
  h = block_sum(h, sh);
  fw = block_min(fw, sh);
  if (threadIdx.x == 0) {
    if (h) atomicAdd(&ctl->it_hash[t & 1u], h);
    if (fw != kNone) atomicMin(&ctl->it_finwit[t & 1u], fw);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const uint32_t nt = (uint32_t)((t + 1u) & 1u);
    ctl->it_hash[nt] = 0;
    ctl->it_finwit[nt] = kNone;
    ctl->it_dcount[nt] = 0;
    ctl->it_fsize[nt] = 0;
  }
}

// demote (map_engine.cpp:123-137): D = F & used, F' = F \ D in place, counts
// |D| and |F'|. The map buffers are left untouched (the last fixpoint vector
// is the result when the run ends here).
__device__ void demote_pass(const RunArgs& a, unsigned int* dcount, unsigned long long* fsize,
                            BlockSh* sh) {
  unsigned long long dc = 0, fs = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.nwords; i += stride) {
    const uint32_t f = __ldcg(a.F + i), u = __ldcg(a.used + i);
    const uint32_t nf = f & ~u;
    dc += __popc(f & u);
    fs += __popc(nf);
    if (u) {
      a.F[i] = nf;
      a.used[i] = 0;
    }
  }
  dc = block_sum(dc, sh);
  fs = block_sum(fs, sh);
  if (threadIdx.x == 0) {
    if (dcount && dc) atomicAdd(dcount, (unsigned)dc);
    if (fs) atomicAdd(fsize, fs);
  }
}

// Start of a fixpoint (setup tag g): both map buffers all-NIL with the
// accepting bit; the initial frontier = every accepting vertex, value id+1
// (bitmap FB[g&1] written in full, FB[(g+1)&1] cleared).
__device__ void reset_pass(const RunArgs& a, uint32_t g, BlockSh* sh) {
  unsigned long long* Tg = a.T[g & 1u];
  uint32_t* fb = a.FB[g & 1u];
  uint32_t* fz = a.FB[(g + 1u) & 1u];
  uint4* bc = a.BC[g & 1u];
  unsigned int* nchunk = &a.ctl->nchunk[g % 3u];
  const uint32_t lane = lane_id();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  StepAcc acc;
  for (uint32_t wi = gw; wi < a.nwords; wi += nw) {
    const uint32_t v = wi * 32u + lane;
    bool small = false;
    if (v < a.n) {
      const bool accv = f_bit(a.F, v);
      const uint32_t val = accv ? kFlag : 0u;
      a.P[0][v] = val;
      a.P[1][v] = val;
      if (accv) {
        const uint32_t b = __ldg(a.poff + v), e = __ldg(a.poff + v + 1);
        if (e > b) Tg[v] = ((unsigned long long)g << 32) | (v + 1u);
        acc.fedges += e - b;
        small = e > b && e - b <= kBigDeg;
        if (e - b > kBigDeg) enlist(a, v, b, e, fb, bc, nchunk);
      }
    }
    const uint32_t word = __ballot_sync(kFull, small);
    if (lane == 0) {
      fb[wi] = word;
      fz[wi] = 0u;
    }
  }
  const unsigned long long fe = block_sum(acc.fedges, sh);
  if (threadIdx.x == 0 && fe) atomicAdd(&a.ctl->fedges[g % 3u], fe);
}

__device__ __forceinline__ void reset_slot(RunCtl* c, uint32_t s) {
  c->fedges[s] = 0;
  c->nchunk[s] = 0;
  c->cand_cnt[s] = 0;
  c->wit[s] = kNone;
  c->changed[s] = 0;
  c->nraised[s] = 0;
}

__global__ void __launch_bounds__(kRunThreads, 1) k_map_run(RunArgs a) {
  __shared__ BlockSh sh;
  // run statistics live in shared memory of block 0 (kept out of registers)
  __shared__ unsigned long long stat[kResTag + 1];
  RunCtl* ctl = a.ctl;
  unsigned long long epoch = 0;
  uint32_t g = a.tag0;
  int cur = 0;
  int cycle = 0;
  uint32_t witness = kNone;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  if (lead)
    for (int k = 0; k <= kResTag; ++k) stat[k] = 0;
#define CYC_STAT(k, v) \
  do {                 \
    if (lead) stat[k] += (v); \
  } while (0)

  // initial F count and first fixpoint setup (tag g)
  demote_pass(a, nullptr, &ctl->it_fsize[0], &sh);
  if (lead) reset_slot(ctl, (g + 1u) % 3u);
  reset_pass(a, g, &sh);
  grid_sync(&ctl->bar, epoch);
  uint64_t t = 0;
  bool truncated = false;
  if (__ldcg(&ctl->it_fsize[0]) != 0) {
    for (;;) {
      unsigned long long steps = 0;
      bool prev_push = true;  // a frontier (bitmap + chunks) of the previous tag exists
      for (;;) {
        ++g;
        ++steps;
        const uint32_t slot = g % 3u, pslot = (g - 1u) % 3u;
        if (lead) reset_slot(ctl, (g + 1u) % 3u);
        int mode = a.mode;
        if (mode != kModePull && mode != kModePush) {
          unsigned long long est;
          if (prev_push) {
            est = __ldcg(&ctl->fedges[pslot]);
          } else {
            const unsigned long long nr = __ldcg(&ctl->nraised[pslot]);
            est = a.n ? nr * a.m / a.n : 0;
          }
          mode = (est * a.alpha < a.m) ? kModePush : kModePull;
        }
        if (mode == kModePush) {
          if (!prev_push) {
            transition_pass(a, g - 1u, cur, &sh);
            grid_sync(&ctl->bar, epoch);
          }
          if (lead) {
            const unsigned long long fe = __ldcg(&ctl->fedges[pslot]);
            stat[kResEdges] += fe;
            stat[kResRows] += __ldcg(&ctl->nraised[pslot]);
            stat[kResBytes] += 8ull * fe + 12ull * __ldcg(&ctl->nraised[pslot]);
            stat[kResPushSteps] += 1;
          }
          push_step(a, g, cur, &sh);
        } else {
          CYC_STAT(kResEdges, a.m);
          CYC_STAT(kResRows, a.n);
          CYC_STAT(kResBytes, 8ull * a.m + 12ull * a.n + 4ull);
          CYC_STAT(kResPullSteps, 1);
          pull_step(a, g, cur, prev_push, &sh);
        }
        grid_sync(&ctl->bar, epoch);
        if (lead && a.trace) {
          const unsigned long long k = stat[kResPullSteps] + stat[kResPushSteps] - 1u;
          if (k < a.trace_cap) {
            unsigned long long* tr = a.trace + 4u * k;
            tr[0] = ((unsigned long long)mode << 32) | (uint32_t)steps;
            tr[1] = mode == kModePush ? __ldcg(&ctl->fedges[pslot]) : a.m;
            tr[2] = __ldcg(&ctl->nraised[slot]);
            tr[3] = clock64();
          }
        }
        if (mode == kModePull) cur ^= 1;
        prev_push = mode == kModePush;
        const uint32_t changed = __ldcg(&ctl->changed[slot]);
        uint32_t w = __ldcg(&ctl->wit[slot]);
        const uint32_t nc = __ldcg(&ctl->cand_cnt[slot]);
        if (nc && a.early_exit) {
          const uint32_t* Cn = a.C[g & 1u];
          const unsigned long long* Tc = a.T[g & 1u];
          uint32_t mine = kNone;
          for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) {
            const uint32_t c = __ldcg(Cn + i);
            if (__ldcg(Tc + c) == (((unsigned long long)g << 32) | (c + 1u))) mine = min(mine, c);
          }
          w = min(w, block_min(mine, &sh));
        }
        if (a.early_exit && w != kNone) {
          cycle = 1;
          witness = w;
          break;
        }
        if (!changed) break;
        if (a.max_steps && steps >= a.max_steps) {
          truncated = true;
          break;
        }
      }
      if (lead) stat[kResStepsLast] = steps;
      if (truncated) {
        CYC_STAT(kResIterations, 1);
        CYC_STAT(kResKernelCalls, steps);
        break;
      }
      finish_pass(a, cur, t, !cycle, &sh);
      grid_sync(&ctl->bar, epoch);
      if (!a.early_exit) {
        const uint32_t fw = __ldcg(&ctl->it_finwit[t & 1u]);
        if (fw != kNone) {
          cycle = 1;
          witness = fw;
        }
      }
      if (lead && t < a.cap) {
        if (a.iter_hash) a.iter_hash[t] = __ldcg(&ctl->it_hash[t & 1u]);
        if (a.iter_steps) a.iter_steps[t] = steps;
      }
      CYC_STAT(kResIterations, 1);
      CYC_STAT(kResKernelCalls, steps);
      if (cycle) break;
      if (a.max_iterations && t + 1 >= a.max_iterations) break;
      demote_pass(a, &ctl->it_dcount[t & 1u], &ctl->it_fsize[(t + 1u) & 1u], &sh);
      grid_sync(&ctl->bar, epoch);
      const uint32_t dc = __ldcg(&ctl->it_dcount[t & 1u]);
      CYC_STAT(kResDemoted, dc);
      if (dc == 0) break;                                      // D empty: no cycle
      ++t;
      if (__ldcg(&ctl->it_fsize[t & 1u]) == 0) break;          // F' empty: no cycle
      ++g;
      if (lead) reset_slot(ctl, (g + 1u) % 3u);
      reset_pass(a, g, &sh);
      grid_sync(&ctl->bar, epoch);
    }
  }
  if (lead) {
    stat[kResCycle] = cycle;
    stat[kResWitness] = witness;
    stat[kResCur] = (unsigned long long)cur;
    stat[kResTag] = g;
    for (int k = 0; k <= kResTag; ++k) ctl->res[k] = stat[k];
  }
#undef CYC_STAT
}

__global__ void k_strip(const uint32_t* __restrict__ P, uint32_t n, uint32_t* __restrict__ out) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) out[v] = P[v] & kCode;
}

// ----------------------------------------------------- standalone kernels
__global__ void k_step_pull(uint32_t n, const uint32_t* __restrict__ goff,
                            const uint32_t* __restrict__ gcol, const uint32_t* __restrict__ x,
                            const uint32_t* __restrict__ accw, uint32_t* __restrict__ out,
                            uint32_t* __restrict__ flags) {
  const uint32_t stride = gridDim.x * blockDim.x;
  bool ch = false;
  uint32_t wit = kNone;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    uint32_t best = x[v];
    for (uint32_t i = goff[v]; i < goff[v + 1]; ++i) {
      uint32_t u = gcol[i];
      uint32_t c = x[u];
      if (((accw[u >> 5] >> (u & 31u)) & 1u) && u + 1u > c) c = u + 1u;
      best = max(best, c);
    }
    out[v] = best;
    ch |= best != x[v];
    if (best == v + 1u && ((accw[v >> 5] >> (v & 31u)) & 1u)) wit = min(wit, v);
  }
  if (__any_sync(__activemask(), ch) && lane_id() == 0) flags[0] = 1u;
  if (wit != kNone) atomicMin(flags + 1, wit);
}

__global__ void k_mark_used(const uint32_t* __restrict__ x, uint32_t n, uint32_t* used) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    uint32_t c = x[v];
    if (c && c - 1u < n) atomicOr(used + ((c - 1u) >> 5), 1u << ((c - 1u) & 31u));
  }
}

__global__ void k_demote_words(uint32_t nwords, const uint32_t* __restrict__ acc,
                               const uint32_t* __restrict__ used, uint32_t* __restrict__ rem,
                               uint32_t* __restrict__ cnt) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += stride) {
    uint32_t f = acc[i], u = used[i];
    rem[i] = f & ~u;
    cnt[i] = __popc(f & u);
  }
}

__global__ void k_demote_list(uint32_t nwords, const uint32_t* __restrict__ acc,
                              const uint32_t* __restrict__ used, const uint32_t* __restrict__ pos,
                              uint32_t* __restrict__ out) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += stride) {
    uint32_t d = acc[i] & used[i];
    uint32_t p = pos[i];
    while (d) {
      int b = __ffs(d) - 1;
      out[p++] = i * 32u + (uint32_t)b;
      d &= d - 1u;
    }
  }
}

}  // namespace

void RunWs::ensure(uint32_t nn, uint32_t mm, cudaStream_t s) {
  if (ctl.p && n == nn && m == mm) return;
  n = nn;
  m = mm;
  const size_t n1 = (size_t)nn + 1;
  const size_t words = ((size_t)nn + 63) / 64 * 2 + 2;
  // a vertex of push degree d > kBigDeg >= ... yields ceil(d/kChunk) <= d/kChunk + 1 chunks
  chunk_cap = (uint32_t)((uint64_t)mm / kChunk + (uint64_t)mm / (kBigDeg + 1) + 16);
  for (int k = 0; k < 2; ++k) {
    P[k].alloc(n1 * 4, s);
    T[k].alloc(n1 * 8, s);
    FB[k].alloc(words * 4, s);
    BC[k].alloc((size_t)chunk_cap * sizeof(uint4), s);
    C[k].alloc(n1 * 4, s);
    CYC_CUDA(cudaMemsetAsync(T[k].p, 0, n1 * 8, s));
  }
  F.alloc(words * 4, s);
  used.alloc(words * 4, s);
  CYC_CUDA(cudaMemsetAsync(used.p, 0, words * 4, s));
  ctl.alloc(sizeof(RunCtl), s);
  tag = 1;
}

void launch_map_run(const DevCsr& snap, const DevCsr& gath, RunWs& ws, int early_exit, int mode,
                    unsigned long long max_iterations, unsigned long long max_steps,
                    uint32_t alpha, unsigned long long cap, uint32_t trace_cap, cudaStream_t s,
                    cudaEvent_t e0, cudaEvent_t e1, RunOut& out) {
  const uint32_t n = gath.n;
  // Tags are u32: restart them (and clear T) long before they could wrap.
  if (ws.tag > 0xF0000000u) {
    for (int k = 0; k < 2; ++k) CYC_CUDA(cudaMemsetAsync(ws.T[k].p, 0, ((size_t)n + 1) * 8, s));
    ws.tag = 1;
  }
  RunCtl init;
  std::memset(&init, 0, sizeof init);
  for (int k = 0; k < 3; ++k) init.wit[k] = kNone;
  for (int k = 0; k < 2; ++k) init.it_finwit[k] = kNone;
  CYC_CUDA(cudaMemcpyAsync(ws.ctl.p, &init, sizeof init, cudaMemcpyHostToDevice, s));
  CYC_CUDA(cudaMemsetAsync(ws.used.p, 0, ws.used.bytes, s));
  if (cap) {
    if (ws.hist.bytes < cap * 16) ws.hist.alloc(cap * 16, s);
  }
  RunArgs a;
  std::memset(&a, 0, sizeof a);
  a.n = n;
  a.m = gath.m;
  a.goff = gath.o();
  a.gcol = gath.c();
  a.poff = snap.o();
  a.pcol = snap.c();
  a.heavy = gath.heavy.as<uint4>();
  a.n_heavy = gath.n_heavy_chunks;
  a.heavy_deg = gath.heavy_deg ? gath.heavy_deg : 0xFFFFFFFFu;
  for (int k = 0; k < 2; ++k) {
    a.P[k] = ws.P[k].as<uint32_t>();
    a.T[k] = ws.T[k].as<unsigned long long>();
    a.FB[k] = ws.FB[k].as<uint32_t>();
    a.BC[k] = ws.BC[k].as<uint4>();
    a.C[k] = ws.C[k].as<uint32_t>();
  }
  a.F = ws.F.as<uint32_t>();
  a.used = ws.used.as<uint32_t>();
  a.nwords = (uint32_t)(((uint64_t)n + 31) / 32);
  a.chunk_cap = ws.chunk_cap;
  a.ctl = ws.ctl.as<RunCtl>();
  a.iter_hash = cap ? ws.hist.as<unsigned long long>() : nullptr;
  a.iter_steps = cap ? ws.hist.as<unsigned long long>() + cap : nullptr;
  a.cap = cap;
  a.max_iterations = max_iterations;
  a.max_steps = max_steps;
  a.tag0 = ws.tag;
  if (trace_cap) {
    if (ws.trace.bytes < (size_t)trace_cap * 32) ws.trace.alloc((size_t)trace_cap * 32, s);
    a.trace = ws.trace.as<unsigned long long>();
    a.trace_cap = trace_cap;
  }
  ws.trace_cap = trace_cap;
  a.alpha = alpha ? alpha : 16u;
  a.early_exit = early_exit;
  a.mode = mode;

  static int blocks_per_sm = -1;
  if (blocks_per_sm < 0) {
    int b = 0;
    CYC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_map_run, kRunThreads, 0));
    blocks_per_sm = b > 0 ? b : 1;
  }
  dim3 grid((unsigned)(sm_count() * blocks_per_sm)), block(kRunThreads);
  void* args[] = {&a};
  CYC_CUDA(cudaEventRecord(e0, s));
  CYC_CUDA(cudaLaunchCooperativeKernel((const void*)k_map_run, grid, block, args, 0, s));
  CYC_LAUNCHED();
  CYC_CUDA(cudaEventRecord(e1, s));
  RunCtl host;
  CYC_CUDA(cudaMemcpyAsync(&host, ws.ctl.p, sizeof host, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  std::memcpy(out.res, host.res, sizeof out.res);
  CYC_CUDA(cudaEventElapsedTime(&out.ms, e0, e1));
  out.grid = grid.x;
  out.block = block.x;
  ws.tag = (uint32_t)host.res[kResTag] + 1u;
  {
    const unsigned long long k = host.res[kResPullSteps] + host.res[kResPushSteps];
    ws.trace_len = (uint32_t)(k < trace_cap ? k : trace_cap);
  }
}

void strip_codes(const RunWs& ws, int cur, uint32_t n, uint32_t* dst, cudaStream_t s) {
  if (!n) return;
  k_strip<<<grid_for(n, 256, 8), 256, 0, s>>>(ws.P[cur].as<uint32_t>(), n, dst);
  CYC_LAUNCHED();
}

void launch_step_pull(const DevCsr& gath, const uint32_t* x, const uint32_t* accw, uint32_t* out,
                      uint32_t* flags, cudaStream_t s) {
  uint32_t init[2] = {0u, kNone};
  CYC_CUDA(cudaMemcpyAsync(flags, init, 8, cudaMemcpyHostToDevice, s));
  if (!gath.n) return;
  k_step_pull<<<grid_for(gath.n, 256, 8), 256, 0, s>>>(gath.n, gath.o(), gath.c(), x, accw, out,
                                                        flags);
  CYC_LAUNCHED();
}

uint64_t run_demote(const uint32_t* x, uint32_t n, const uint32_t* accw, uint32_t* remaining,
                    uint32_t* demoted, cudaStream_t s) {
  const uint32_t nwords = (uint32_t)(((uint64_t)n + 31) / 32);
  DevBuf used(((size_t)nwords + 1) * 4, s), cnt(((size_t)nwords + 1) * 4, s),
      pos(((size_t)nwords + 2) * 4, s), scratch;
  CYC_CUDA(cudaMemsetAsync(used.p, 0, used.bytes, s));
  if (n) {
    k_mark_used<<<grid_for(n, 256, 8), 256, 0, s>>>(x, n, used.as<uint32_t>());
    CYC_LAUNCHED();
    k_demote_words<<<grid_for(nwords, 256, 8), 256, 0, s>>>(nwords, accw, used.as<uint32_t>(),
                                                             remaining, cnt.as<uint32_t>());
    CYC_LAUNCHED();
  }
  exclusive_scan(cnt.as<uint32_t>(), pos.as<uint32_t>(), nwords, nullptr, s, scratch);
  if (n && demoted) {
    k_demote_list<<<grid_for(nwords, 256, 8), 256, 0, s>>>(nwords, accw, used.as<uint32_t>(),
                                                            pos.as<uint32_t>(), demoted);
    CYC_LAUNCHED();
  }
  uint32_t nd = 0;
  CYC_CUDA(cudaMemcpyAsync(&nd, pos.as<uint32_t>() + nwords, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  return nd;
}

}  // namespace cyc
