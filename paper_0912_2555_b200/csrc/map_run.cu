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
// after k steps x[v] = max{u in F : path u -> v of length 1..k}. Every step
// reads the frozen map buffer P[cur] (= x_{k-1}) and produces P[cur^1]
// (= x_k), which then becomes current. P[cur^1] enters the step holding
// x_{k-2}, which differs from x_{k-1} exactly at the vertices changed in
// step k-1 — the frontier, kept as a bitmap. Two step kinds:
//   pull  dense over all rows of the gather index (the north_star SpMV in
//         the (max, vertex-id) semiring); each lane walks R rows of the
//         column-major HYB slab in lock-step (several independent gathers in
//         flight); rows longer than kHeavyDeg as kHeavyChunk-edge warp chunks
//         (grouped by L2-sized column blocks on large graphs).
//   push  only frontier vertices act: each max-copies its own x_{k-1} into
//         P[cur^1] and scatters cand = max(x_{k-1}[u], u+1 if accepting) to
//         its targets with atomicMax. A vertex that did not change cannot
//         change anyone's max, so this equals the dense step.
// Both kinds record the vertices they raise in the next frontier bitmap (with
// a one-bit-per-word summary so a sparse frontier is found without scanning
// all n/32 words); vertices of push degree > kBigDeg are also split into
// kChunk-edge chunks expanded by whole warps. The step kind is chosen on the
// device from the frontier's edge count (push when edges * alpha < m,
// alpha 16 by default): direction-optimising traversal.
//
// Self-witness (map_engine.cpp:66): exact per row in pull; push (and heavy
// pull rows) record raises to exactly v+1 of accepting v as candidates,
// confirmed after the barrier by reading the new buffer.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/cyc_gen.h"
#include "map_run.cuh"

namespace cg = cooperative_groups;

namespace cyc {

namespace {

constexpr int kRunThreads = 1024;
// threads of the degree-ordered instantiation (C3 loop, 8 steps: 512 -> 28.9
// ms, 768 -> 25.8, 1024 -> 24.8; scripts/build_variant.sh)
#ifndef CYC_RL_THREADS
#define CYC_RL_THREADS 1024
#endif
constexpr int kRunThreadsRL = CYC_RL_THREADS;
#ifndef CYC_SLAB_B
#define CYC_SLAB_B 2
#endif
template <bool RL>
constexpr int run_threads() { return RL ? kRunThreadsRL : kRunThreads; }
constexpr int kModePull = 1, kModePush = 2;
constexpr int kRows = 4;            // rows per lane in a pull step (the ovf test below assumes 4)
static_assert(kRows == 4, "pull overflow test unrolled for 4 rows");
constexpr int kBatch = 4;           // frontier vertices per lane in a push step
#ifndef CYC_HEAVY_UNIT
#define CYC_HEAVY_UNIT 64               // heavy-slab chunks per dynamic claim (pull_heavy_slab)
#endif
#ifndef CYC_LIGHT_UNIT
#define CYC_LIGHT_UNIT 16               // light slices per dynamic claim (pull_sell; 8-32 best on C3, 64+ leaves tails)
#endif
constexpr int kHeavyPerLane = kHeavyChunk / 32;  // pull heavy chunk edges per lane
constexpr int kHeavyBatch = 4;                     // heavy chunks in flight per warp

// Column streams of a degree-ordered plan (sliced ELL, heavy slab) are larger
// than L2 and read once per step: load them evict-first so they do not push
// the hot map words out (ld.global.cs). The identity layout's HYB slab is not
// hinted: on L2-resident graphs (config 2) it is re-read by every step.
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) {
#ifdef CYC_STREAM_NA  // no L1 allocation, L2 evict-first policy
  uint32_t v;
  asm volatile("{\n\t.reg .b64 pol;\n\tcreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
               "ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], pol;\n\t}"
               : "=r"(v) : "l"(p));
  return v;
#else
  return __ldcs(p);
#endif
}
__device__ __forceinline__ uint4 ld_stream(const uint4* p) { return __ldcs(p); }

// A map word of the frozen buffer at a gathered position, L1-allocating:
// measured on config 3, letting the colder positions bypass L1
// (ld.global.nc.L1::no_allocate) doubles a run (21.2 -> 45.1 ms) — random
// gathers need the L1 allocation path.
__device__ __forceinline__ uint32_t ld_gather(const uint32_t* __restrict__ P, uint32_t u) { return __ldca(P + u); }

// Frontier filter of a pull step on a degree-ordered plan. Step k's pull
// only needs the sources that changed in step k-1: x_{k-1}[v] already
// dominates cand_{k-2}(u) for every gathered u, and F is fixed within a
// fixpoint, so an unchanged source cannot raise anyone (map_engine.cpp:56-63
// computes the same maximum over all sources). The previous step's frontier
// bits of positions [0, k) -- the most-gathered vertices, ~65 % of all
// gathers on config 3 for k = 2^19 -- are staged in shared memory; a gather
// from such a position is issued only if its bit is set. Measured: the random
// L2 gathers are what bounds a dense step (~283 G/s per GPU,
// scripts/micro/gather_bw.cu), so every skipped one counts.
// (the array is referenced directly, not through a pointer, so the compiler
// addresses it in the shared window without per-access conversions)
extern __shared__ uint32_t hot_sh[];

struct Hot {
  uint32_t k;     // positions with staged frontier bits (0: no filter)
  uint32_t vmax;  // the largest value of this fixpoint (max id+1 over F): a row
                  // already holding it cannot rise, its gathers are skipped
};

__device__ __forceinline__ uint32_t ld_word(const Hot& h, const uint32_t* __restrict__ P, uint32_t u) {
  bool need = true;
  if (u < h.k) need = (hot_sh[u >> 5] >> (u & 31u)) & 1u;
  uint32_t w = 0;  // NIL: contributes nothing to the maximum
  if (need) w = ld_gather(P, u);
  return w;
}

__device__ __forceinline__ bool bit_of(const uint32_t* words, uint32_t v) {
  return (__ldcg(words + (v >> 5)) >> (v & 31u)) & 1u;
}

__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// This rank's view of the grid (rank-relative block and warp indices).
__device__ __forceinline__ uint32_t vblk(const RunArgs& a) { return blockIdx.x - a.blk0; }
__device__ __forceinline__ uint32_t gwarp(const RunArgs& a) { return (vblk(a) * blockDim.x + threadIdx.x) >> 5; }
__device__ __forceinline__ uint32_t nwarps(const RunArgs& a) { return (a.nblk * blockDim.x) >> 5; }
// The same warps numbered across the blocks first (warp w of block b ->
// w * nblk + b): loops over few items (push steps of small frontiers) then
// spread them over every SM. Numbered block-major, config 5's 128 frontier
// groups all ran on 4 SMs, whose load units (one divergent-load wavefront per
// clock) spent ~5 us of each 10 us step on their scattered loads.
__device__ __forceinline__ uint32_t swarp(const RunArgs& a) { return (threadIdx.x >> 5) * a.nblk + vblk(a); }

// Trace hook: latest time any warp passed phase `ph` of the current step.
__device__ __forceinline__ void phase_mark(const RunArgs& a, unsigned long long k, int ph) {
  if (a.trace && k < a.trace_cap && lane_id() == 0) {
    const uint32_t spread = (gwarp(a)) & 15u;
    atomicMax(a.trace + 64u * k + 16u + 16u * ph + spread, gtimer());
  }
}

// vertex id of storage position p (plan.cuh; identity without a plan)
// (RL: the run uses a relabelled plan; a separate instantiation keeps the
// identity layout's loops free of the lookups)
template <bool RL>
__device__ __forceinline__ uint32_t oid(const RunArgs& a, uint32_t p) {
  if constexpr (RL) return __ldg(a.orig + p);
  return p;
}

// A self-witness candidate (raised to exactly id+1): appended while the
// list has room; a step whose candidates overflow it (a vertex can be raised to
// id+1 by several sources) is confirmed by a dense scan instead.
__device__ __forceinline__ void add_cand(const RunArgs& a, uint32_t* Cn, unsigned int* cnt, uint32_t v) {
  const uint32_t pos = atomicAdd(cnt, 1u);
  if (pos < a.cand_cap) Cn[pos] = v;
}

// candidate value the vertex at position u with map word w contributes to its
// successors: max(x[u], id(u)+1 if accepting) (map_engine.cpp:56-63)
template <bool RL>
__device__ __forceinline__ uint32_t cand_of(const RunArgs& a, uint32_t w, uint32_t u) {
  if constexpr (RL) return (w & kFlag) ? max(w & kCode, oid<RL>(a, u) + 1u) : w;
  return max(w & kCode, (w >> 31) * (u + 1u));
}

// ---------------------------------------------------------- block helpers
constexpr uint32_t kWlCap = 1024;  // per-CTA list of newly non-zero frontier words

constexpr uint32_t kBigCap = 128;   // per-CTA big vertices awaiting chunk expansion

struct BlockSh {
  unsigned long long w[32][3];
  unsigned long long bcast;
  uint32_t wmin[33];
  uint32_t wl_n, wl_base, wl_cnt;
  uint32_t wl[kWlCap];
  uint32_t big_n;
  uint32_t bigv[kBigCap];
  uint32_t bigb[kBigCap];   // first edge
  uint32_t bige[kBigCap];   // end edge
  uint32_t bigc[kBigCap];   // first chunk slot
};

// A frontier word became non-zero in this step: remember it for the next
// push step (block-local, flushed once per CTA by wl_flush).
__device__ __forceinline__ void note_word(BlockSh* sh, uint32_t wi) {
  const uint32_t pos = atomicAdd(&sh->wl_n, 1u);
  if (pos < kWlCap) sh->wl[pos] = wi;
}

// Appends the CTA's noted words to the step's global word list with one
// atomic; an overflowing CTA flags the list incomplete (the next push step then
// scans the whole bitmap). Call with the whole CTA after its notes are done.
__device__ void wl_flush(BlockSh* sh, SlotCtl* sl, uint32_t* wl, uint32_t wl_cap) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t n = sh->wl_n;
    const uint32_t cnt = n < kWlCap ? n : kWlCap;
    uint32_t base = 0;
    if (cnt) base = atomicAdd(&sl->wl_count, cnt);
    if (n > kWlCap || base + cnt > wl_cap) *(volatile unsigned int*)&sl->wl_over = 1u;
    sh->wl_base = base;
    sh->wl_n = cnt;
  }
  __syncthreads();
  const uint32_t cnt = sh->wl_n, base = sh->wl_base;
  for (uint32_t i = threadIdx.x; i < cnt && base + i < wl_cap; i += blockDim.x) wl[base + i] = sh->wl[i];
  __syncthreads();
  if (threadIdx.x == 0) sh->wl_n = 0;
}

__device__ unsigned long long block_sum(unsigned long long x, BlockSh* sh) {
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  x = warp_sum64(x);
  if (lane == 0) sh->w[wid][0] = x;
  __syncthreads();
  if (wid == 0) {
    unsigned long long y = lane < nw ? sh->w[lane][0] : 0ull;
    y = warp_sum64(y);
    if (lane == 0) sh->bcast = y;
  }
  __syncthreads();
  const unsigned long long r = sh->bcast;
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
  unsigned long long first = 0;   // vertices newly entered in the next frontier
  unsigned long long fedges = 0;  // their push degrees (when known)
};

// One fused 3-value reduction, one flag store and two atomics per CTA, then
// the CTA's frontier-word list is flushed.
__device__ unsigned long long big_flush(const RunArgs& a, BlockSh* sh, uint4* bc, SlotCtl* sl,
                                        bool flag_overflow);
__device__ void step_flags(const RunArgs& a, const StepAcc& acc, SlotCtl* sl, BlockSh* sh,
                           uint32_t* wl, uint32_t wl_cap, uint4* bc) {
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned long long bigdeg = big_flush(a, sh, bc, sl, true);  // begins with a CTA barrier
  // the CTA's slice of the word list (wl_flush's job, folded in): thread 0's
  // atomic is in flight while the counters are reduced (one round trip and
  // two CTA barriers less per step than reducing first)
  uint32_t wl_base = 0, wl_cnt = 0;
  bool wl_ovf = false;
  if (threadIdx.x == 0) {
    const uint32_t n = sh->wl_n;  // every note_word of the step came before the barrier
    wl_cnt = n < kWlCap ? n : kWlCap;
    if (wl_cnt) wl_base = atomicAdd(&sl->wl_count, wl_cnt);
    wl_ovf = n > kWlCap;
  }
  const unsigned long long r = warp_sum64(acc.raised), f = warp_sum64(acc.first),
                           e = warp_sum64(acc.fedges) + (threadIdx.x == 0 ? bigdeg : 0ull);
  if (lane == 0) {
    sh->w[wid][0] = r;
    sh->w[wid][1] = f;
    sh->w[wid][2] = e;
  }
  __syncthreads();
  if (wid == 0) {
    unsigned long long rr = lane < nw ? sh->w[lane][0] : 0ull;
    unsigned long long ff = lane < nw ? sh->w[lane][1] : 0ull;
    unsigned long long ee = lane < nw ? sh->w[lane][2] : 0ull;
    rr = warp_sum64(rr);
    ff = warp_sum64(ff);
    ee = warp_sum64(ee);
    if (lane == 0) {
      if (rr) *(volatile unsigned int*)&sl->changed = 1u;
      if (ff) atomicAdd(&sl->nraised, (unsigned)ff);
      if (ee) atomicAdd(&sl->fedges, ee);
    }
  }
  if (threadIdx.x == 0) {
    if (wl_ovf || wl_base + wl_cnt > wl_cap) *(volatile unsigned int*)&sl->wl_over = 1u;
    sh->wl_base = wl_base;
    sh->wl_cnt = wl_cnt;
    sh->wl_n = 0;  // next written after the grid barrier that ends the step
  }
  __syncthreads();
  const uint32_t cnt = sh->wl_cnt, base = sh->wl_base;
  for (uint32_t i = threadIdx.x; i < cnt && base + i < wl_cap; i += blockDim.x) wl[base + i] = sh->wl[i];
}

// A step's final counters, read once after the barrier that ends it: the
// loop's exit tests, the next step's direction choice and the push step's
// word list all come from this one round trip (small steps are latency
// bound: config 5 runs 16767 of them).
struct SlotView {
  unsigned long long fedges;
  uint32_t nraised, changed, nchunk, cand_cnt, wit, wl_count, wl_over;
};
static_assert(offsetof(SlotCtl, fedges) == 0 && offsetof(SlotCtl, nraised) == 8 && offsetof(SlotCtl, changed) == 12 &&
                  offsetof(SlotCtl, nchunk) == 16 && offsetof(SlotCtl, cand_cnt) == 20 &&
                  offsetof(SlotCtl, wit) == 24 && offsetof(SlotCtl, wl_count) == 28 &&
                  offsetof(SlotCtl, wl_over) == 32,
              "ld_slot unpacks SlotCtl by offset");
__device__ __forceinline__ SlotView ld_slot(const SlotCtl* s) {
  const uint4* q = reinterpret_cast<const uint4*>(s);
  const uint4 x = __ldcg(q), y = __ldcg(q + 1);
  SlotView v;
  v.fedges = ((unsigned long long)x.y << 32) | x.x;
  v.nraised = x.z;
  v.changed = x.w;
  v.nchunk = y.x;
  v.cand_cnt = y.y;
  v.wit = y.z;
  v.wl_count = y.w;
  v.wl_over = __ldcg(&s->wl_over);
  return v;
}

// Sets bit v of the frontier bitmap (and its summary bit); true iff new.
__device__ __forceinline__ bool mark(uint32_t* fb, BlockSh* sh, uint32_t v, bool precheck = false) {
  const uint32_t w = v >> 5, bit = 1u << (v & 31u);
  // hub rows / large frontiers raise one vertex many times: a read first
  // avoids contended atomics (skipped on latency-bound small frontiers)
  if (precheck && (__ldcg(fb + w) & bit)) return false;
  const uint32_t old = atomicOr(fb + w, bit);
  if (old == 0u) note_word(sh, w);
  return !(old & bit);
}

// Chunks of a big-degree vertex for the next push step, written by one lane
// (fallback when the CTA's list is full); returns the degree.
__device__ uint32_t enlist_now(const RunArgs& a, uint32_t v, uint4* bc, unsigned int* nchunk) {
  const uint32_t b = __ldg(a.poff + v), e = __ldg(a.poff + v + 1);
  const uint32_t nc = (e - b + kChunk - 1) / kChunk;
  const uint32_t base = atomicAdd(nchunk, nc) & ~kChunkOver;
  for (uint32_t c = 0; c < nc && base + c < a.chunk_cap; ++c)
    bc[base + c] = make_uint4(v, b + c * kChunk, min(e, b + (c + 1) * kChunk), 0u);
  return e - b;
}

// A big-degree vertex entered the next frontier: note it in the CTA's list;
// the whole CTA writes its chunk descriptors at step end (big_flush), so no
// single lane serialises hundreds of stores. When the list is full the
// vertex is left out and big_flush flags the step (chunk_over): a following
// push step re-chunks the whole frontier, and a following pull step — what
// large frontiers lead to — needs no chunks at all (config 3's first push
// step spent most of its 2.7 ms in one-lane fallback expansions). Returns the
// degree if it was not queued, else 0 (big_flush accounts it).
__device__ __forceinline__ uint32_t enlist(const RunArgs& a, uint32_t v, uint4* bc,
                                           unsigned int* nchunk, BlockSh* sh) {
  const uint32_t pos = atomicAdd(&sh->big_n, 1u);
  if (pos < kBigCap) {
    sh->bigv[pos] = v;
    return 0u;
  }
  return __ldg(a.poff + v + 1) - __ldg(a.poff + v);
}

// Same, expanding here when the list is full (re-chunking passes).
__device__ __forceinline__ uint32_t enlist_all(const RunArgs& a, uint32_t v, uint4* bc,
                                               unsigned int* nchunk, BlockSh* sh) {
  const uint32_t pos = atomicAdd(&sh->big_n, 1u);
  if (pos < kBigCap) {
    sh->bigv[pos] = v;
    return 0u;
  }
  return enlist_now(a, v, bc, nchunk);
}

// Expands the CTA's noted big vertices into chunks (whole CTA); returns the
// sum of their degrees in thread 0.
__device__ unsigned long long big_flush(const RunArgs& a, BlockSh* sh, uint4* bc, SlotCtl* sl,
                                        bool flag_overflow = true) {
  unsigned int* nchunk = &sl->nchunk;
  __syncthreads();
  // the list overflowed (enlist left vertices out): flag the step in the
  // count's top bit, so the next step learns it from the load it makes anyway
  if (flag_overflow && sh->big_n > kBigCap && threadIdx.x == 0) atomicOr(nchunk, kChunkOver);
  const uint32_t nb = min(sh->big_n, kBigCap);
  unsigned long long deg = 0;
  if (nb == 0) return 0;
  for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) {
    const uint32_t v = sh->bigv[i];
    sh->bigb[i] = __ldg(a.poff + v);
    sh->bige[i] = __ldg(a.poff + v + 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t total = 0;
    for (uint32_t i = 0; i < nb; ++i) {
      sh->bigc[i] = total;
      total += (sh->bige[i] - sh->bigb[i] + kChunk - 1) / kChunk;
      deg += sh->bige[i] - sh->bigb[i];
    }
    const uint32_t base = atomicAdd(nchunk, total) & ~kChunkOver;
    for (uint32_t i = 0; i < nb; ++i) sh->bigc[i] += base;
  }
  __syncthreads();
  for (uint32_t i = 0; i < nb; ++i) {
    const uint32_t v = sh->bigv[i], b = sh->bigb[i], e = sh->bige[i], c0 = sh->bigc[i];
    const uint32_t nc = (e - b + kChunk - 1) / kChunk;
    for (uint32_t c = threadIdx.x; c < nc; c += blockDim.x)
      if (c0 + c < a.chunk_cap) bc[c0 + c] = make_uint4(v, b + c * kChunk, min(e, b + (c + 1) * kChunk), 0u);
  }
  __syncthreads();
  if (threadIdx.x == 0) sh->big_n = 0;
  return deg;
}

struct PushCtx {
  const uint32_t* Pc;  // frozen x_{k-1}
  uint32_t* Pn;        // x_k under construction
  uint32_t* fb;        // next frontier
  BlockSh* sh;
  uint4* bc;
  unsigned int* nchunk;
  uint32_t* Cn;
  unsigned int* ccnt;
  bool contend;  // large frontier: check Pn before atomics (hub targets)
};

// Batched Jacobi push of val[r] into tgt[r], as predicated stages (read the
// frozen value, fire-and-forget atomicMax, frontier mark, big-vertex chunks)
// so the R chains of a lane overlap.
template <bool RL, int R>
__device__ __forceinline__ void raise_batch(const RunArgs& a, const PushCtx& c,
                                            const uint32_t (&tgt)[R], const uint32_t (&val)[R],
                                            StepAcc& acc) {
  uint32_t old[R];
  bool go[R];
  uint32_t bw[R], b[R], e[R];
  // small frontiers (latency bound): the target's big bit and degree are
  // loaded with its value, before knowing it is raised (one round trip less)
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const bool spec = !c.contend && tgt[r] != kNone;
    old[r] = tgt[r] != kNone ? __ldca(c.Pc + tgt[r]) : kCode;
    bw[r] = spec ? __ldcg(a.bigm + (tgt[r] >> 5)) : 0u;
    b[r] = spec ? __ldg(a.poff + tgt[r]) : 0u;
    e[r] = spec ? __ldg(a.poff + tgt[r] + 1) : 0u;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) go[r] = tgt[r] != kNone && val[r] > (old[r] & kCode);
  uint32_t cur[R];  // hub targets: many sources raise the same word, skip settled atomics
#pragma unroll
  for (int r = 0; r < R; ++r) cur[r] = go[r] && c.contend ? __ldcg(c.Pn + tgt[r]) : 0u;
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (go[r] && ((old[r] & kFlag) | val[r]) > cur[r]) atomicMax(c.Pn + tgt[r], (old[r] & kFlag) | val[r]);
  // frontier bits of the raised targets: every atomic of the batch in flight
  // together (a per-target mark() would wait for each result before the next)
  bool first[R], need[R];
  uint32_t prev[R];
#pragma unroll
  for (int r = 0; r < R; ++r) need[r] = go[r];
  if (c.contend) {  // hub targets: read first, skip bits already set
#pragma unroll
    for (int r = 0; r < R; ++r) prev[r] = need[r] ? __ldcg(c.fb + (tgt[r] >> 5)) : 0u;
#pragma unroll
    for (int r = 0; r < R; ++r) need[r] = need[r] && !((prev[r] >> (tgt[r] & 31u)) & 1u);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) prev[r] = need[r] ? atomicOr(c.fb + (tgt[r] >> 5), 1u << (tgt[r] & 31u)) : ~0u;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    first[r] = need[r] && !((prev[r] >> (tgt[r] & 31u)) & 1u);
    if (need[r] && prev[r] == 0u) note_word(c.sh, tgt[r] >> 5);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {  // large frontiers: one round trip for the big bit and degree of new ones
    if (c.contend) {
      bw[r] = first[r] ? __ldcg(a.bigm + (tgt[r] >> 5)) : 0u;
      b[r] = first[r] ? __ldg(a.poff + tgt[r]) : 0u;
      e[r] = first[r] ? __ldg(a.poff + tgt[r] + 1) : 0u;
    } else if (!first[r]) {
      bw[r] = b[r] = e[r] = 0u;
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    acc.raised += go[r];
    acc.first += first[r];
    acc.fedges += e[r] - b[r];
    if (a.world == 1 && ((bw[r] >> (tgt[r] & 31u)) & 1u)) acc.fedges += enlist(a, tgt[r], c.bc, c.nchunk, c.sh);
    if (go[r] && (old[r] & kFlag) && val[r] == oid<RL>(a, tgt[r]) + 1u) add_cand(a, c.Cn, c.ccnt, tgt[r]);
  }
}

// ------------------------------------------------------------------ pull
// End of a light row group (R rows per lane, rows base + 32k + lane): write
// the new words (rows flagged in `skip` belong to the heavy-chunk pass), the
// exact self-witness, the next frontier words and big-vertex chunks.
template <bool RL, int R>
__device__ __forceinline__ void rows_epilogue(const RunArgs& a, uint32_t base, const uint32_t (&own)[R],
                                              const uint32_t (&best)[R], uint32_t skip, uint32_t* __restrict__ Q,
                                              uint32_t* fb, BlockSh* sh, uint32_t* fp, uint4* bc, SlotCtl* sl,
                                              StepAcc& acc) {
  const uint32_t lane = lane_id();
  uint32_t words[R], hvy[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const uint32_t v = base + 32u * k + lane;
    const bool up = !((skip >> k) & 1u) && best[k] > (own[k] & kCode);
    if (!((skip >> k) & 1u)) Q[v] = (own[k] & kFlag) | best[k];
    if ((own[k] & kFlag) && !((skip >> k) & 1u)) {
      const uint32_t id = oid<RL>(a, v);
      if (best[k] == id + 1u) atomicMin(&sl->wit, id);
    }
    words[k] = __ballot_sync(kFull, up);
    hvy[k] = __ballot_sync(kFull, (skip >> k) & 1u);
    acc.raised += up;
    acc.first += up;
  }
  // next frontier words (the bitmap is zero at step start; heavy rows are
  // disjoint): fire-and-forget ORs, previous frontier words consumed. A word
  // holding heavy rows may also be marked by their warps (mark(), which lists
  // the word when it finds it zero): list it here only if this OR found it
  // zero too, so the next push step's word list has no duplicates.
  if (lane < (uint32_t)R) {
    uint32_t wd = 0, hw = 0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      wd = lane == (uint32_t)k ? words[k] : wd;
      hw = lane == (uint32_t)k ? hvy[k] : hw;
    }
    const uint32_t wi = (base >> 5) + lane;
    fp[wi] = 0u;
    if (wd) {
      if (!hw) {
        atomicOr(fb + wi, wd);
        note_word(sh, wi);
      } else if (atomicOr(fb + wi, wd) == 0u) {
        note_word(sh, wi);
      }
    }
  }
  // raised vertices of big push degree: chunks for the next push step
  uint32_t big[R];
#pragma unroll
  for (int k = 0; k < R; ++k) big[k] = words[k] ? __ldcg(a.bigm + (base >> 5) + k) & words[k] : 0u;
#pragma unroll
  for (int k = 0; k < R; ++k)
    if (a.world == 1 && ((big[k] >> lane) & 1u)) acc.fedges += enlist(a, base + 32u * k + lane, bc, &sl->nchunk, sh);
}

// Light rows of a pull step. Each lane owns R rows (32*R consecutive rows per
// warp, rows padded to a multiple of kRowPad so no bound checks). Their first
// K columns come from the column-major HYB slab; absent entries point at the
// always-NIL padding slot, so every gather is unconditional and the inner loop
// is straight-line: one round trip for own values + slab, one for gathers.
// Rows flagged in `ovf` (longer than K, or heavy) take a slow path.
template <bool RL, int K, int R>
__device__ __forceinline__ void pull_light(const RunArgs& a, const uint32_t* __restrict__ P,
                                           uint32_t* __restrict__ Q, uint32_t* fb, BlockSh* sh,
                                           uint32_t* fp, uint4* bc, SlotCtl* sl, StepAcc& acc) {
  const uint32_t lane = lane_id();
  const uint32_t gw = gwarp(a);
  const uint32_t nw = nwarps(a);
  static_assert(32u * R <= kRowPad && kRowPad % (32u * R) == 0, "a row group must not run past the row padding");
  const uint32_t np = a.n_pad;
  for (uint32_t base = gw * (32u * R); base < np; base += nw * (32u * R)) {
    uint32_t own[R], best[R];
    uint32_t anyov = 0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      own[k] = __ldca(P + base + 32u * k + lane);
      anyov |= __ldg(a.ovf + (base >> 5) + k);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      uint32_t u[R];
#pragma unroll
      for (int k = 0; k < R; ++k) u[k] = __ldg(a.ell + (size_t)j * np + base + 32u * k + lane);
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const uint32_t w = __ldca(P + u[k]);
        const uint32_t c = cand_of<RL>(a, w, u[k]);
        best[k] = j == 0 ? max(own[k] & kCode, c) : max(best[k], c);
      }
    }
    if (K == 0) {
#pragma unroll
      for (int k = 0; k < R; ++k) best[k] = own[k] & kCode;
    }
    uint32_t skip = 0;  // bit k: heavy row (owned by the chunk pass)
    if (anyov) {
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const uint32_t v = base + 32u * k + lane;
        if ((__ldg(a.ovf + (base >> 5) + k) >> lane) & 1u) {
          const uint32_t b = __ldg(a.goff + v), e = __ldg(a.goff + v + 1);
          if (e - b > a.heavy_deg) {
            skip |= 1u << k;
          } else {
            for (uint32_t i = b + K; i < e; ++i) {
              const uint32_t u = __ldg(a.gcol + i);
              best[k] = max(best[k], cand_of<RL>(a, __ldca(P + u), u));
            }
          }
        }
      }
    }
    rows_epilogue<RL, R>(a, base, own, best, skip, Q, fb, sh, fp, bc, sl, acc);
  }
}

// Light rows from the sliced-ELL layout of a degree-ordered plan (plan.cuh):
// slice s = rows [32s, 32s+32), padded to its own widest row, column-major, so
// every column load is one coalesced 128 B line and no row takes a serial
// overflow path (rows of similar length are neighbours in degree order). A
// warp takes R slices; J columns of each per round, all R*J gathers in flight.
template <bool RL, int R, int J>
__device__ __forceinline__ void pull_sell(const RunArgs& a, const uint32_t* __restrict__ P,
                                          uint32_t* __restrict__ Q, uint32_t* fb, BlockSh* sh,
                                          uint32_t* fp, uint4* bc, SlotCtl* sl, StepAcc& acc, const Hot& hot) {
  const uint32_t lane = lane_id();
  const uint32_t gw = gwarp(a);
  const uint32_t nw = nwarps(a);
  static_assert((kRowPad / 32u) % R == 0, "slices per row padding must be a multiple of R");
  const uint32_t np = a.n_pad, nsl = (a.row_hi - a.row_lo) / 32u;  // this rank's slices
  // Slices are claimed kLightUnit at a time from a per-step counter, the next
  // claim in flight while the current unit runs: warps that finished their
  // share of the heavy slab early take more light rows, so the step ends
  // together (static shares left up to ~20 % of warp time at the barriers).
  constexpr uint32_t kLightUnit = CYC_LIGHT_UNIT;
  static_assert(kLightUnit % R == 0, "a unit holds whole slice groups");
  (void)gw;
  (void)nw;
  uint32_t u0 = 0;
  if (lane_id() == 0) u0 = atomicAdd(&sl->light_next, kLightUnit);
  u0 = __shfl_sync(kFull, u0, 0);
  while (u0 < nsl) {
    uint32_t u1 = 0;  // the next claim, in flight meanwhile
    if (lane_id() == 0) u1 = atomicAdd(&sl->light_next, kLightUnit);
    for (uint32_t s0 = u0; s0 < min(u0 + kLightUnit, nsl); s0 += R) {
      const uint32_t base = a.row_lo + s0 * 32u;
      uint4 d[R];
      uint32_t own[R], best[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        d[k] = __ldg(a.sdesc + s0 + k);
        own[k] = __ldca(P + base + 32u * k + lane);
      }
      uint32_t wmax = 0, skip = 0;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        best[k] = own[k] & kCode;
        wmax = max(wmax, d[k].y);
        skip |= ((d[k].z >> lane) & 1u) << k;
      }
      uint32_t wlim[R];  // a saturated row reads no columns at all
#pragma unroll
      for (int k = 0; k < R; ++k) wlim[k] = best[k] == hot.vmax ? 0u : d[k].y;
      for (uint32_t j = 0; j < wmax; j += J) {
        uint32_t u[R][J], w[R][J];
#pragma unroll
        for (int k = 0; k < R; ++k)
#pragma unroll
          for (int t = 0; t < J; ++t)
            u[k][t] = j + t < wlim[k] ? ld_stream(a.sell + ((size_t)d[k].x + j + t) * 32u + lane) : np;
#pragma unroll
        for (int k = 0; k < R; ++k)
#pragma unroll
          for (int t = 0; t < J; ++t) w[k][t] = ld_word(hot, P, u[k][t]);
        if constexpr (RL) {
#pragma unroll
          for (int k = 0; k < R; ++k)
#pragma unroll
            for (int t = 0; t < J; ++t)
              if (w[k][t] & kFlag) u[k][t] = __ldg(a.orig + u[k][t]);
        }
#pragma unroll
        for (int k = 0; k < R; ++k)
#pragma unroll
          for (int t = 0; t < J; ++t)
            best[k] = max(best[k], max(w[k][t] & kCode, (w[k][t] >> 31) * (u[k][t] + 1u)));
      }
      rows_epilogue<RL, R>(a, base, own, best, skip, Q, fb, sh, fp, bc, sl, acc);
    }
    u0 = __shfl_sync(kFull, u1, 0);
  }
}

// Heavy rows of a pull step (the long poles): a warp takes B chunks of at
// most 32*kHeavyPerLane edges at once, every lane issuing all its loads
// together; lane k finalises chunk k (own value prefetched) with an atomicMax
// into Q (Q holds x_{k-2}, never larger).
template <bool RL, int B, bool PRE>
__device__ __forceinline__ void pull_heavy(const RunArgs& a, const uint32_t* __restrict__ P,
                                           uint32_t* __restrict__ Q, uint32_t* fb, BlockSh* sh, uint4* bc,
                                           SlotCtl* sl, uint32_t* Cn, StepAcc& acc) {
  const uint32_t lane = lane_id();
  const uint32_t gw = gwarp(a);
  const uint32_t nw = nwarps(a);
  // a warp takes B consecutive chunks (often of one hub row: their results
  // merge before a single finalisation); tail warps do fewer light rows
  for (uint32_t c0 = (nw - 1u - gw) * B; c0 < a.n_heavy; c0 += nw * B) {
    uint4 ch[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const uint32_t c = c0 + (uint32_t)k;
      ch[k] = c < a.n_heavy ? a.heavy[c] : make_uint4(0u, 0u, 0u, 0u);
    }
    uint32_t own = 0;
#pragma unroll
    for (int k = 0; k < B; ++k)
      if (lane == (uint32_t)k && ch[k].z > ch[k].y) own = __ldca(P + ch[k].x);
    // every gather unconditional (absent edges read the always-NIL slot
    // n_pad), all issued before any is used: B*kHeavyPerLane in flight per lane
    uint32_t u[B][kHeavyPerLane], w[B][kHeavyPerLane];
#pragma unroll
    for (int k = 0; k < B; ++k)
#pragma unroll
      for (int r = 0; r < kHeavyPerLane; ++r) {
        const uint32_t i = ch[k].y + lane + 32u * r;
        u[k][r] = i < ch[k].z ? __ldg(a.gcol + i) : a.n_pad;
      }
#pragma unroll
    for (int k = 0; k < B; ++k)
#pragma unroll
      for (int r = 0; r < kHeavyPerLane; ++r) w[k][r] = __ldca(P + u[k][r]);
    if constexpr (RL) {  // ids of the accepting sources only, again all in flight together
#pragma unroll
      for (int k = 0; k < B; ++k)
#pragma unroll
        for (int r = 0; r < kHeavyPerLane; ++r)
          if (w[k][r] & kFlag) u[k][r] = __ldg(a.orig + u[k][r]);
    }
    uint32_t best[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      best[k] = 0;
#pragma unroll
      for (int r = 0; r < kHeavyPerLane; ++r)
        best[k] = max(best[k], max(w[k][r] & kCode, (w[k][r] >> 31) * (u[k][r] + 1u)));
    }
#pragma unroll
    for (int k = 0; k < B; ++k) best[k] = __reduce_max_sync(kFull, best[k]);
    uint32_t mine = 0, v = 0;
    bool live = false;
#pragma unroll
    for (int k = 0; k < B; ++k)
      if (lane == (uint32_t)k) {
        v = ch[k].x;
        // first chunk of its row within the group finalises the merged max
        live = ch[k].z > ch[k].y && (k == 0 || ch[k - 1].x != v || ch[k - 1].z <= ch[k - 1].y);
#pragma unroll
        for (int j = 0; j < B; ++j)
          if (ch[j].x == v && ch[j].z > ch[j].y) mine = max(mine, best[j]);
      }
    if (live) {
      mine = max(mine, own & kCode);
      // chunks of one hub row run on neighbouring warps: skip the atomic when
      // another chunk already raised Q[v] at least as far
      if (!PRE || ((own & kFlag) | mine) > __ldcg(Q + v)) atomicMax(Q + v, (own & kFlag) | mine);
      if (mine > (own & kCode)) {
        ++acc.raised;
        if (mark(fb, sh, v, PRE)) {
          ++acc.first;
          if (a.world == 1 && bit_of(a.bigm, v)) acc.fedges += enlist(a, v, bc, &sl->nchunk, sh);
        }
        if ((own & kFlag) && mine == oid<RL>(a, v) + 1u) add_cand(a, Cn, &sl->cand_cnt, v);
      }
    }
  }
}

// Finished heavy rows, one per lane (pv = row, pm = max of its chunks seen by
// this warp, po = its frozen word): written back together so the dependent
// round trips (Q precheck, frontier mark) are paid once per 32 rows.
template <bool RL>
__device__ __forceinline__ void heavy_flush(const RunArgs& a, bool live, uint32_t pv, uint32_t pm, uint32_t po,
                                            uint32_t* __restrict__ Q, uint32_t* fb, BlockSh* sh, uint4* bc,
                                            SlotCtl* sl, uint32_t* Cn, StepAcc& acc) {
  if (!live) return;
  const uint32_t mine = max(pm, po & kCode), word = (po & kFlag) | mine;
  // a row split between two warps is merged by atomicMax (Q holds x_{k-2} <= x_{k-1})
  if (word > __ldcg(Q + pv)) atomicMax(Q + pv, word);
  if (mine > (po & kCode)) {
    ++acc.raised;
    if (mark(fb, sh, pv, true)) {
      ++acc.first;
      if (a.world == 1 && bit_of(a.bigm, pv)) acc.fedges += enlist(a, pv, bc, &sl->nchunk, sh);
    }
    if ((po & kFlag) && mine == oid<RL>(a, pv) + 1u) add_cand(a, Cn, &sl->cand_cnt, pv);
  }
}

// Heavy rows of a degree-ordered plan: chunk c = 128 columns at hcol[128c..]
// (padded with the NIL slot n_pad), row hrow[c]; a row's chunks are
// consecutive. A warp owns a contiguous chunk range and walks it B chunks per
// round with the next round's columns, rows and own words prefetched, so the
// critical path is one gather round trip per round. Rows are merged in
// registers while the warp stays on them (a hub row's thousands of chunks
// cost one write-back per warp, not one atomic per chunk).
template <bool RL>
__device__ __forceinline__ void pull_heavy_slab(const RunArgs& a, const uint32_t* __restrict__ P,
                                                uint32_t* __restrict__ Q, uint32_t* fb, BlockSh* sh, uint4* bc,
                                                SlotCtl* sl, uint32_t* Cn, StepAcc& acc, const Hot& hot) {
  constexpr int B = CYC_SLAB_B, H = kHeavyPerLane;
  const uint32_t lane = lane_id();
  const uint32_t gw = gwarp(a);
  const uint32_t nw = nwarps(a);
  const uint32_t nh = a.n_hchunks, np = a.n_pad;
  // Chunks go in units of kHeavyUnit: unit gw first, then units claimed from
  // a per-step counter (the next claim in flight while a unit runs), so the
  // saturation skips' uneven savings do not leave warps idle at the barrier.
  constexpr uint32_t kHeavyUnit = CYC_HEAVY_UNIT;
  static_assert(kHeavyUnit % B == 0, "a unit holds whole rounds");
  uint32_t ub = gw * kHeavyUnit;
  if (ub >= nh) return;
  uint32_t ue = min(ub + kHeavyUnit, nh);
  uint32_t claim = 0;
  if (lane == 0) claim = atomicAdd(&sl->heavy_next, kHeavyUnit);
  uint32_t u[B][H], rr[B], ro[B];
#pragma unroll
  for (int k = 0; k < B; ++k) {
    const bool ok = ub + k < ue;
    rr[k] = ok ? ld_stream(a.hrow + ub + k) : kNone;
#pragma unroll
    for (int r = 0; r < H; ++r) u[k][r] = ok ? ld_stream(a.hcol + (size_t)(ub + k) * kHeavyChunk + 32u * r + lane) : np;
  }
#pragma unroll
  for (int k = 0; k < B; ++k) ro[k] = rr[k] != kNone ? __ldca(P + rr[k]) : 0u;
  uint32_t row = kNone, rmax = 0, rown = 0;       // the row this warp is on (uniform)
  uint32_t pv = 0, pm = 0, po = 0, npend = 0;     // finished rows awaiting write-back
  for (uint32_t c = ub; c < nh;) {
    uint32_t w[B][H];
    // saturated row (at step start, or its maximum so far in this warp's walk
    // already reached vmax): its chunk cannot raise it, gather nothing
    const bool row_sat = rmax == hot.vmax;
#pragma unroll
    for (int k = 0; k < B; ++k)
      if ((ro[k] & kCode) == hot.vmax || (row_sat && rr[k] == row))
#pragma unroll
        for (int r = 0; r < H; ++r) u[k][r] = np;
#pragma unroll
    for (int k = 0; k < B; ++k)
#pragma unroll
      for (int r = 0; r < H; ++r) w[k][r] = ld_word(hot, P, u[k][r]);
    uint32_t cn = c + B;  // the next round: on in this unit, or the claimed one
    if (cn >= ue) {
      ub = nw * kHeavyUnit + __shfl_sync(kFull, claim, 0);
      ue = min(ub + kHeavyUnit, nh);
      cn = ub;
      if (lane == 0 && ub < nh) claim = atomicAdd(&sl->heavy_next, kHeavyUnit);
    }
    uint32_t un[B][H], rn[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const bool ok = cn + k < ue;
      rn[k] = ok ? ld_stream(a.hrow + cn + k) : kNone;
#pragma unroll
      for (int r = 0; r < H; ++r)
        un[k][r] = ok ? ld_stream(a.hcol + (size_t)(cn + k) * kHeavyChunk + 32u * r + lane) : np;
    }
    if constexpr (RL) {
#pragma unroll
      for (int k = 0; k < B; ++k)
#pragma unroll
        for (int r = 0; r < H; ++r)
          if (w[k][r] & kFlag) u[k][r] = __ldg(a.orig + u[k][r]);
    }
    uint32_t best[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      best[k] = 0;
#pragma unroll
      for (int r = 0; r < H; ++r) best[k] = max(best[k], max(w[k][r] & kCode, (w[k][r] >> 31) * (u[k][r] + 1u)));
      best[k] = __reduce_max_sync(kFull, best[k]);
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {
      if (rr[k] == kNone) continue;
      if (rr[k] != row) {
        if (row != kNone) {
          if (lane == npend) {
            pv = row;
            pm = rmax;
            po = rown;
          }
          if (++npend == 32u) {
            heavy_flush<RL>(a, true, pv, pm, po, Q, fb, sh, bc, sl, Cn, acc);
            npend = 0;
          }
        }
        row = rr[k];
        rmax = 0;
        rown = ro[k];
      }
      rmax = max(rmax, best[k]);
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {  // next round's own words: its rows have arrived by now
      rr[k] = rn[k];
      ro[k] = rn[k] != kNone ? __ldca(P + rn[k]) : 0u;
#pragma unroll
      for (int r = 0; r < H; ++r) u[k][r] = un[k][r];
    }
    c = cn;
  }
  if (row != kNone) {
    if (lane == npend) {
      pv = row;
      pm = rmax;
      po = rown;
    }
    ++npend;
  }
  heavy_flush<RL>(a, lane < npend, pv, pm, po, Q, fb, sh, bc, sl, Cn, acc);
}

template <bool RL>
__device__ void pull_step(const RunArgs& a, uint32_t g, int cur, uint32_t vmax, BlockSh* sh,
                          unsigned long long tk) {
  const uint32_t* __restrict__ P = a.P[cur];
  uint32_t* __restrict__ Q = a.P[cur ^ 1];
  SlotCtl* sl = &a.ctl->slot[g % 3u];
  uint32_t* fb = a.FB[g & 1u];
  uint32_t* fp = a.FB[(g - 1u) & 1u];
  uint4* bc = a.BC[g & 1u];
  uint32_t* Cn = a.C[g & 1u];
  const uint32_t lane = lane_id();
  const uint32_t gw = gwarp(a);
  const uint32_t nw = nwarps(a);
  StepAcc acc;
  Hot hot{0u, vmax};
  if (RL && a.hot_k) {  // stage the previous step's frontier bits of the hottest positions
    for (uint32_t i = threadIdx.x; i < a.hot_k / 32u; i += blockDim.x) hot_sh[i] = __ldcg(fp + i);
    // rows_epilogue clears fp words as it goes: every CTA stages first
    cg::this_grid().sync();
    hot.k = a.hot_k;
  }
  if (a.world > 1) {
    // vertices of other ranks that changed in step k-1: this replica of x_k
    // still holds x_{k-2} for them; bring it up to x_{k-1} (their owners store
    // x_k over it if they change again -- atomicMax makes either order right)
    // and consume the word (the buffer is written again in step k+1)
    const uint32_t w0 = a.row_lo / 32u, w1 = a.row_hi / 32u;
    for (uint32_t wi = gw; wi < a.nwords_pad; wi += nw) {
      if (wi >= w0 && wi < w1) continue;  // own words: rows_epilogue consumes them
      const uint32_t word = __ldcg(fp + wi);
      if (!word) continue;
      const uint32_t v = wi * 32u + lane;
      if ((word >> lane) & 1u) atomicMax(Q + v, __ldcg(P + v));
      __syncwarp();
      if (lane == 0) fp[wi] = 0u;
    }
  }
  // many chunks per warp (R-MAT hubs): four in flight, and reads before the
  // contended atomics; few (config 2's connectors): one per warp, spread over
  // more warps, no extra round trip
  if (a.hcol) pull_heavy_slab<RL>(a, P, Q, fb, sh, bc, sl, Cn, acc, hot);
  else if (a.n_heavy > 4u * nw) pull_heavy<RL, kHeavyBatch, true>(a, P, Q, fb, sh, bc, sl, Cn, acc);
  else pull_heavy<RL, 1, false>(a, P, Q, fb, sh, bc, sl, Cn, acc);
  phase_mark(a, tk, 0);
  if (a.sdesc) {
    pull_sell<RL, 2, 4>(a, P, Q, fb, sh, fp, bc, sl, acc, hot);
  } else switch (a.ell_k) {
    case 1: pull_light<RL, 1, 8>(a, P, Q, fb, sh, fp, bc, sl, acc); break;
    case 2: pull_light<RL, 2, 8>(a, P, Q, fb, sh, fp, bc, sl, acc); break;
    case 4: pull_light<RL, 4, 4>(a, P, Q, fb, sh, fp, bc, sl, acc); break;
    default: pull_light<RL, 8, 4>(a, P, Q, fb, sh, fp, bc, sl, acc); break;
  }
  phase_mark(a, tk, 1);
  step_flags(a, acc, sl, sh, a.WL[g & 1u], a.wl_cap, a.BC[g & 1u]);
  phase_mark(a, tk, 2);
}

// ------------------------------------------------------------------ push
// Chunk descriptors of every big vertex in the words src[w] & bigm[w] (a
// frontier), written without per-vertex global atomics: each CTA counts the
// chunks of its contiguous word range (pass A), claims its slice with ONE
// atomicAdd, and writes the descriptors at the same positions in pass B,
// a warp per vertex at a time so hubs' thousands of chunks are written 32
// at once. Replaces per-CTA shared lists that overflowed on whole frontiers
// (config 3's F: the overflow sent its first push step through lane-by-lane
// expansion against one global counter, ~0.5 ms of a 1.4 ms step).
__device__ void chunk_words(const RunArgs& a, const uint32_t* src, uint4* bc, unsigned int* nchunk, BlockSh* sh) {
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  const uint32_t per = (a.nwords + a.nblk - 1u) / a.nblk;
  const uint32_t w0 = min(vblk(a) * per, a.nwords), w1 = min(w0 + per, a.nwords);
  auto chunks_of = [&](uint32_t m, uint32_t wi) {  // this lane's word: its big vertices' chunk count
    uint32_t nc = 0;
    while (m) {
      const uint32_t v = wi * 32u + (__ffs(m) - 1u);
      m &= m - 1u;
      nc += (__ldg(a.poff + v + 1) - __ldg(a.poff + v) + kChunk - 1u) / kChunk;
    }
    return nc;
  };
  // pass A: chunks per warp (each warp takes 32 consecutive words per round)
  uint32_t mine = 0;
  for (uint32_t base = w0 + wid * 32u; base < w1; base += nwb * 32u) {
    const uint32_t wi = base + lane;
    const uint32_t m = wi < w1 ? __ldcg(src + wi) & __ldcg(a.bigm + wi) : 0u;
    mine += chunks_of(m, wi);
  }
  mine = __reduce_add_sync(kFull, mine);
  __syncthreads();
  if (lane == 0) sh->wmin[wid] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {  // warps' offsets, then the CTA's slice of the list
    uint32_t tot = 0;
    for (uint32_t w = 0; w < nwb; ++w) {
      const uint32_t x = sh->wmin[w];
      sh->wmin[w] = tot;
      tot += x;
    }
    sh->wmin[32] = tot ? atomicAdd(nchunk, tot) & ~kChunkOver : 0u;
  }
  __syncthreads();
  uint32_t off = sh->wmin[32] + sh->wmin[wid];
  // pass B: the same words in the same order
  for (uint32_t base = w0 + wid * 32u; base < w1; base += nwb * 32u) {
    const uint32_t wi = base + lane;
    uint32_t m = wi < w1 ? __ldcg(src + wi) & __ldcg(a.bigm + wi) : 0u;
    const uint32_t nc = chunks_of(m, wi);
    const uint32_t incl = warp_incl_scan(nc);
    uint32_t o = off + incl - nc;
    off += __shfl_sync(kFull, incl, 31);
    for (uint32_t live = __ballot_sync(kFull, m != 0u); live; live = __ballot_sync(kFull, m != 0u)) {
      const uint32_t l = __ffs(live) - 1u;
      const uint32_t ml = __shfl_sync(kFull, m, l), ol = __shfl_sync(kFull, o, l), wl = __shfl_sync(kFull, wi, l);
      const uint32_t v = wl * 32u + (__ffs(ml) - 1u);
      const uint32_t b = __ldg(a.poff + v), e = __ldg(a.poff + v + 1);
      const uint32_t n = (e - b + kChunk - 1u) / kChunk;
      for (uint32_t c = lane; c < n; c += 32u)
        if (ol + c < a.chunk_cap) bc[ol + c] = make_uint4(v, b + c * kChunk, min(e, b + (c + 1u) * kChunk), 0u);
      if (lane == l) {
        m &= m - 1u;
        o += n;
      }
    }
  }
}

// Chunks of every big vertex of the frontier of step g-1, over this rank's
// push rows, replacing the list step g-1 built: sharded runs (local raises
// enlist nothing; other ranks raise most of the frontier) and steps whose
// big-vertex lists overflowed (enlist). Between steps, not inside push_step:
// barriers there keep the push step's loads from being scheduled early.
__device__ void rechunk_pass(const RunArgs& a, uint32_t g, BlockSh* sh, cg::grid_group& grid) {
  SlotCtl* plw = &a.ctl->slot[(g - 1u) % 3u];
  uint4* bpw = a.BC[(g - 1u) & 1u];
  const uint32_t* fp = a.FB[(g - 1u) & 1u];
  const uint32_t lane = lane_id(), gw = gwarp(a), nw = nwarps(a);
  grid.sync();  // every block has read the count before it is reset
  if (vblk(a) == 0 && threadIdx.x == 0) plw->nchunk = 0;
  grid.sync();
  chunk_words(a, fp, bpw, &plw->nchunk, sh);
  grid.sync();
}

template <bool RL>
__device__ void push_step(const RunArgs& a, uint32_t g, int cur, uint32_t nchunk, const SlotView& pv, BlockSh* sh,
                          unsigned long long tk) {
  SlotCtl* sl = &a.ctl->slot[g % 3u];
  PushCtx c;
  c.Pc = a.P[cur];
  c.Pn = a.P[cur ^ 1];
  c.fb = a.FB[g & 1u];
  c.sh = sh;
  c.bc = a.BC[g & 1u];
  c.nchunk = &sl->nchunk;
  c.Cn = a.C[g & 1u];
  c.ccnt = &sl->cand_cnt;
  // previous step's frontier edges: small frontiers are latency-bound (one
  // more round trip costs), large ones meet hub targets (atomics contend)
  c.contend = pv.fedges > (1ull << 20);
  uint32_t* fp = a.FB[(g - 1u) & 1u];
  const uint32_t* wlp = a.WL[(g - 1u) & 1u];
  const uint4* bp = a.BC[(g - 1u) & 1u];
  const uint32_t lane = lane_id();
  const uint32_t gw = swarp(a);
  const uint32_t nw = nwarps(a);
  StepAcc acc;
  const uint32_t wlc = pv.wl_count;
  const uint32_t wl_over = pv.wl_over;
  // big frontier vertices first: one warp per kChunk-edge chunk, each lane
  // raising kChunk/32 targets as one batch
  const uint32_t nch = min(nchunk & ~kChunkOver, a.chunk_cap);
  for (uint32_t k = gw; k < nch; k += nw) {
    const uint4 ch = bp[k];
    const uint32_t vv = cand_of<RL>(a, __ldca(c.Pc + ch.x), ch.x);
    uint32_t t[kChunk / 32], val[kChunk / 32];
#pragma unroll
    for (int r = 0; r < (int)(kChunk / 32); ++r) {
      const uint32_t i = ch.y + lane + 32u * r;
      t[r] = i < ch.z ? __ldg(a.pcol + i) : kNone;
      val[r] = vv;
    }
    raise_batch<RL>(a, c, t, val, acc);
  }
  phase_mark(a, tk, 0);
  // every frontier vertex: max-copy itself into the new buffer, and push its
  // edges unless it is big (chunks above). Frontier words come from the
  // previous step's word list (4 per warp iteration, interleaved over the
  // grid, so a contiguous wave of raised ids spreads over many warps), or from
  // a scan of the whole bitmap when that list overflowed. Lane i owns bit i of
  // each word; each word is cleared by the warp that consumes it.
  // sharded: the word lists only know this rank's raises; scan the replicated bitmap
  const bool scan = a.world > 1 || wl_over != 0u;
  // one group = four frontier words (lane i owns bit i of each)
  // up to 32 frontier vertices, one per lane (vx, kNone for none): their
  // loads in one round trip, their edges flattened over the warp 32 at a
  // time, so a vertex of degree d costs ceil(d/32) rounds, not d (a lane
  // walking its own vertex's edges one round trip each)
  auto sparse = [&](const uint32_t vx) {
    const bool on = vx != kNone;
    const uint32_t xv = on ? __ldca(c.Pc + vx) : 0u;
    const uint32_t bw1 = on ? __ldcg(a.bigm + (vx >> 5)) : 0u;
    const uint32_t b1 = on ? __ldg(a.poff + vx) : 0u;
    uint32_t e1 = on ? __ldg(a.poff + vx + 1) : 0u;
    uint32_t val1 = 0u;
    if (on) {
      atomicMax(c.Pn + vx, xv);  // bring x_{k-2} up to x_{k-1}
      val1 = cand_of<RL>(a, xv, vx);
      if ((bw1 >> (vx & 31u)) & 1u) e1 = b1;  // big: chunks push its edges
    }
    const uint32_t d1 = e1 - b1;
    if (__reduce_max_sync(kFull, d1) <= (uint32_t)kBatch) {  // low degrees (chains): each lane its own edges
      uint32_t t[kBatch], tv[kBatch];
#pragma unroll
      for (int k = 0; k < kBatch; ++k) {
        t[k] = (uint32_t)k < d1 ? __ldg(a.pcol + b1 + k) : kNone;
        tv[k] = val1;
      }
      raise_batch<RL>(a, c, t, tv, acc);
      return;
    }
    const uint32_t incl = warp_incl_scan(d1), excl = incl - d1;
    const uint32_t T = __shfl_sync(kFull, incl, 31);
    for (uint32_t e0 = 0; e0 < T; e0 += 32u * kBatch) {
      uint32_t t[kBatch], tv[kBatch];
#pragma unroll
      for (int k = 0; k < kBatch; ++k) {
        const uint32_t idx = e0 + 32u * k + lane;
        uint32_t l = 0;  // owner: the last lane whose edges start at or before idx
#pragma unroll
        for (uint32_t st = 16; st > 0; st >>= 1)
          if (__shfl_sync(kFull, excl, l + st) <= idx) l += st;
        const uint32_t lb = __shfl_sync(kFull, b1, l), lx = __shfl_sync(kFull, excl, l);
        tv[k] = __shfl_sync(kFull, val1, l);
        t[k] = idx < T ? __ldg(a.pcol + lb + (idx - lx)) : kNone;
      }
      raise_batch<RL>(a, c, t, tv, acc);
    }
  };
  auto group = [&](const uint32_t (&wi)[kBatch], const uint32_t (&wd)[kBatch]) {
    if (!(wd[0] | wd[1] | wd[2] | wd[3])) return;
    __syncwarp();
    {
      uint32_t mw = 0, mi = kNone;  // lane r < 4 clears word r (select chain, no local memory)
#pragma unroll
      for (int r = 0; r < kBatch; ++r)
        if (lane == (uint32_t)r) {
          mw = wd[r];
          mi = wi[r];
        }
      if (mw) fp[mi] = 0u;
    }
    uint32_t cnt[kBatch], pre[kBatch + 1];
    pre[0] = 0;
#pragma unroll
    for (int r = 0; r < kBatch; ++r) {
      cnt[r] = __popc(wd[r]);
      pre[r + 1] = pre[r] + cnt[r];
    }
    if (pre[kBatch] <= 32u) {  // sparse group: its vertices compacted one per lane
      uint32_t vx = kNone;
#pragma unroll
      for (int r = 0; r < kBatch; ++r)
        if (lane >= pre[r] && lane < pre[r + 1]) vx = wi[r] * 32u + __fns(wd[r], 0u, (int)(lane - pre[r] + 1u));
      sparse(vx);
      return;
    }
    uint32_t v[kBatch], b[kBatch], e[kBatch], val[kBatch], xu[kBatch], bwv[kBatch];
    // every load of the four vertices first, in one round trip: an atomic on
    // Pn between them would serialise the batch (Pn may alias Pc for the
    // compiler), which on config 5's chain cost four DRAM latencies a step
#pragma unroll
    for (int r = 0; r < kBatch; ++r) {
      v[r] = (wd[r] >> lane) & 1u ? wi[r] * 32u + lane : kNone;
      const bool on = v[r] != kNone;
      xu[r] = on ? __ldca(c.Pc + v[r]) : 0u;
      bwv[r] = on ? __ldcg(a.bigm + (v[r] >> 5)) : 0u;
      b[r] = on ? __ldg(a.poff + v[r]) : 0u;
      e[r] = on ? __ldg(a.poff + v[r] + 1) : 0u;
    }
#pragma unroll
    for (int r = 0; r < kBatch; ++r) {
      val[r] = 0u;
      if (v[r] != kNone) {
        atomicMax(c.Pn + v[r], xu[r]);  // bring x_{k-2} up to x_{k-1}
        val[r] = cand_of<RL>(a, xu[r], v[r]);
        if ((bwv[r] >> (v[r] & 31u)) & 1u) e[r] = b[r];  // big: chunks push its edges
      }
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
      raise_batch<RL>(a, c, t, val, acc);
    }
  };
  // 32 frontier words, one per lane (myw = 0: none). Sparse windows (<= 64
  // vertices, small frontiers) are compacted 32 vertices per round; dense ones
  // go four words at a time, four vertices per lane.
  auto window = [&](const uint32_t myi, const uint32_t myw) {
    const uint32_t cw = __popc(myw), incl = warp_incl_scan(cw), excl = incl - cw;
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    if (total == 0u) return;
    if (total <= 64u) {
      if (myw) fp[myi] = 0u;
      for (uint32_t c0 = 0; c0 < total; c0 += 32u) {
        const uint32_t i = c0 + lane;
        uint32_t l = 0;  // the lane whose word holds vertex i
#pragma unroll
        for (uint32_t st = 16; st > 0; st >>= 1)
          if (__shfl_sync(kFull, excl, l + st) <= i) l += st;
        const uint32_t w = __shfl_sync(kFull, myw, l), wi = __shfl_sync(kFull, myi, l);
        const uint32_t k = i - __shfl_sync(kFull, excl, l);
        sparse(i < total ? wi * 32u + __fns(w, 0u, (int)(k + 1u)) : kNone);
      }
      return;
    }
    for (uint32_t live = __ballot_sync(kFull, myw != 0u); live;) {
      uint32_t wi[kBatch], wd[kBatch];
#pragma unroll
      for (int r = 0; r < kBatch; ++r) {
        const uint32_t l = live ? __ffs(live) - 1u : 0u;
        const uint32_t xi = __shfl_sync(kFull, myi, l), xw = __shfl_sync(kFull, myw, l);
        wi[r] = live ? xi : kNone;
        wd[r] = live ? xw : 0u;
        live &= live - 1u;
      }
      group(wi, wd);
    }
  };
  // windows: 32 consecutive words of the bitmap, or 4 entries of the list
  // (list entries are few or come in contiguous waves of dense words: spread
  // them over many warps; config 2 lost 14 % with 32-entry windows)
  const uint32_t nwin = scan ? (a.nwords + 31u) / 32u : (wlc + 3u) / 4u;
  for (uint32_t it = gw; it < nwin; it += nw) {
    const uint32_t e = scan ? it * 32u + lane : it * 4u + lane;
    const uint32_t myi = scan ? (e < a.nwords ? e : kNone)
                              : (lane < 4u && e < wlc ? __ldcg(wlp + e) : kNone);
    const uint32_t myw = myi != kNone ? __ldcg(fp + myi) : 0u;
    window(myi, myw);
  }
  phase_mark(a, tk, 1);
  step_flags(a, acc, sl, sh, a.WL[g & 1u], a.wl_cap, a.BC[g & 1u]);
  phase_mark(a, tk, 2);
}

// ------------------------------------------------------- iteration passes
// Dense pass over the fixpoint vector: iteration hash, full self-witness (for
// early_exit = false, map_engine.cpp:108-112) and the "used" bitmap of demote
// (map_engine.cpp:124-126).
template <bool RL>
__device__ void finish_pass(const RunArgs& a, int cur, uint64_t t, bool mark_used, BlockSh* sh) {
  const uint32_t* P = a.P[cur];
  RunCtl* ctl = a.ctl;
  const uint32_t lane = lane_id();
  const uint32_t gw = gwarp(a);
  const uint32_t nw = nwarps(a);
  unsigned long long h = 0;
  uint32_t fw = kNone;
  for (uint32_t base = gw * 32u; base < a.n; base += nw * 32u) {
    const uint32_t v = base + lane;
    uint32_t code = 0;
    if (v < a.n) {
      const uint32_t x = __ldcg(P + v);
      const uint32_t id = oid<RL>(a, v);
      code = x & kCode;
      h += cyc_splitmix64(((unsigned long long)id << 32) | code);
      if ((x & kFlag) && code == id + 1u) fw = min(fw, id);
    }
    if (mark_used) {
      const uint32_t peers = __match_any_sync(kFull, code);
      if (code && (__ffs(peers) - 1) == (int)lane) {
        // the value is a vertex id + 1; its accepting bit lives at its position
        const uint32_t u = RL ? __ldg(a.perm + (code - 1u)) : code - 1u, bit = 1u << (u & 31u);
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
  if (vblk(a) == 0 && threadIdx.x == 0) {
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
  const uint32_t stride = a.nblk * blockDim.x;
  for (uint32_t i = vblk(a) * blockDim.x + threadIdx.x; i < a.nwords; i += stride) {
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
// accepting bit; the initial frontier is the accepting set itself (every
// accepting u offers cand = u+1), FB[(g+1)&1] cleared.
template <bool RL>
__device__ void reset_pass(const RunArgs& a, uint32_t g, uint64_t t, BlockSh* sh) {
  uint32_t* fb = a.FB[g & 1u];
  uint32_t* fz = a.FB[(g + 1u) & 1u];
  SlotCtl* sl = &a.ctl->slot[g % 3u];
  uint4* bc = a.BC[g & 1u];
  const uint32_t lane = lane_id();
  const uint32_t gw = gwarp(a);
  const uint32_t nw = nwarps(a);
  unsigned long long fe = 0;
  uint32_t vm = 0;  // max id+1 over F: no map value of this fixpoint can exceed it
  // 32 words (1024 vertices) per warp iteration
  for (uint32_t s = gw; s * 32u < a.nwords_pad; s += nw) {
    const uint32_t wi = s * 32u + lane;
    const uint32_t f = wi < a.nwords ? __ldcg(a.F + wi) : 0u;
    if (wi < a.nwords_pad) {
      fb[wi] = f;
      fz[wi] = 0u;
      if (f) note_word(sh, wi);
    }
    // eight words per round: their degree / id loads in flight together
    // (one load round trip per word serialised ~120 of them per warp)
    for (uint32_t j0 = 0; j0 < 32u; j0 += 8u) {
      uint32_t dv[8], iv[8];
#pragma unroll
      for (uint32_t q = 0; q < 8u; ++q) {
        const uint32_t fj = __shfl_sync(kFull, f, j0 + q);
        const uint32_t v = (s * 32u + j0 + q) * 32u + lane;
        const bool accv = v < a.n && ((fj >> lane) & 1u);
        if (v < a.n) {
          const uint32_t val = accv ? kFlag : 0u;
          a.P[0][v] = val;
          a.P[1][v] = val;
        }
        dv[q] = accv ? __ldg(a.poff + v + 1) - __ldg(a.poff + v) : 0u;
        iv[q] = accv ? oid<RL>(a, v) + 1u : 0u;
      }
#pragma unroll
      for (uint32_t q = 0; q < 8u; ++q) {
        fe += dv[q];
        vm = max(vm, iv[q]);
      }
    }
  }
  // chunks of F's big vertices for the first push step (single device;
  // sharded push steps re-chunk their rows every step)
  if (a.world == 1) chunk_words(a, a.F, bc, &sl->nchunk, sh);
  fe = block_sum(fe, sh);
  vm = ~block_min(~vm, sh);
  if (threadIdx.x == 0 && fe) atomicAdd(&sl->fedges, fe);
  if (threadIdx.x == 0 && vm) atomicMax(&a.ctl->it_vmax[t & 1u], vm);
  if (vblk(a) == 0 && threadIdx.x == 0) a.ctl->it_vmax[(t + 1u) & 1u] = 0u;  // the next fixpoint's
  wl_flush(sh, sl, a.WL[g & 1u], a.wl_cap);
}

__device__ __forceinline__ void reset_slot(RunCtl* c, uint32_t s) {
  SlotCtl& sl = c->slot[s];
  sl.fedges = 0;
  sl.nraised = 0;
  sl.changed = 0;
  sl.nchunk = 0;
  sl.cand_cnt = 0;
  sl.wit = kNone;
  sl.wl_count = 0;
  sl.wl_over = 0;
  sl.light_next = 0;
  sl.heavy_next = 0;
}

// ------------------------------------------------------- sharded exchange
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Every rank's writes so far (local and into peers) visible to every rank.
// Emulated ranks share the grid, so its barrier is the cross-rank barrier;
// real ranks also meet at system-scope counters in each rank's memory (the
// lead spins with a 30 s timeout that traps instead of hanging the GPU).
__device__ void rank_sync(const RunArgs& a, cg::grid_group& grid, unsigned long long& bars) {
  __threadfence_system();
  grid.sync();
  if (a.world > 1 && !a.emulated) {
    if (vblk(a) == 0 && threadIdx.x == 0) {
      for (int p = 0; p < a.world; ++p) atomicAdd_system(a.peerBar[p], 1ull);
      ++bars;
      const unsigned long long target = bars * (unsigned long long)a.world, t0 = gtimer();
      while (ld_acquire_sys(a.bar) < target)
        if (gtimer() - t0 > 30000000000ull) __trap();
    }
    grid.sync();
  }
}

__device__ __forceinline__ ShardRec ld_rec(const ShardRec* r) {
  ShardRec x;
  x.fedges = __ldcg(&r->fedges);
  x.nraised = __ldcg(&r->nraised);
  x.changed = __ldcg(&r->changed);
  x.wit = __ldcg(&r->wit);
  x.pad = 0;
  return x;
}

// End of a sharded step (or setup, publish = false): this rank's record goes
// to every rank, the rows it changed (its frontier words of tag g) are stored
// into every peer's buffers, then the records of all ranks are reduced.
__device__ ShardRec exchange_step(const RunArgs& a, cg::grid_group& grid, uint32_t g, int cur_new,
                                  const SlotCtl* sl, uint32_t wit, bool publish, unsigned long long& bars) {
  const uint32_t par = g & 1u;
  if (vblk(a) == 0 && threadIdx.x == 0) {
    ShardRec r;
    r.fedges = __ldcg(&sl->fedges);
    r.nraised = __ldcg(&sl->nraised);
    r.changed = __ldcg(&sl->changed);
    r.wit = wit;
    r.pad = 0;
    for (int p = 0; p < a.world; ++p) a.peerRec[p][par * kMaxWorld + a.rank] = r;
  }
  if (publish) {
    const uint32_t lane = lane_id(), gw = gwarp(a), nw = nwarps(a);
    const uint32_t* fbw = a.FB[par];
    const uint32_t* Pn = a.P[cur_new];
    for (uint32_t wi = a.row_lo / 32u + gw; wi < a.row_hi / 32u; wi += nw) {
      const uint32_t word = __ldcg(fbw + wi);
      if (!word) continue;
      const uint32_t v = wi * 32u + lane;
      const bool on = (word >> lane) & 1u;
      const uint32_t x = on ? __ldcg(Pn + v) : 0u;
      for (int p = 0; p < a.world; ++p) {
        if (p == a.rank) continue;
        if (on) a.peerP[p][cur_new][v] = x;
        if (lane == 0) a.peerFB[p][par][wi] = word;
      }
    }
  }
  rank_sync(a, grid, bars);
  ShardRec t;
  t.fedges = 0;
  t.nraised = 0;
  t.changed = 0;
  t.wit = kNone;
  t.pad = 0;
  for (int p = 0; p < a.world; ++p) {
    const ShardRec r = ld_rec(a.rec + par * kMaxWorld + p);
    t.fedges += r.fedges;
    t.nraised += r.nraised;
    t.changed |= r.changed;
    t.wit = min(t.wit, r.wit);
  }
  return t;
}

template <bool RL, bool SH>
__device__ __forceinline__ void map_run_body(const RunArgs& a) {
  __shared__ BlockSh sh;
  __shared__ SlotView spv;  // the last finished step's counters (ld_slot)
  // run statistics live in shared memory of block 0 (kept out of registers)
  __shared__ unsigned long long stat[kResRaised + 1];
  cg::grid_group grid = cg::this_grid();
  RunCtl* ctl = a.ctl;
  uint32_t g = 1;
  int cur = 0;
  int cycle = 0;
  uint32_t witness = kNone;
  const bool lead = vblk(a) == 0 && threadIdx.x == 0;
  if (lead)
    for (int k = 0; k <= kResRaised; ++k) stat[k] = 0;
  if (threadIdx.x == 0) {
    sh.wl_n = 0;
    sh.big_n = 0;
  }
  __syncthreads();
#define CYC_STAT(k, v) \
  do {                 \
    if (lead) stat[k] += (v); \
  } while (0)

  // initial F count and first fixpoint setup (tag g)
  demote_pass(a, nullptr, &ctl->it_fsize[0], &sh);
  if (lead) reset_slot(ctl, (g + 1u) % 3u);
  reset_pass<RL>(a, g, 0, &sh);
  grid.sync();
  unsigned long long bars = a.bar_base;
  // sharded: global push degree of F (each rank counts its own push rows)
  unsigned long long g_fe = 0, g_nr = 0;
  if (SH && a.world > 1) g_fe = exchange_step(a, grid, g, 0, &ctl->slot[g % 3u], kNone, false, bars).fedges;
  uint64_t t = 0;
  uint32_t vmax = __ldcg(&ctl->it_vmax[0]);
  bool truncated = false;
  if (__ldca(&ctl->it_fsize[0]) != 0) {
    for (;;) {
      unsigned long long steps = 0;
      bool prev_push = true;  // the previous tag's fedges is exact (push or setup)
      if (threadIdx.x == 0) spv = ld_slot(&ctl->slot[g % 3u]);  // the setup's counters
      __syncthreads();
      for (;;) {
        ++g;
        ++steps;
        const uint32_t slot = g % 3u, pslot = (g - 1u) % 3u;
        if (lead) reset_slot(ctl, (g + 1u) % 3u);
        int mode = a.mode;
        // the previous step's (global) frontier size
        const bool xch = SH && a.world > 1;  // records come from the exchange
        const unsigned long long p_fe = xch ? g_fe : spv.fedges;
        const unsigned long long p_nr = xch ? g_nr : spv.nraised;
        unsigned int p_nchunk = spv.nchunk;
        if (mode != kModePull && mode != kModePush) {
          unsigned long long est;
          if (prev_push) {
            est = p_fe;
          } else {  // pull steps count big-vertex degrees exactly, the rest by average
            est = p_fe + (a.n ? p_nr * a.m / a.n : 0);
          }
          mode = (est * a.alpha < a.m) ? kModePush : kModePull;
        }
        // trace slot of this step (every block derives the same index from the tag)
        const unsigned long long tkk = (unsigned long long)(g - 2u);
        if (a.trace && lead && tkk < a.trace_cap) a.trace[64u * tkk + 3u] = gtimer();
        if (mode == kModePush) {
          if (lead) {
            stat[kResEdges] += p_fe;
            stat[kResRows] += p_nr;
            stat[kResBytes] += 8ull * p_fe + 12ull * p_nr;
            stat[kResPushSteps] += 1;
          }
          // every sharded rank re-chunks (ranks emulated in one grid stay in step)
          if (xch || (p_nchunk & kChunkOver)) {
            rechunk_pass(a, g, &sh, grid);
            p_nchunk = __ldcg(&ctl->slot[pslot].nchunk);
          }
          push_step<RL>(a, g, cur, p_nchunk, spv, &sh, a.trace ? tkk : ~0ull);
        } else {
          CYC_STAT(kResEdges, a.m);
          CYC_STAT(kResRows, a.n);
          CYC_STAT(kResBytes, 8ull * a.m + 12ull * a.n + 4ull);
          CYC_STAT(kResPullSteps, 1);
          pull_step<RL>(a, g, cur, vmax, &sh, a.trace ? tkk : ~0ull);
        }
        grid.sync();
        cur ^= 1;
        prev_push = mode == kModePush;
        const SlotCtl* sl = &ctl->slot[slot];
        if (threadIdx.x == 0) spv = ld_slot(sl);  // one round trip for the block; read from shared below
        __syncthreads();
        uint32_t changed = spv.changed;
        uint32_t w = spv.wit;
        const uint32_t nc = spv.cand_cnt;
        if (lead && a.trace && tkk < a.trace_cap) {
          unsigned long long* tr = a.trace + 64u * tkk;
          tr[0] = ((unsigned long long)mode << 60) |
                  ((unsigned long long)__ldca(&ctl->slot[pslot].nchunk) << 24) | (steps & 0xFFFFFFull);
          tr[1] = mode == kModePush ? __ldca(&ctl->slot[pslot].fedges) : a.m;
          tr[2] = __ldca(&sl->nraised);
          tr[7] = gtimer();
        }
        if (nc && a.early_exit) {
          const uint32_t* Cn = a.C[g & 1u];
          const uint32_t* Pn = a.P[cur];
          uint32_t mine = kNone;
          if (nc > a.cand_cap) {  // list overflowed: every position of the new buffer (rare)
            for (uint32_t v = threadIdx.x; v < a.n; v += blockDim.x) {
              const uint32_t x = __ldcg(Pn + v);
              if (x & kFlag) {
                const uint32_t id = oid<RL>(a, v);
                if ((x & kCode) == id + 1u) mine = min(mine, id);
              }
            }
          }
          for (uint32_t i = threadIdx.x; i < min(nc, a.cand_cap); i += blockDim.x) {
            const uint32_t c = __ldcg(Cn + i);
            const uint32_t id = oid<RL>(a, c);
            if ((__ldcg(Pn + c) & kCode) == id + 1u) mine = min(mine, id);
          }
          w = min(w, block_min(mine, &sh));
        }
        if (SH && a.world > 1) {  // every rank gets the others' changed rows and the global record
          const ShardRec gr = exchange_step(a, grid, g, cur, sl, w, true, bars);
          changed = gr.changed;
          w = gr.wit;
          g_fe = gr.fedges;
          g_nr = gr.nraised;
          CYC_STAT(kResRaised, g_nr);  // rows stored into every peer this step
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
      finish_pass<RL>(a, cur, t, !cycle, &sh);
      grid.sync();
      if (!a.early_exit) {
        const uint32_t fw = __ldca(&ctl->it_finwit[t & 1u]);
        if (fw != kNone) {
          cycle = 1;
          witness = fw;
        }
      }
      if (lead && t < a.cap) {
        if (a.iter_hash) a.iter_hash[t] = __ldca(&ctl->it_hash[t & 1u]);
        if (a.iter_steps) a.iter_steps[t] = steps;
      }
      CYC_STAT(kResIterations, 1);
      CYC_STAT(kResKernelCalls, steps);
      if (cycle) break;
      if (a.max_iterations && t + 1 >= a.max_iterations) break;
      demote_pass(a, &ctl->it_dcount[t & 1u], &ctl->it_fsize[(t + 1u) & 1u], &sh);
      grid.sync();
      const uint32_t dc = __ldca(&ctl->it_dcount[t & 1u]);
      CYC_STAT(kResDemoted, dc);
      if (dc == 0) break;                                      // D empty: no cycle
      ++t;
      if (__ldca(&ctl->it_fsize[t & 1u]) == 0) break;          // F' empty: no cycle
      ++g;
      if (lead) reset_slot(ctl, (g + 1u) % 3u);
      reset_pass<RL>(a, g, t, &sh);
      cur = 0;
      grid.sync();
      if (SH && a.world > 1) g_fe = exchange_step(a, grid, g, 0, &ctl->slot[g % 3u], kNone, false, bars).fedges;
      vmax = __ldcg(&ctl->it_vmax[t & 1u]);
    }
  }
  if (lead) {
    stat[kResCycle] = cycle;
    stat[kResWitness] = witness;
    stat[kResCur] = (unsigned long long)cur;
    stat[kResTag] = g;
    stat[kResBars] = bars;
    for (int k = 0; k <= kResRaised; ++k) ctl->res[k] = stat[k];
  }
#undef CYC_STAT
}

template <bool RL, bool SH>
__global__ void __launch_bounds__(run_threads<RL>(), 1) k_map_run(RunArgs a) {
  map_run_body<RL, SH>(a);
}

// Tests on one GPU: every rank of a sharded run in ONE cooperative grid (rank
// r = blocks [r*nblk, (r+1)*nblk)), each with its own arguments; the grid
// barrier doubles as the cross-rank barrier (B200_PROFILING.md: ranks that
// wait on one another must not be separate launches on one GPU).
template <bool RL>
__global__ void __launch_bounds__(run_threads<RL>(), 1) k_map_run_emul(const RunArgs* __restrict__ ranks, int world) {
  map_run_body<RL, true>(ranks[blockIdx.x / (gridDim.x / (uint32_t)world)]);
}

__global__ void k_big_mask(uint32_t n, const uint32_t* __restrict__ poff, uint32_t* __restrict__ bigm) {
  const uint32_t lane = lane_id();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t nwords = (n + 31u) / 32u;
  for (uint32_t wi = gw; wi < nwords; wi += nw) {
    const uint32_t v = wi * 32u + lane;
    const bool big = v < n && __ldg(poff + v + 1) - __ldg(poff + v) > kBigDeg;
    const uint32_t word = __ballot_sync(kFull, big);
    if (lane == 0) bigm[wi] = word;
  }
}

__global__ void k_strip(const uint32_t* __restrict__ P, uint32_t n, uint32_t* __restrict__ out) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) out[v] = P[v] & kCode;
}

// storage positions back to vertex ids: out[orig[p]] = code(P[p])
__global__ void k_strip_perm(const uint32_t* __restrict__ P, const uint32_t* __restrict__ orig, uint32_t n,
                             uint32_t* __restrict__ out) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) out[__ldg(orig + p)] = P[p] & kCode;
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

// Sharded dense step over rows [lo, hi). Rows longer than `heavy` start from
// x[v] here and are finished by k_step_range_chunks (one warp per heavy
// chunk, atomicMax into out) and k_step_range_heavy (their flags).
__device__ __forceinline__ uint32_t cand_of(uint32_t u, const uint32_t* __restrict__ x,
                                            const uint32_t* __restrict__ accw) {
  uint32_t c = x[u];
  if (((accw[u >> 5] >> (u & 31u)) & 1u) && u + 1u > c) c = u + 1u;
  return c;
}

// Range (pull) kernels skip when the fixpoint is decided, a sparse step is
// blocked, or (first_only: the sparse protocol) a push step takes this step.
__device__ __forceinline__ bool range_skip(const long long* st, int first_only) {
  return st && (st[0] | st[4] | (first_only ? st[1] : 0));
}

__device__ __forceinline__ void shard_flags(bool ch, uint32_t wit, unsigned long long* rec) {
  wit = __reduce_min_sync(__activemask(), wit);
  if (__any_sync(__activemask(), ch) && lane_id() == 0) atomicMax(rec, 1ull);
  if (wit != kNone && lane_id() == 0) atomicMax(rec + 1, (unsigned long long)(kNone - wit));
}

__global__ void k_step_range(uint32_t lo, uint32_t hi, uint32_t heavy, const uint32_t* __restrict__ goff,
                             const uint32_t* __restrict__ gcol, const uint32_t* __restrict__ x,
                             const uint32_t* __restrict__ accw, uint32_t* __restrict__ out,
                             unsigned long long* __restrict__ rec, const long long* __restrict__ state,
                             int first_only) {
  if (range_skip(state, first_only)) return;  // decided, blocked, or a push step follows
  const uint32_t stride = gridDim.x * blockDim.x;
  bool ch = false;
  uint32_t wit = kNone;
  for (uint32_t v = lo + blockIdx.x * blockDim.x + threadIdx.x; v < hi; v += stride) {
    const uint32_t b = goff[v], e = goff[v + 1];
    uint32_t best = x[v];
    if (e - b > heavy) {
      out[v - lo] = best;
      continue;
    }
    for (uint32_t i = b; i < e; ++i) best = max(best, cand_of(gcol[i], x, accw));
    out[v - lo] = best;
    ch |= best != x[v];
    if (best == v + 1u && ((accw[v >> 5] >> (v & 31u)) & 1u)) wit = min(wit, v);
  }
  shard_flags(ch, wit, rec);
}

// Same step reading each row's first K columns from the column-major HYB slab
// (coalesced across lanes; sentinel entries >= n are NIL); rows flagged in
// ovf continue from column K in the CSR, heavy ones are left to the chunks.
template <int K>
__global__ void k_step_range_ell(uint32_t lo, uint32_t hi, uint32_t n, uint32_t np, uint32_t heavy,
                                 const uint32_t* __restrict__ ell, const uint32_t* __restrict__ ovf,
                                 const uint32_t* __restrict__ goff, const uint32_t* __restrict__ gcol,
                                 const uint32_t* __restrict__ x, const uint32_t* __restrict__ accw,
                                 uint32_t* __restrict__ out, unsigned long long* __restrict__ rec,
                                 const long long* __restrict__ state, int first_only) {
  if (range_skip(state, first_only)) return;
  const uint32_t stride = gridDim.x * blockDim.x;
  bool ch = false;
  uint32_t wit = kNone;
  for (uint32_t v = lo + blockIdx.x * blockDim.x + threadIdx.x; v < hi; v += stride) {
    const uint32_t own = x[v];
    uint32_t u[K];
#pragma unroll
    for (int j = 0; j < K; ++j) u[j] = __ldg(ell + (size_t)j * np + v);
    uint32_t best = own;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (u[j] < n) best = max(best, cand_of(u[j], x, accw));
    if ((__ldg(ovf + (v >> 5)) >> (v & 31u)) & 1u) {
      const uint32_t b = goff[v], e = goff[v + 1];
      if (e - b > heavy) {
        out[v - lo] = own;
        continue;
      }
      for (uint32_t i = b + K; i < e; ++i) best = max(best, cand_of(gcol[i], x, accw));
    }
    out[v - lo] = best;
    ch |= best != own;
    if (best == v + 1u && ((accw[v >> 5] >> (v & 31u)) & 1u)) wit = min(wit, v);
  }
  shard_flags(ch, wit, rec);
}

__global__ void k_step_range_chunks(const uint4* __restrict__ chunks, uint32_t nch, uint32_t lo, uint32_t hi,
                                    const uint32_t* __restrict__ gcol, const uint32_t* __restrict__ x,
                                    const uint32_t* __restrict__ accw, uint32_t* __restrict__ out,
                                    const long long* __restrict__ state, int first_only) {
  if (range_skip(state, first_only)) return;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t k = gw; k < nch; k += nw) {
    const uint4 ch = chunks[k];
    if (ch.x < lo || ch.x >= hi) continue;
    uint32_t best = 0;
    for (uint32_t i = ch.y + lane; i < ch.z; i += 32u) best = max(best, cand_of(gcol[i], x, accw));
    best = __reduce_max_sync(kFull, best);
    if (lane == 0 && best > x[ch.x]) atomicMax(out + (ch.x - lo), best);
  }
}

__global__ void k_step_range_heavy(const uint4* __restrict__ chunks, uint32_t nch, uint32_t lo, uint32_t hi,
                                   const uint32_t* __restrict__ goff, const uint32_t* __restrict__ x,
                                   const uint32_t* __restrict__ accw, const uint32_t* __restrict__ out,
                                   unsigned long long* __restrict__ rec, const long long* __restrict__ state,
                                   int first_only) {
  if (range_skip(state, first_only)) return;
  bool chg = false;
  uint32_t wit = kNone;
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nch; k += gridDim.x * blockDim.x) {
    const uint4 ch = chunks[k];
    const uint32_t v = ch.x;
    if (v < lo || v >= hi || ch.y != goff[v]) continue;  // first chunk of an in-range row
    const uint32_t best = out[v - lo];
    chg |= best != x[v];
    if (best == v + 1u && ((accw[v >> 5] >> (v & 31u)) & 1u)) wit = min(wit, v);
  }
  shard_flags(chg, wit, rec);
}

__global__ void k_shard_post(const long long* __restrict__ rec, long long* state,
                             const uint32_t* __restrict__ x_pad, const uint32_t* __restrict__ bounds,
                             int world, uint32_t maxrows, uint32_t* __restrict__ x) {
  const uint64_t total = (uint64_t)world * maxrows;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = (uint32_t)(e / maxrows), i = (uint32_t)(e % maxrows);
    const uint32_t lo = bounds[r];
    if (lo + i < bounds[r + 1]) x[lo + i] = x_pad[e];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && !state[0]) {
    const uint32_t wit = kNone - (uint32_t)rec[1];
    state[1] += 1;
    if ((state[3] && wit != kNone) || !rec[0]) {
      state[0] = 1;
      state[2] = wit;
    }
  }
}

// Sparse exchange: this rank's changed rows as (v, value) after the step;
// sp[0] = {count, 0}, entries sp[1..cap]; a count above cap marks overflow.
// After a pull step (or list_mode off) the slice is scanned; after a push step
// the raised list is read (and its bits cleared), and the step record comes
// from it: changed = any raised, witness = min raised t with t accepting and
// out[t] = t + 1 (early exit only: a self-valued row that is not raised now
// would have stopped the fixpoint at an earlier step).
__global__ void k_shard_collect(uint32_t lo, uint32_t hi, const uint32_t* __restrict__ x,
                                const uint32_t* __restrict__ out, uint32_t cap, uint2* sp,
                                const long long* __restrict__ state, int list_mode,
                                const uint32_t* __restrict__ rlist, const uint32_t* __restrict__ rcnt,
                                uint32_t* rbits, const uint32_t* __restrict__ accw, unsigned long long* rec) {
  if (state[0] | state[4]) return;
  const uint32_t stride = gridDim.x * blockDim.x;
  if (list_mode && state[1] != 0) {
    const uint32_t k = *rcnt;
    bool chg = false;
    uint32_t wit = kNone;
    for (uint32_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; i0 < k; i0 += stride) {
      const uint32_t i = i0 + lane_id();
      const bool in = i < k;
      const uint32_t t = in ? rlist[i] : 0u;  // local row index
      const uint32_t v = lo + t, val = in ? out[t] : 0u;
      if (in) {
        atomicAnd(rbits + (t >> 5), ~(1u << (t & 31u)));
        chg = true;
        if (val == v + 1u && ((accw[v >> 5] >> (v & 31u)) & 1u)) wit = min(wit, v);
      }
      const uint32_t bal = __ballot_sync(kFull, in);
      uint32_t base = 0;
      if (lane_id() == 0) base = atomicAdd(&sp[0].x, (uint32_t)__popc(bal));
      base = __shfl_sync(kFull, base, 0);
      const uint32_t idx = base + __popc(bal & lanemask_lt());
      if (in && idx < cap) sp[1 + idx] = make_uint2(v, val);
    }
    shard_flags(chg, wit, rec);
    return;
  }
  for (uint32_t v0 = lo + ((blockIdx.x * blockDim.x + threadIdx.x) & ~31u); v0 < hi; v0 += stride) {
    const uint32_t v = v0 + lane_id();
    const bool ch = v < hi && out[v - lo] != x[v];
    const uint32_t bal = __ballot_sync(kFull, ch);
    if (!bal) continue;
    uint32_t base = 0;
    if (lane_id() == 0) base = atomicAdd(&sp[0].x, (uint32_t)__popc(bal));
    base = __shfl_sync(kFull, base, 0);
    const uint32_t idx = base + __popc(bal & lanemask_lt());
    if (ch && idx < cap) sp[1 + idx] = make_uint2(v, out[v - lo]);
  }
}

// Sparse protocol, steps after the first: push from every rank's changes of
// the previous step (sp_all, applied to x already) along the snapshot rows,
// restricted to this rank's targets [lo, hi) (rows are sorted: two binary
// searches per source). out holds x's slice; raised targets are listed once.
__device__ __forceinline__ uint32_t lbound(const uint32_t* p, uint32_t len, uint32_t x) {
  uint32_t lo = 0, hi = len;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (p[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_shard_push(const uint2* __restrict__ sp_all, int world, uint32_t cap,
                             const uint32_t* __restrict__ soff, const uint32_t* __restrict__ scol, uint32_t lo,
                             uint32_t hi, const uint32_t* __restrict__ accw, uint32_t* out, uint32_t* rbits,
                             uint32_t* rlist, uint32_t* rcnt, const long long* __restrict__ state) {
  if (state[0] | state[4] | (state[1] == 0)) return;
  const uint32_t lane = lane_id();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const uint64_t total = (uint64_t)world * cap;
  for (uint64_t e = gw; e < total; e += nw) {
    const uint32_t r = (uint32_t)(e / cap), i = (uint32_t)(e % cap);
    const uint2* b = sp_all + (size_t)r * (cap + 1);
    if (i >= b[0].x) continue;
    const uint2 pr = b[1 + i];
    const uint32_t u = pr.x;
    const uint32_t cu = ((accw[u >> 5] >> (u & 31u)) & 1u) ? max(pr.y, u + 1u) : pr.y;
    const uint32_t rb = soff[u], re = soff[u + 1];
    const uint32_t s0 = rb + lbound(scol + rb, re - rb, lo), s1 = rb + lbound(scol + rb, re - rb, hi);
    for (uint32_t k = s0 + lane; k < s1; k += 32u) {
      const uint32_t t = scol[k] - lo;
      if (cu > out[t] && atomicMax(out + t, cu) < cu) {
        const uint32_t m = 1u << (t & 31u);
        if (!(atomicOr(rbits + (t >> 5), m) & m)) rlist[atomicAdd(rcnt, 1u)] = t;
      }
    }
  }
}

// After the all-gather of every rank's sparse buffer (sp_all: world x (cap+1))
// and the MAX all-reduce of rec: apply all changes (idempotent) and advance
// the state, unless some rank overflowed — then block the batch (state[4])
// and keep rec in state[6..7] for the host's dense completion of this step.
__global__ void k_shard_post_sparse(const long long* __restrict__ rec, long long* state,
                                    const uint2* __restrict__ sp_all, int world, uint32_t cap,
                                    uint32_t* __restrict__ x) {
  uint32_t maxc = 0;
  for (int r = 0; r < world; ++r) maxc = max(maxc, sp_all[(size_t)r * (cap + 1)].x);
  const bool over = maxc > cap;
  if (!over) {
    const uint64_t total = (uint64_t)world * cap;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
      const uint32_t r = (uint32_t)(e / cap), i = (uint32_t)(e % cap);
      const uint2* b = sp_all + (size_t)r * (cap + 1);
      if (i < b[0].x) {
        const uint2 t = b[1 + i];
        x[t.x] = t.y;
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && !(state[0] | state[4])) {
    state[5] = max(state[5], (long long)maxc);
    if (over) {
      state[4] = 1;
      state[6] = rec[0];
      state[7] = rec[1];
    } else {
      const uint32_t wit = kNone - (uint32_t)rec[1];
      state[1] += 1;
      if ((state[3] && wit != kNone) || !rec[0]) {
        state[0] = 1;
        state[2] = wit;
      }
    }
  }
}

__global__ void k_demote_count(uint32_t nwords, const uint32_t* __restrict__ acc,
                               uint32_t* __restrict__ used, uint32_t* __restrict__ rem,
                               unsigned long long* __restrict__ counts) {
  unsigned long long d = 0, f = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += stride) {
    const uint32_t a = acc[i], u = used[i];
    rem[i] = a & ~u;
    d += __popc(a & u);
    f += __popc(a & ~u);
    used[i] = 0u;
  }
  for (int o = 16; o > 0; o >>= 1) {
    d += __shfl_xor_sync(kFull, d, o);
    f += __shfl_xor_sync(kFull, f, o);
  }
  if (lane_id() == 0) {
    if (d) atomicAdd(counts, d);
    if (f) atomicAdd(counts + 1, f);
  }
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

void RunWs::ensure(uint32_t nn, uint32_t mm, const uint32_t* poff, cudaStream_t s) {
  if (ctl.p && n == nn && m == mm) {
    if (poff != bigm_src && nn) {  // layout changed: big-degree mask of the new push rows
      k_big_mask<<<grid_for((uint64_t)nn, 256, 8), 256, 0, s>>>(nn, poff, bigm.as<uint32_t>());
      CYC_LAUNCHED();
      bigm_src = poff;
    }
    return;
  }
  bigm_src = poff;
  n = nn;
  m = mm;
  n_pad = (uint32_t)(((uint64_t)nn + kRowPad - 1) / kRowPad * kRowPad);
  const size_t np1 = (size_t)n_pad + 1;
  const size_t words = (size_t)n_pad / 32 + 2;
  // a vertex of push degree d > kBigDeg yields ceil(d/kChunk) <= d/kChunk + 1 chunks
  chunk_cap = (uint32_t)((uint64_t)mm / kChunk + (uint64_t)mm / (kBigDeg + 1) + 16);
  wl_cap = (uint32_t)(2 * words + 64);
  for (int k = 0; k < 2; ++k) WL[k].alloc((size_t)wl_cap * 4, s);
  for (int k = 0; k < 2; ++k) {
    P[k].alloc(np1 * 4, s);
    CYC_CUDA(cudaMemsetAsync(P[k].p, 0, np1 * 4, s));  // padding rows stay NIL forever
    FB[k].alloc(words * 4, s);
    BC[k].alloc((size_t)chunk_cap * sizeof(uint4), s);
    C[k].alloc(np1 * 4, s);
  }
  F.alloc(words * 4, s);
  used.alloc(words * 4, s);
  bigm.alloc(words * 4, s);
  CYC_CUDA(cudaMemsetAsync(F.p, 0, words * 4, s));
  CYC_CUDA(cudaMemsetAsync(used.p, 0, words * 4, s));
  CYC_CUDA(cudaMemsetAsync(bigm.p, 0, words * 4, s));
  if (nn) {
    k_big_mask<<<grid_for((uint64_t)nn, 256, 8), 256, 0, s>>>(nn, poff, bigm.as<uint32_t>());
    CYC_LAUNCHED();
  }
  ctl.alloc(sizeof(RunCtl), s);
}

namespace {

// The arguments every run shares (workspace, CSRs, layout, options); resets
// the control block and the demotion scratch on s.
RunArgs base_args(const DevCsr& snap, const DevCsr& gath, uint32_t n, const uint32_t* orig, const uint32_t* perm,
                  const uint4* sdesc, const uint32_t* sell, const uint32_t* hcol, const uint32_t* hrow,
                  uint32_t n_hchunks, RunWs& ws, int early_exit, int mode, unsigned long long max_iterations,
                  unsigned long long max_steps, uint32_t alpha, unsigned long long cap, cudaStream_t s) {
  RunCtl init;
  std::memset(&init, 0, sizeof init);
  for (int k = 0; k < 3; ++k) init.slot[k].wit = kNone;
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
  a.world = 1;  // single device: the whole grid, all rows
  a.row_lo = 0;
  a.row_hi = ws.n_pad;
  a.goff = gath.o();
  a.gcol = gath.c();
  a.ell = gath.ell.as<uint32_t>();
  a.ovf = gath.ovf.as<uint32_t>();
  a.ell_k = gath.ell_k;
  a.n_pad = ws.n_pad;
  a.poff = snap.o();
  a.pcol = snap.c();
  a.bigm = ws.bigm.as<uint32_t>();
  a.heavy = gath.heavy.as<uint4>();
  a.n_heavy = gath.n_heavy_chunks;
  a.heavy_deg = gath.heavy_deg ? gath.heavy_deg : 0xFFFFFFFFu;
  for (int k = 0; k < 2; ++k) {
    a.P[k] = ws.P[k].as<uint32_t>();
    a.FB[k] = ws.FB[k].as<uint32_t>();
    a.BC[k] = ws.BC[k].as<uint4>();
    a.C[k] = ws.C[k].as<uint32_t>();
  }
  for (int k = 0; k < 2; ++k) a.WL[k] = ws.WL[k].as<uint32_t>();
  a.wl_cap = ws.wl_cap;
  a.F = ws.F.as<uint32_t>();
  a.used = ws.used.as<uint32_t>();
  a.orig = orig;
  a.perm = perm;
  a.sdesc = sdesc;
  a.sell = sell;
  a.hcol = hcol;
  a.hrow = hrow;
  a.n_hchunks = n_hchunks;
  ws.orig = orig;
  a.nwords = (uint32_t)(((uint64_t)n + 31) / 32);
  a.nwords_pad = ws.n_pad / 32u;
  a.chunk_cap = ws.chunk_cap;
  a.cand_cap = ws.n_pad + 1;
  a.ctl = ws.ctl.as<RunCtl>();
  a.iter_hash = cap ? ws.hist.as<unsigned long long>() : nullptr;
  a.iter_steps = cap ? ws.hist.as<unsigned long long>() + cap : nullptr;
  a.cap = cap;
  a.max_iterations = max_iterations;
  a.max_steps = max_steps;
  a.alpha = alpha ? alpha : 16u;  // swept on config 2: 4 81.2, 8 70.4, 16 69.4, 24 70.3, 64 71.4 ms
  a.early_exit = early_exit;
  a.mode = mode;
  return a;
}

}  // namespace

void launch_map_run(const DevCsr& snap, const DevCsr& gath, const uint32_t* orig, const uint32_t* perm,
                    const uint4* sdesc, const uint32_t* sell, const uint32_t* hcol, const uint32_t* hrow,
                    uint32_t n_hchunks, RunWs& ws, int early_exit, int mode,
                    unsigned long long max_iterations, unsigned long long max_steps,
                    uint32_t alpha, unsigned long long cap, uint32_t trace_cap, cudaStream_t s,
                    cudaEvent_t e0, cudaEvent_t e1, RunOut& out) {
  RunArgs a = base_args(snap, gath, gath.n, orig, perm, sdesc, sell, hcol, hrow, n_hchunks, ws, early_exit, mode,
                        max_iterations, max_steps, alpha, cap, s);
  // shared-memory staging of the hottest map words (degree-ordered plans only)
  static const size_t hot_cap = [] {  // thread-safe one-time init
    int dev = 0, optin = 0;
    CYC_CUDA(cudaGetDevice(&dev));
    CYC_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa;
    CYC_CUDA(cudaFuncGetAttributes(&fa, k_map_run<true, false>));
    // measured (scripts/micro/gather_mix.cu): random L2 gathers hold ~283 G/s
    // per GPU with up to 128 KB of shared memory per SM and halve at 200 KB
    // (the L1 carve-out that tracks in-flight loads shrinks), so stop at 128 KB
    size_t cap = (size_t)optin > fa.sharedSizeBytes + 1024 ? (size_t)optin - fa.sharedSizeBytes - 1024 : 0;
    cap = std::min<size_t>(cap, 128u << 10);
    for (const void* f : {(const void*)k_map_run<true, false>, (const void*)k_map_run<true, true>,
                          (const void*)k_map_run<false, true>})
      CYC_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap));
    return cap;
  }();
  // frontier bits of the first CYC_HOT_POS positions (tested at 2^19 = 64 KB)
  const char* hk = std::getenv("CYC_HOT_POS");
  uint64_t hot_pos = hk ? std::strtoull(hk, nullptr, 10) : 0ull;  // off by default: no gain measured on C3
  hot_pos = orig ? std::min<uint64_t>({hot_pos, (uint64_t)hot_cap * 8, (uint64_t)ws.n_pad}) : 0;
  a.hot_k = (uint32_t)(hot_pos / 32u * 32u);
  if (trace_cap) {
    if (ws.trace.bytes < (size_t)trace_cap * 512) ws.trace.alloc((size_t)trace_cap * 512, s);
    CYC_CUDA(cudaMemsetAsync(ws.trace.p, 0, (size_t)trace_cap * 512, s));
    a.trace = ws.trace.as<unsigned long long>();
    a.trace_cap = trace_cap;
  }

  static const int blocks_per_sm = [] {  // thread-safe one-time init
    int b = 0;
    CYC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_map_run<false, false>, kRunThreads, 0));
    return b > 0 ? b : 1;
  }();
  const size_t dyn = (size_t)a.hot_k / 8;
  int bps = blocks_per_sm;
  if (orig) {
    CYC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_map_run<true, false>, kRunThreadsRL, dyn));
    if (bps < 1) bps = 1;
  }
  dim3 grid((unsigned)(sm_count() * bps)), block(orig ? kRunThreadsRL : kRunThreads);
  a.blk0 = 0;
  a.nblk = grid.x;
  void* args[] = {&a};
  CYC_CUDA(cudaEventRecord(e0, s));
  coop_launch(orig ? (const void*)k_map_run<true, false> : (const void*)k_map_run<false, false>, grid, block, args,
              dyn, s);
  CYC_LAUNCHED();
  CYC_CUDA(cudaEventRecord(e1, s));
  RunCtl host;
  CYC_CUDA(cudaMemcpyAsync(&host, ws.ctl.p, sizeof host, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  std::memcpy(out.res, host.res, sizeof out.res);
  CYC_CUDA(cudaEventElapsedTime(&out.ms, e0, e1));
  out.grid = grid.x;
  out.block = block.x;
  const unsigned long long k = host.res[kResTag];  // trace slots are indexed by step tag
  ws.trace_len = (uint32_t)(k < trace_cap ? k : trace_cap);
}

void launch_map_run_shards(ShardRunIn* in, int k, bool emulated, int early_exit, int mode,
                           unsigned long long max_iterations, unsigned long long max_steps, uint32_t alpha,
                           unsigned long long cap, RunOut* outs) {
  std::vector<RunArgs> args(k);
  const bool rl = in[0].orig != nullptr;
  for (int i = 0; i < k; ++i) {
    ShardRunIn& r = in[i];
    CYC_CUDA(cudaSetDevice(r.device));
    if (cap && r.ws->hist.bytes < cap * 16) r.ws->hist.alloc(cap * 16, r.s);
    RunArgs& a = args[i];
    a = base_args(*r.push, *r.gath, r.n, r.orig, r.perm, r.sdesc, r.sell, r.hcol, r.hrow, r.n_hchunks, *r.ws,
                  early_exit, mode, max_iterations, max_steps, alpha, cap, r.s);
    a.m = (uint32_t)r.m_global;  // decisions and MapStats are about the whole graph
    a.bigm = r.bigm;
    for (int b = 0; b < 2; ++b) {
      a.P[b] = r.P[b];
      a.FB[b] = r.FB[b];
    }
    a.world = r.world;
    a.rank = r.rank;
    a.emulated = emulated;
    a.row_lo = r.row_lo;
    a.row_hi = r.row_hi;
    std::memcpy(a.peerP, r.peerP, sizeof a.peerP);
    std::memcpy(a.peerFB, r.peerFB, sizeof a.peerFB);
    a.rec = r.rec;
    std::memcpy(a.peerRec, r.peerRec, sizeof a.peerRec);
    a.bar = r.bar;
    std::memcpy(a.peerBar, r.peerBar, sizeof a.peerBar);
    a.bar_base = r.bar_base;
  }
  const dim3 block(rl ? kRunThreadsRL : kRunThreads);
  std::vector<cudaEvent_t> ev(2 * k);
  for (int i = 0; i < k; ++i) {
    CYC_CUDA(cudaSetDevice(in[i].device));
    CYC_CUDA(cudaEventCreate(&ev[2 * i]));
    CYC_CUDA(cudaEventCreate(&ev[2 * i + 1]));
  }
  if (emulated) {  // one grid, rank i = blocks [i*nblk, (i+1)*nblk)
    const uint32_t nblk = (uint32_t)sm_count() / (uint32_t)k;
    for (int i = 0; i < k; ++i) {
      args[i].blk0 = (uint32_t)i * nblk;
      args[i].nblk = nblk;
    }
    DevBuf dargs(sizeof(RunArgs) * k, in[0].s);
    CYC_CUDA(cudaMemcpyAsync(dargs.p, args.data(), sizeof(RunArgs) * k, cudaMemcpyHostToDevice, in[0].s));
    const RunArgs* pa = dargs.as<RunArgs>();
    int world = k;
    void* kargs[] = {&pa, &world};
    CYC_CUDA(cudaEventRecord(ev[0], in[0].s));
    coop_launch(rl ? (const void*)k_map_run_emul<true> : (const void*)k_map_run_emul<false>, dim3(nblk * k), block,
                kargs, 0, in[0].s);
    CYC_LAUNCHED();
    CYC_CUDA(cudaEventRecord(ev[1], in[0].s));
    for (int i = 1; i < k; ++i) {
      ev[2 * i] = ev[0];
      ev[2 * i + 1] = ev[1];
    }
    CYC_CUDA(cudaStreamSynchronize(in[0].s));
  } else {  // one cooperative grid per device, all in flight together
    const dim3 grid((unsigned)sm_count());
    for (int i = 0; i < k; ++i) {
      CYC_CUDA(cudaSetDevice(in[i].device));
      args[i].blk0 = 0;
      args[i].nblk = grid.x;
      void* kargs[] = {&args[i]};
      CYC_CUDA(cudaEventRecord(ev[2 * i], in[i].s));
      coop_launch(rl ? (const void*)k_map_run<true, true> : (const void*)k_map_run<false, true>, grid, block, kargs,
                  0, in[i].s);
      CYC_LAUNCHED();
      CYC_CUDA(cudaEventRecord(ev[2 * i + 1], in[i].s));
    }
  }
  for (int i = 0; i < k; ++i) {
    CYC_CUDA(cudaSetDevice(in[i].device));
    RunCtl host;
    CYC_CUDA(cudaMemcpyAsync(&host, in[i].ws->ctl.p, sizeof host, cudaMemcpyDeviceToHost, in[i].s));
    CYC_CUDA(cudaStreamSynchronize(in[i].s));
    std::memcpy(outs[i].res, host.res, sizeof outs[i].res);
    CYC_CUDA(cudaEventElapsedTime(&outs[i].ms, ev[2 * i], ev[2 * i + 1]));
    outs[i].grid = emulated ? (uint32_t)sm_count() / (uint32_t)k : (uint32_t)sm_count();
    outs[i].block = block.x;
    in[i].ws->orig = in[i].orig;
  }
  for (int i = 0; i < (emulated ? 1 : k); ++i) {
    CYC_CUDA(cudaSetDevice(in[i].device));
    cudaEventDestroy(ev[2 * i]);
    cudaEventDestroy(ev[2 * i + 1]);
  }
  CYC_CUDA(cudaSetDevice(in[0].device));
}

void strip_codes(const RunWs& ws, int cur, uint32_t n, uint32_t* dst, cudaStream_t s) {
  if (!n) return;
  if (ws.orig) {
    k_strip_perm<<<grid_for(n, 256, 8), 256, 0, s>>>(ws.P[cur].as<uint32_t>(), ws.orig, n, dst);
  } else {
    k_strip<<<grid_for(n, 256, 8), 256, 0, s>>>(ws.P[cur].as<uint32_t>(), n, dst);
  }
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

void launch_step_range(const DevCsr& gath, uint32_t lo, uint32_t hi, const uint32_t* x,
                       const uint32_t* accw, uint32_t* out, long long* rec, const long long* state,
                       int first_only, cudaStream_t s) {
  CYC_CUDA(cudaMemsetAsync(rec, 0, 16, s));
  if (hi <= lo) return;
  auto* r = reinterpret_cast<unsigned long long*>(rec);
  const uint32_t heavy = gath.n_heavy_chunks ? gath.heavy_deg : kNone;
  const uint32_t g = grid_for(hi - lo, 256, 8);
  const uint32_t n = gath.n, np = gath.ell_n;
  const uint32_t* ell = gath.ell.as<uint32_t>();
  const uint32_t* ovf = gath.ovf.as<uint32_t>();
  switch (gath.ell_k) {
    case 1: k_step_range_ell<1><<<g, 256, 0, s>>>(lo, hi, n, np, heavy, ell, ovf, gath.o(), gath.c(), x, accw, out, r, state, first_only); break;
    case 2: k_step_range_ell<2><<<g, 256, 0, s>>>(lo, hi, n, np, heavy, ell, ovf, gath.o(), gath.c(), x, accw, out, r, state, first_only); break;
    case 4: k_step_range_ell<4><<<g, 256, 0, s>>>(lo, hi, n, np, heavy, ell, ovf, gath.o(), gath.c(), x, accw, out, r, state, first_only); break;
    case 8: k_step_range_ell<8><<<g, 256, 0, s>>>(lo, hi, n, np, heavy, ell, ovf, gath.o(), gath.c(), x, accw, out, r, state, first_only); break;
    default: k_step_range<<<g, 256, 0, s>>>(lo, hi, heavy, gath.o(), gath.c(), x, accw, out, r, state, first_only); break;
  }
  CYC_LAUNCHED();
  if (gath.n_heavy_chunks) {
    const uint32_t nch = gath.n_heavy_chunks;
    k_step_range_chunks<<<grid_for((uint64_t)nch * 32, 256, 8), 256, 0, s>>>(
        gath.heavy.as<uint4>(), nch, lo, hi, gath.c(), x, accw, out, state, first_only);
    CYC_LAUNCHED();
    k_step_range_heavy<<<grid_for(nch, 256, 4), 256, 0, s>>>(gath.heavy.as<uint4>(), nch, lo, hi, gath.o(), x,
                                                             accw, out, r, state, first_only);
    CYC_LAUNCHED();
  }
}

void launch_shard_collect(uint32_t lo, uint32_t hi, const uint32_t* x, const uint32_t* out, uint32_t cap,
                          uint2* sp, const long long* state, int list_mode, const uint32_t* rlist,
                          const uint32_t* rcnt, uint32_t* rbits, const uint32_t* accw, long long* rec,
                          cudaStream_t s) {
  CYC_CUDA(cudaMemsetAsync(sp, 0, 8, s));
  if (hi <= lo) return;
  k_shard_collect<<<grid_for(hi - lo, 256, 8), 256, 0, s>>>(lo, hi, x, out, cap, sp, state, list_mode, rlist, rcnt,
                                                            rbits, accw,
                                                            reinterpret_cast<unsigned long long*>(rec));
  CYC_LAUNCHED();
}

void launch_shard_push(const uint2* sp_all, int world, uint32_t cap, const DevCsr& snap, uint32_t lo, uint32_t hi,
                       const uint32_t* accw, uint32_t* out, uint32_t* rbits, uint32_t* rlist, uint32_t* rcnt,
                       const long long* state, cudaStream_t s) {
  CYC_CUDA(cudaMemsetAsync(rcnt, 0, 4, s));
  k_shard_push<<<grid_for((uint64_t)world * cap * 32 + 32, 256, 8), 256, 0, s>>>(
      sp_all, world, cap, snap.o(), snap.c(), lo, hi, accw, out, rbits, rlist, rcnt, state);
  CYC_LAUNCHED();
}

void launch_shard_post_sparse(const long long* rec, long long* state, const uint2* sp_all, int world,
                              uint32_t cap, uint32_t* x, cudaStream_t s) {
  k_shard_post_sparse<<<grid_for((uint64_t)world * cap + 1, 256, 8), 256, 0, s>>>(rec, state, sp_all, world,
                                                                                  cap, x);
  CYC_LAUNCHED();
}

void launch_shard_post(const long long* rec, long long* state, const uint32_t* x_pad,
                       const uint32_t* bounds, int world, uint32_t maxrows, uint32_t* x, cudaStream_t s) {
  k_shard_post<<<grid_for((uint64_t)world * maxrows + 1, 256, 8), 256, 0, s>>>(rec, state, x_pad, bounds,
                                                                               world, maxrows, x);
  CYC_LAUNCHED();
}

void launch_demote_async(const uint32_t* x, uint32_t n, const uint32_t* accw, uint32_t* remaining,
                         unsigned long long* counts, uint32_t* used, cudaStream_t s) {
  const uint32_t nwords = (uint32_t)(((uint64_t)n + 31) / 32);
  CYC_CUDA(cudaMemsetAsync(counts, 0, 16, s));
  if (!n) return;
  k_mark_used<<<grid_for(n, 256, 8), 256, 0, s>>>(x, n, used);
  CYC_LAUNCHED();
  k_demote_count<<<grid_for(nwords, 256, 8), 256, 0, s>>>(nwords, accw, used, remaining, counts);
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
