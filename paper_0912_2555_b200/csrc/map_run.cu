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
//         (max, vertex-id) semiring.
//   push  only the vertices raised in the previous step scatter their
//         frozen previous-step value with atomicMax into P[cur] in place.
//         A vertex that did not change cannot change anyone's max, so this
//         equals the dense step. The frozen value of a raised vertex is the
//         maximum raise it received in that step, kept per step parity in
//         T[] as (tag << 32 | value); tags grow monotonically, so T never
//         needs clearing and "first raise in this step" is a 64-bit
//         atomicMax whose previous tag is older.
// Step kind is chosen on the device from the previous frontier's edge count
// (push when edges * alpha < m): direction-optimising traversal.
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

__device__ __forceinline__ bool f_bit(const uint32_t* F, uint32_t v) {
  return (__ldcg(F + (v >> 5)) >> (v & 31u)) & 1u;
}

__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

// Frontier append, warp-aggregated: one 64-bit atomic hands out both the list
// position and the edge prefix, so Le[] is increasing along the list.
__device__ __forceinline__ void warp_append(bool want, uint32_t item, uint32_t deg,
                                            unsigned long long* ctr, uint32_t* Lv, uint32_t* Le) {
  const uint32_t mask = __ballot_sync(kFull, want);
  if (!mask) return;
  const uint32_t lane = lane_id();
  const uint32_t d = want ? deg : 0u;
  const uint32_t incl = warp_incl_scan(d);
  const uint32_t tot = __shfl_sync(kFull, incl, 31);
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(ctr, ((unsigned long long)__popc(mask) << 32) | tot);
  base = __shfl_sync(kFull, base, 0);
  if (want) {
    uint32_t pos = (uint32_t)(base >> 32) + __popc(mask & lanemask_lt());
    Lv[pos] = item;
    Le[pos] = (uint32_t)base + incl - d;
  }
}

__device__ __forceinline__ void warp_push_list(bool want, uint32_t item, unsigned int* ctr,
                                               uint32_t* list) {
  const uint32_t mask = __ballot_sync(kFull, want);
  if (!mask) return;
  uint32_t base = 0;
  if (lane_id() == 0) base = atomicAdd(ctr, (unsigned)__popc(mask));
  base = __shfl_sync(kFull, base, 0);
  if (want) list[base + __popc(mask & lanemask_lt())] = item;
}

__device__ __forceinline__ void warp_flags(bool raised, bool counted, RunCtl* ctl, uint32_t slot) {
  const uint32_t r = __ballot_sync(kFull, raised);
  const uint32_t c = __ballot_sync(kFull, counted);
  if (lane_id() == 0) {
    if (r) *(volatile unsigned int*)&ctl->changed[slot] = 1u;
    if (c) atomicAdd(&ctl->nraised[slot], (unsigned)__popc(c));
  }
}

__device__ uint32_t block_min(uint32_t x, uint32_t* red) {
  x = __reduce_min_sync(kFull, x);
  __syncthreads();
  if (lane_id() == 0) red[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t y = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : kNone;
    y = __reduce_min_sync(kFull, y);
    if (threadIdx.x == 0) red[32] = y;
  }
  __syncthreads();
  uint32_t r = red[32];
  __syncthreads();
  return r;
}

// ------------------------------------------------------------------ pull
__device__ void pull_step(const RunArgs& a, uint32_t g, int cur) {
  const uint32_t slot = g % 3u;
  const uint32_t* __restrict__ P = a.P[cur];
  uint32_t* __restrict__ Q = a.P[cur ^ 1];
  unsigned long long* Tc = a.T[g & 1u];
  uint32_t* Cn = a.C[g & 1u];
  RunCtl* ctl = a.ctl;
  const uint32_t lane = lane_id();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  // light rows: one lane per row, 32 consecutive rows per warp
  for (uint32_t base = gw * 32u; base < a.n; base += nw * 32u) {
    const uint32_t v = base + lane;
    bool raised = false;
    if (v < a.n) {
      const uint32_t b = __ldg(a.goff + v), e = __ldg(a.goff + v + 1);
      if (e - b <= a.heavy_deg) {
        const uint32_t own = __ldcg(P + v);
        uint32_t best = own & kCode;
        uint32_t i = b;
        for (; i + 4 <= e; i += 4) {
          uint32_t u0 = __ldg(a.gcol + i), u1 = __ldg(a.gcol + i + 1);
          uint32_t u2 = __ldg(a.gcol + i + 2), u3 = __ldg(a.gcol + i + 3);
          uint32_t w0 = __ldcg(P + u0), w1 = __ldcg(P + u1), w2 = __ldcg(P + u2), w3 = __ldcg(P + u3);
          uint32_t c0 = (w0 & kFlag) ? max(w0 & kCode, u0 + 1u) : w0;
          uint32_t c1 = (w1 & kFlag) ? max(w1 & kCode, u1 + 1u) : w1;
          uint32_t c2 = (w2 & kFlag) ? max(w2 & kCode, u2 + 1u) : w2;
          uint32_t c3 = (w3 & kFlag) ? max(w3 & kCode, u3 + 1u) : w3;
          best = max(best, max(max(c0, c1), max(c2, c3)));
        }
        for (; i < e; ++i) {
          uint32_t u = __ldg(a.gcol + i);
          uint32_t w = __ldcg(P + u);
          uint32_t c = (w & kFlag) ? max(w & kCode, u + 1u) : w;
          best = max(best, c);
        }
        Q[v] = (own & kFlag) | best;
        raised = best > (own & kCode);
        if ((own & kFlag) && best == v + 1u) atomicMin(&ctl->wit[slot], v);
      }
    }
    warp_flags(raised, raised, ctl, slot);
  }
  // heavy rows: one warp per chunk, combined with atomicMax into Q (Q holds an
  // earlier, never larger, value of the same fixpoint)
  for (uint32_t c = gw; c < a.n_heavy; c += nw) {
    const uint4 ch = a.heavy[c];
    const uint32_t v = ch.x;
    uint32_t best = 0;
    for (uint32_t i = ch.y + lane; i < ch.z; i += 32u) {
      uint32_t u = __ldg(a.gcol + i);
      uint32_t w = __ldcg(P + u);
      uint32_t cv = (w & kFlag) ? max(w & kCode, u + 1u) : w;
      best = max(best, cv);
    }
    best = __reduce_max_sync(kFull, best);
    bool raised = false, counted = false, cand = false;
    if (lane == 0) {
      const uint32_t own = __ldcg(P + v);
      best = max(best, own & kCode);
      atomicMax(Q + v, (own & kFlag) | best);
      if (best > (own & kCode)) {
        raised = true;
        unsigned long long pt = atomicMax(Tc + v, ((unsigned long long)g << 32) | best);
        counted = (uint32_t)(pt >> 32) < g;
        cand = (own & kFlag) && best == v + 1u;
      }
    }
    warp_flags(raised, counted, ctl, slot);
    warp_push_list(cand, v, &ctl->cand_cnt[slot], Cn);
  }
}

// After a pull step, rebuild the frontier of that step (tag gp) from the two
// buffers so that a push step can follow.
__device__ void transition_pass(const RunArgs& a, uint32_t gp, int cur) {
  const uint32_t* P = a.P[cur];
  const uint32_t* Q = a.P[cur ^ 1];
  unsigned long long* Tp = a.T[gp & 1u];
  unsigned long long* ctr = &a.ctl->list_ctr[gp % 3u];
  uint32_t* Lv = a.Lv[gp & 1u];
  uint32_t* Le = a.Le[gp & 1u];
  const uint32_t lane = lane_id();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t base = gw * 32u; base < a.n; base += nw * 32u) {
    const uint32_t v = base + lane;
    bool want = false;
    uint32_t deg = 0;
    if (v < a.n) {
      uint32_t xb = __ldcg(P + v) & kCode, xa = __ldcg(Q + v) & kCode;
      if (xb != xa) {
        Tp[v] = ((unsigned long long)gp << 32) | xb;
        deg = __ldg(a.poff + v + 1) - __ldg(a.poff + v);
        want = deg > 0;
      }
    }
    warp_append(want, v, deg, ctr, Lv, Le);
  }
}

// ------------------------------------------------------------------ push
__device__ void push_step(const RunArgs& a, uint32_t g, int cur) {
  const uint32_t slot = g % 3u, pslot = (g - 1u) % 3u;
  RunCtl* ctl = a.ctl;
  const unsigned long long lc = __ldcg(&ctl->list_ctr[pslot]);
  const uint32_t cnt = (uint32_t)(lc >> 32), Ef = (uint32_t)lc;
  if (Ef == 0) return;
  const uint32_t* Lv = a.Lv[(g - 1u) & 1u];
  const uint32_t* Le = a.Le[(g - 1u) & 1u];
  const unsigned long long* Tp = a.T[(g - 1u) & 1u];
  unsigned long long* Tc = a.T[g & 1u];
  uint32_t* Nv = a.Lv[g & 1u];
  uint32_t* Ne = a.Le[g & 1u];
  uint32_t* Cn = a.C[g & 1u];
  uint32_t* P = a.P[cur];
  const uint32_t lane = lane_id();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t per = (((Ef + nw - 1u) / nw) + 31u) & ~31u;
  const uint64_t lo64 = (uint64_t)gw * per;
  if (lo64 >= Ef) return;
  const uint32_t lo = (uint32_t)lo64;
  const uint32_t hi = min(Ef, lo + per);
  // i0 = largest list index with Le[i0] <= lo (32-ary search)
  uint32_t l = 0, h = cnt;  // invariant: Le[l] <= lo, answer in [l, h)
  while (h - l > 32u) {
    const uint32_t step = (h - l + 31u) / 32u;
    const uint32_t p = l + lane * step;
    const bool ok = p < h && __ldcg(Le + p) <= lo;
    const uint32_t bal = __ballot_sync(kFull, ok);
    const uint32_t j = 31u - __clz(bal);
    l = l + j * step;
    h = min(h, l + step);
  }
  {
    const uint32_t p = l + lane;
    const bool ok = p < h && __ldcg(Le + p) <= lo;
    l += 31u - __clz(__ballot_sync(kFull, ok));
  }
  uint32_t i0 = l;
  for (uint32_t t0 = lo; t0 < hi; t0 += 32u) {
    const uint32_t idx = i0 + lane;
    const bool inl = idx < cnt;
    const uint32_t E = inl ? __ldcg(Le + idx) : kNone;
    uint32_t V = 0, rowb = 0, pv = 0;
    if (inl && E < t0 + 32u) {
      V = __ldcg(Lv + idx);
      rowb = __ldg(a.poff + V);
      pv = (uint32_t)__ldcg(Tp + V);
      if (f_bit(a.F, V)) pv = max(pv, V + 1u);
    }
    const uint32_t e = t0 + lane;
    uint32_t o = 0;
#pragma unroll
    for (uint32_t s = 16; s > 0; s >>= 1) {
      const uint32_t j = o + s;
      const uint32_t Ej = __shfl_sync(kFull, E, j & 31u);
      if (j < 32u && Ej <= e) o = j;
    }
    const uint32_t w = __shfl_sync(kFull, V, o);
    const uint32_t eb = __shfl_sync(kFull, E, o);
    const uint32_t rb = __shfl_sync(kFull, rowb, o);
    const uint32_t val = __shfl_sync(kFull, pv, o);
    (void)w;
    bool raised = false, first = false, cand = false;
    uint32_t tgt = 0, deg = 0;
    if (e < hi) {
      tgt = __ldg(a.pcol + rb + (e - eb));
      const uint32_t old = __ldcg(P + tgt);
      if (val > (old & kCode)) {
        const uint32_t prev = atomicMax(P + tgt, (old & kFlag) | val);
        if ((prev & kCode) < val) {
          raised = true;
          const unsigned long long pt = atomicMax(Tc + tgt, ((unsigned long long)g << 32) | val);
          if ((uint32_t)(pt >> 32) < g) {
            first = true;
            deg = __ldg(a.poff + tgt + 1) - __ldg(a.poff + tgt);
          }
          cand = (old & kFlag) && val == tgt + 1u;
        }
      }
    }
    warp_flags(raised, first, ctl, slot);
    warp_append(first && deg > 0, tgt, deg, &ctl->list_ctr[slot], Nv, Ne);
    warp_push_list(cand, tgt, &ctl->cand_cnt[slot], Cn);
    // advance to the owner of t0 + 32 (within [i0, i0 + 32])
    const uint32_t nxt = t0 + 32u;
    const uint32_t le = __popc(__ballot_sync(kFull, E <= nxt));
    i0 += le - 1u;
    if (le == 32u && i0 + 1u < cnt && __ldcg(Le + i0 + 1u) <= nxt) i0 += 1u;
  }
}

// ------------------------------------------------------- iteration passes
// Dense pass over the fixpoint vector: iteration hash, full self-witness (for
// early_exit = false, map_engine.cpp:108-112) and the "used" bitmap of demote
// (map_engine.cpp:124-126).
__device__ void finish_pass(const RunArgs& a, int cur, uint64_t t, bool mark_used) {
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
  h = warp_sum64(h);
  fw = __reduce_min_sync(kFull, fw);
  if (lane == 0) {
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

// demote (map_engine.cpp:123-137) + start of the next fixpoint: F' = F \ used,
// |D| counted, both map buffers reset to all-NIL with the new accepting bits,
// and the initial frontier (every accepting vertex, value id+1, tag g).
__device__ void rebuild_pass(const RunArgs& a, uint32_t g, unsigned int* dcount,
                             unsigned long long* fsize) {
  RunCtl* ctl = a.ctl;
  const uint32_t lane = lane_id();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  unsigned long long* Tg = a.T[g & 1u];
  uint32_t* Lv = a.Lv[g & 1u];
  uint32_t* Le = a.Le[g & 1u];
  unsigned long long* ctr = &ctl->list_ctr[g % 3u];
  uint32_t dc = 0;
  unsigned long long fs = 0;
  for (uint32_t wb = gw * 32u; wb < a.nwords; wb += nw * 32u) {
    const uint32_t i = wb + lane;
    uint32_t nf = 0;
    if (i < a.nwords) {
      const uint32_t f = __ldcg(a.F + i), u = __ldcg(a.used + i);
      nf = f & ~u;
      dc += __popc(f & u);
      fs += __popc(nf);
      if (u) {
        a.F[i] = nf;
        a.used[i] = 0;
      }
    }
    const uint32_t jmax = min(32u, a.nwords - wb);
    for (uint32_t j = 0; j < jmax; ++j) {
      const uint32_t nfj = __shfl_sync(kFull, nf, j);
      const uint32_t v = (wb + j) * 32u + lane;
      bool want = false;
      uint32_t deg = 0;
      if (v < a.n) {
        const bool acc = (nfj >> lane) & 1u;
        const uint32_t val = acc ? kFlag : 0u;
        a.P[0][v] = val;
        a.P[1][v] = val;
        if (acc) {
          deg = __ldg(a.poff + v + 1) - __ldg(a.poff + v);
          want = deg > 0;
          if (want) Tg[v] = ((unsigned long long)g << 32) | (v + 1u);
        }
      }
      warp_append(want, v, deg, ctr, Lv, Le);
    }
  }
  dc = __reduce_add_sync(kFull, dc);
  fs = warp_sum64(fs);
  if (lane == 0) {
    if (dcount && dc) atomicAdd(dcount, dc);
    if (fs) atomicAdd(fsize, fs);
  }
}

__device__ __forceinline__ void reset_slot(RunCtl* c, uint32_t s) {
  c->list_ctr[s] = 0;
  c->cand_cnt[s] = 0;
  c->wit[s] = kNone;
  c->changed[s] = 0;
  c->nraised[s] = 0;
}

__global__ void __launch_bounds__(kRunThreads, 1) k_map_run(RunArgs a) {
  __shared__ uint32_t red[33];
  RunCtl* ctl = a.ctl;
  unsigned long long epoch = 0;
  uint32_t g = a.tag0;
  int cur = 0;
  unsigned long long iterations = 0, kernel_calls = 0, demoted = 0, steps_last = 0;
  unsigned long long pull_steps = 0, push_steps = 0, edges = 0, rows = 0, bytes = 0;
  int cycle = 0;
  uint32_t witness = kNone;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;

  rebuild_pass(a, g, nullptr, &ctl->it_fsize[0]);
  grid_sync(&ctl->bar, epoch);
  uint64_t t = 0;
  bool truncated = false;
  for (;;) {
    if (__ldcg(&ctl->it_fsize[t & 1u]) == 0) break;  // front.any() == false
    unsigned long long steps = 0;
    bool prev_list = true;
    for (;;) {
      ++g;
      ++steps;
      const uint32_t slot = g % 3u, pslot = (g - 1u) % 3u;
      if (lead) reset_slot(ctl, (g + 1u) % 3u);
      int mode = a.mode;
      if (mode != kModePull && mode != kModePush) {
        if (prev_list) {
          const uint32_t Ef = (uint32_t)__ldcg(&ctl->list_ctr[pslot]);
          mode = ((unsigned long long)Ef * a.alpha < a.m) ? kModePush : kModePull;
        } else {
          const unsigned long long nr = __ldcg(&ctl->nraised[pslot]);
          const unsigned long long est = a.n ? nr * a.m / a.n : 0;
          mode = (est * a.alpha < a.m) ? kModePush : kModePull;
        }
      }
      if (mode == kModePush) {
        if (!prev_list) {
          transition_pass(a, g - 1u, cur);
          grid_sync(&ctl->bar, epoch);
        }
        const unsigned long long lc = __ldcg(&ctl->list_ctr[pslot]);
        edges += (uint32_t)lc;
        rows += lc >> 32;
        bytes += 8ull * (uint32_t)lc + 12ull * (lc >> 32);
        ++push_steps;
        push_step(a, g, cur);
      } else {
        edges += a.m;
        rows += a.n;
        bytes += 8ull * a.m + 12ull * a.n + 4ull;
        ++pull_steps;
        pull_step(a, g, cur);
      }
      grid_sync(&ctl->bar, epoch);
      if (mode == kModePull) cur ^= 1;
      prev_list = mode == kModePush;
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
        w = min(w, block_min(mine, red));
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
    steps_last = steps;
    if (truncated) {
      ++iterations;
      kernel_calls += steps;
      break;
    }
    finish_pass(a, cur, t, !cycle);
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
    ++iterations;
    kernel_calls += steps;
    if (cycle) break;
    if (a.max_iterations && iterations >= a.max_iterations) break;
    ++g;
    rebuild_pass(a, g, &ctl->it_dcount[t & 1u], &ctl->it_fsize[(t + 1u) & 1u]);
    grid_sync(&ctl->bar, epoch);
    const uint32_t dc = __ldcg(&ctl->it_dcount[t & 1u]);
    demoted += dc;
    if (dc == 0) break;
    ++t;
  }
  if (lead) {
    unsigned long long* r = ctl->res;
    r[kResCycle] = cycle;
    r[kResWitness] = witness;
    r[kResIterations] = iterations;
    r[kResKernelCalls] = kernel_calls;
    r[kResDemoted] = demoted;
    r[kResStepsLast] = steps_last;
    r[kResPullSteps] = pull_steps;
    r[kResPushSteps] = push_steps;
    r[kResEdges] = edges;
    r[kResRows] = rows;
    r[kResBytes] = bytes;
    r[kResCur] = (unsigned long long)cur;
    r[kResTag] = g;
  }
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

void RunWs::ensure(uint32_t nn, cudaStream_t s) {
  if (ctl.p && n == nn) return;
  n = nn;
  const size_t n1 = (size_t)nn + 1;
  for (int k = 0; k < 2; ++k) {
    P[k].alloc(n1 * 4, s);
    T[k].alloc(n1 * 8, s);
    Lv[k].alloc(n1 * 4, s);
    Le[k].alloc(n1 * 4, s);
    C[k].alloc(n1 * 4, s);
    CYC_CUDA(cudaMemsetAsync(T[k].p, 0, n1 * 8, s));
  }
  const size_t words = ((size_t)nn + 63) / 64 * 2 + 2;
  F.alloc(words * 4, s);
  used.alloc(words * 4, s);
  CYC_CUDA(cudaMemsetAsync(used.p, 0, words * 4, s));
  ctl.alloc(sizeof(RunCtl), s);
  tag = 1;
}

void launch_map_run(const DevCsr& snap, const DevCsr& gath, RunWs& ws, int early_exit, int mode,
                    unsigned long long max_iterations, unsigned long long max_steps,
                    uint32_t alpha, unsigned long long cap, cudaStream_t s, cudaEvent_t e0,
                    cudaEvent_t e1, RunOut& out) {
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
    a.Lv[k] = ws.Lv[k].as<uint32_t>();
    a.Le[k] = ws.Le[k].as<uint32_t>();
    a.C[k] = ws.C[k].as<uint32_t>();
  }
  a.F = ws.F.as<uint32_t>();
  a.used = ws.used.as<uint32_t>();
  a.nwords = (uint32_t)(((uint64_t)n + 31) / 32);
  a.ctl = ws.ctl.as<RunCtl>();
  a.iter_hash = cap ? ws.hist.as<unsigned long long>() : nullptr;
  a.iter_steps = cap ? ws.hist.as<unsigned long long>() + cap : nullptr;
  a.cap = cap;
  a.max_iterations = max_iterations;
  a.max_steps = max_steps;
  a.tag0 = ws.tag;
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
