// fused.cu — row-sharded MAP with the exchange fused into the step kernel
// (the NCCL protocol in sharded.py is the baseline).
//
// One persistent cooperative kernel per rank runs the whole run_map loop for
// its row range [lo, hi) of the gather index. Every rank holds the full
// replicated map vector, double-buffered (X[cur] read, X[nxt] written). In a
// step each row's new value is stored into the local X[nxt] AND straight into
// every peer's X[nxt] over NVLink (CUDA IPC pointers), tile by tile as it is
// computed — the transfer overlaps the math, no separate collective. The
// step record {changed, min self-witness} goes to every peer's flag slot, then
// a cross-GPU barrier (system-scope counters in each rank's memory, release by
// a system fence, acquire by the waiting thread) makes the step visible; every
// rank reduces the same records, so all stop at the same step with the same
// witness (kernel_calls identical to one device). Demotion (map_engine.cpp:
// 123-137) is replicated on the full local vector.
//
// Memory ordering: every writing thread issues __threadfence_system() before
// the local grid barrier; the lead then signals the peers with system-scope
// atomics; a peer's lead spins with ld.acquire.sys before its own grid
// barrier releases its blocks, which read X through L2 (ld.cg).
#include <cooperative_groups.h>

#include <vector>

#include "fused.cuh"

namespace cyc {

namespace {

namespace cg = cooperative_groups;
constexpr int kFT = 1024;

struct FusedArgs {
  const uint32_t* goff;
  const uint32_t* gcol;
  uint32_t n, lo, hi;
  int rank, world;
  uint32_t* X[2];                      // local replicated vector (codes)
  uint32_t* PX[kFusedMaxWorld][2];     // every rank's X (self = local)
  uint32_t* flags;                     // local flag slots [2][world][2], written by peers
  uint32_t* Pflags[kFusedMaxWorld];
  unsigned long long* bar;             // local barrier counter, incremented by every rank
  unsigned long long* Pbar[kFusedMaxWorld];
  uint32_t* acc;                       // local accepting words (u32), demoted in place
  uint32_t* used;                      // demotion scratch bitmap
  unsigned int* ctl;  // [0..4) step records (2 parities x {changed, witness}), [4..6) decision,
                      // [6] demoted count, [7] F non-empty
  unsigned long long* res;             // results
  int early_exit;
  unsigned long long barrier_base;     // barriers completed by earlier runs
};

__device__ __forceinline__ bool accb(const uint32_t* acc, uint32_t u) { return (acc[u >> 5] >> (u & 31u)) & 1u; }
__device__ __forceinline__ uint32_t cand(const uint32_t* acc, const uint32_t* X, uint32_t u) {
  const uint32_t x = __ldcg(X + u);
  return accb(acc, u) ? max(x, u + 1u) : x;
}
__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_acq_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// The whole run_map for this rank.
__global__ void __launch_bounds__(kFT, 1) k_fused_run(FusedArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned int s_ch, s_wit;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x, nthreads = gridDim.x * blockDim.x;
  const uint32_t gw = gtid >> 5, nw = nthreads >> 5;
  const uint32_t nwords = (a.n + 31u) / 32u;
  unsigned long long barriers = a.barrier_base, steps_total = 0, iterations = 0, demoted = 0;
  int cur = 0, cycle = 0;
  uint32_t witness = kNone;
  auto cross_barrier = [&]() {  // lead only
    __threadfence_system();
    for (int p = 0; p < a.world; ++p) atomicAdd_system(a.Pbar[p], 1ull);
    ++barriers;
    const unsigned long long target = barriers * (unsigned long long)a.world;
    const unsigned long long t0 = now_ns();
    while (ld_acq_sys(a.bar) < target)
      if (now_ns() - t0 > 30000000000ull) __trap();  // a peer is gone: fail loudly, never hang the GPU
  };
  // F count (replicated)
  for (;;) {
    // ---- fixpoint from all-NIL (both buffers reset, then every rank synced)
    for (uint32_t v = gtid; v <= a.n; v += nthreads) {
      a.X[0][v] = 0u;
      a.X[1][v] = 0u;
    }
    if (lead) a.ctl[7] = 0;  // F non-empty check below
    grid.sync();
    // F empty => no cycle
    {
      uint32_t any = 0;
      for (uint32_t w = gtid; w < nwords; w += nthreads) any |= a.acc[w];
      if (__any_sync(kFull, any != 0u) && lane == 0) atomicOr(&a.ctl[7], 1u);
    }
    __threadfence_system();
    grid.sync();
    if (lead) cross_barrier();  // nobody writes the next fixpoint's values before all reset
    grid.sync();
    if (__ldcg(&a.ctl[7]) == 0u) break;
    cur = 0;
    unsigned long long steps = 0;
    uint32_t wit_all = kNone;
    for (;;) {
      const uint32_t* Xc = a.X[cur];
      const int nx = cur ^ 1;
      if (threadIdx.x == 0) {
        s_ch = 0;
        s_wit = kNone;
      }
      __syncthreads();
      bool ch = false;
      uint32_t wit = kNone;
      // own rows: lanes take consecutive rows; rows longer than 32 by the warp
      for (uint32_t v0 = a.lo + gw * 32u; v0 < a.hi; v0 += nw * 32u) {
        const uint32_t v = v0 + lane;
        uint32_t b = 0, e = 0, best = 0, own = 0;
        if (v < a.hi) {
          b = a.goff[v];
          e = a.goff[v + 1];
          own = __ldcg(Xc + v);
          best = own;
        }
        const bool wide = e - b > 32u;
        if (v < a.hi && !wide)
          for (uint32_t i = b; i < e; ++i) best = max(best, cand(a.acc, Xc, a.gcol[i]));
        for (uint32_t wb = __ballot_sync(kFull, wide); wb; wb &= wb - 1u) {
          const uint32_t l = __ffs(wb) - 1u;
          const uint32_t rb = __shfl_sync(kFull, b, l), re = __shfl_sync(kFull, e, l);
          uint32_t m = 0;
          for (uint32_t i = rb + lane; i < re; i += 32u) m = max(m, cand(a.acc, Xc, a.gcol[i]));
          m = __reduce_max_sync(kFull, m);
          if (lane == l) best = max(best, m);
        }
        if (v < a.hi) {
          for (int p = 0; p < a.world; ++p) a.PX[p][nx][v] = best;  // self included (local store)
          ch |= best != own;
          if (best == v + 1u && accb(a.acc, v)) wit = min(wit, v);
        }
      }
      wit = __reduce_min_sync(kFull, wit);
      if (__any_sync(kFull, ch) && lane == 0) atomicOr(&s_ch, 1u);
      if (lane == 0 && wit != kNone) atomicMin(&s_wit, wit);
      __syncthreads();
      if (threadIdx.x == 0) {
        const uint32_t slot = (uint32_t)(steps % 2u) * 2u;
        if (s_ch) atomicOr(&a.ctl[slot], 1u);
        if (s_wit != kNone) atomicMin(&a.ctl[slot + 1], s_wit);
      }
      __threadfence_system();  // this thread's remote X stores before the signal
      grid.sync();
      if (lead) {
        const uint32_t slot = (uint32_t)(steps % 2u) * 2u;
        const uint32_t mc = __ldcg(&a.ctl[slot]), mw = __ldcg(&a.ctl[slot + 1]);
        a.ctl[slot] = 0u;  // reused two steps later, after two more grid barriers
        a.ctl[slot + 1] = kNone;
        const uint32_t fs = (uint32_t)(steps & 1u) * (uint32_t)a.world * 2u;
        for (int p = 0; p < a.world; ++p) {
          a.Pflags[p][fs + 2u * a.rank] = mc;
          a.Pflags[p][fs + 2u * a.rank + 1u] = mw;
        }
        cross_barrier();
        uint32_t c_all = 0, w_all = kNone;
        for (int r = 0; r < a.world; ++r) {
          c_all |= __ldcg(a.flags + fs + 2u * r);
          w_all = min(w_all, __ldcg(a.flags + fs + 2u * r + 1u));
        }
        a.ctl[4] = c_all;
        a.ctl[5] = w_all;
      }
      grid.sync();
      ++steps;
      cur = nx;
      const uint32_t c_all = __ldcg(&a.ctl[4]), w_all = __ldcg(&a.ctl[5]);
      if (a.early_exit && w_all != kNone) {
        wit_all = w_all;
        break;
      }
      if (!c_all) {
        wit_all = w_all;
        break;
      }
    }
    steps_total += steps;
    ++iterations;
    if (wit_all != kNone) {
      cycle = 1;
      witness = wit_all;
      break;
    }
    // ---- demote (replicated): used = {x - 1 : x != NIL}; D = F & used; F' = F \ D
    for (uint32_t w = gtid; w < nwords; w += nthreads) a.used[w] = 0u;
    if (lead) a.ctl[6] = 0;
    grid.sync();
    const uint32_t* Xf = a.X[cur];
    for (uint32_t v = gtid; v < a.n; v += nthreads) {
      const uint32_t x = __ldcg(Xf + v);
      if (x) atomicOr(&a.used[(x - 1u) >> 5], 1u << ((x - 1u) & 31u));
    }
    grid.sync();
    uint32_t dcount = 0;
    for (uint32_t w = gtid; w < nwords; w += nthreads) {
      const uint32_t d = a.acc[w] & a.used[w];
      dcount += __popc(d);
      a.acc[w] &= ~d;
    }
    dcount = __reduce_add_sync(kFull, dcount);
    if (lane == 0 && dcount) atomicAdd(&a.ctl[6], dcount);
    grid.sync();
    const uint32_t dc = __ldcg(&a.ctl[6]);
    demoted += dc;
    if (dc == 0) break;  // D empty: no cycle
    grid.sync();         // everyone read ctl[6] before the next fixpoint reuses ctl
  }
  if (lead) {
    a.res[0] = (unsigned long long)cycle;
    a.res[1] = witness;
    a.res[2] = iterations;
    a.res[3] = steps_total;
    a.res[4] = demoted;
    a.res[5] = (unsigned long long)cur;
    a.res[6] = barriers;
  }
}

}  // namespace

FusedShard::~FusedShard() {
  for (int p = 0; p < world; ++p)
    if (p != rank && peer_base[p]) cudaIpcCloseMemHandle(peer_base[p]);
  if (base) cudaFree(base);
}

void FusedShard::open(const DevCsr& gath_in, uint32_t lo_in, uint32_t hi_in, int rank_in, int world_in,
                      void* handle_out) {
  require_fused(world_in >= 1 && world_in <= kFusedMaxWorld && rank_in >= 0 && rank_in < world_in,
                "fused shard: bad rank / world");
  require_fused(lo_in <= hi_in && hi_in <= gath_in.n, "fused shard: bad row range");
  gath = &gath_in;
  lo = lo_in;
  hi = hi_in;
  rank = rank_in;
  world = world_in;
  const uint32_t n = gath_in.n;
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  off_x0 = 0;
  off_x1 = align(((size_t)n + 1) * 4);
  off_flags = off_x1 + align(((size_t)n + 1) * 4);
  off_bar = off_flags + align((size_t)2 * kFusedMaxWorld * 2 * 4);
  bytes = off_bar + 256;
  CYC_CUDA(cudaMalloc(&base, bytes));  // plain cudaMalloc: exportable through CUDA IPC
  CYC_CUDA(cudaMemset(base, 0, bytes));
  cudaIpcMemHandle_t h;
  CYC_CUDA(cudaIpcGetMemHandle(&h, base));
  std::memcpy(handle_out, &h, sizeof h);
}

void FusedShard::connect(const void* handles) {
  const auto* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
  for (int p = 0; p < world; ++p) {
    if (p == rank) {
      peer_base[p] = base;
      continue;
    }
    void* ptr = nullptr;
    CYC_CUDA(cudaIpcOpenMemHandle(&ptr, hs[p], cudaIpcMemLazyEnablePeerAccess));
    peer_base[p] = ptr;
  }
  connected = true;
}

void FusedShard::run(const uint64_t* acc_words, int early_exit, cudaStream_t s, unsigned long long res[6]) {
  unsigned long long hres[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  require_fused(connected, "fused shard: connect() first");
  const uint32_t n = gath->n;
  const size_t nwords = ((size_t)n + 31) / 32 + 1;
  DevBuf acc(nwords * 4, s), used(nwords * 4, s), ctl(64, s), dres(64, s);
  CYC_CUDA(cudaMemsetAsync(acc.p, 0, nwords * 4, s));
  if (n) CYC_CUDA(cudaMemcpyAsync(acc.p, acc_words, ((size_t)n + 63) / 64 * 8, cudaMemcpyDefault, s));
  // trim tail bits beyond n (Bitset::trim)
  if (n & 31u) {
    const uint32_t keep = (1u << (n & 31u)) - 1u;
    uint32_t last = 0;
    CYC_CUDA(cudaMemcpyAsync(&last, acc.as<uint32_t>() + n / 32, 4, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
    last &= keep;
    CYC_CUDA(cudaMemcpyAsync(acc.as<uint32_t>() + n / 32, &last, 4, cudaMemcpyHostToDevice, s));
  }
  unsigned int init[8] = {0u, kNone, 0u, kNone, 0u, kNone, 0u, 0u};
  CYC_CUDA(cudaMemcpyAsync(ctl.p, init, sizeof init, cudaMemcpyHostToDevice, s));
  FusedArgs a{};
  a.goff = gath->o();
  a.gcol = gath->c();
  a.n = n;
  a.lo = lo;
  a.hi = hi;
  a.rank = rank;
  a.world = world;
  auto at = [](void* b, size_t o) { return reinterpret_cast<char*>(b) + o; };
  a.X[0] = reinterpret_cast<uint32_t*>(at(base, off_x0));
  a.X[1] = reinterpret_cast<uint32_t*>(at(base, off_x1));
  a.flags = reinterpret_cast<uint32_t*>(at(base, off_flags));
  a.bar = reinterpret_cast<unsigned long long*>(at(base, off_bar));
  for (int p = 0; p < world; ++p) {
    a.PX[p][0] = reinterpret_cast<uint32_t*>(at(peer_base[p], off_x0));
    a.PX[p][1] = reinterpret_cast<uint32_t*>(at(peer_base[p], off_x1));
    a.Pflags[p] = reinterpret_cast<uint32_t*>(at(peer_base[p], off_flags));
    a.Pbar[p] = reinterpret_cast<unsigned long long*>(at(peer_base[p], off_bar));
  }
  a.acc = acc.as<uint32_t>();
  a.used = used.as<uint32_t>();
  a.ctl = ctl.as<unsigned int>();
  a.res = dres.as<unsigned long long>();
  a.early_exit = early_exit;
  // barrier counters only grow (zeroed at open, before any peer connects);
  // every rank runs the same barrier sequence, so the count so far is shared
  a.barrier_base = barriers_done;
  CYC_CUDA(cudaStreamSynchronize(s));
  static int grid = [] {
    int b = 0;
    CYC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_fused_run, kFT, 0));
    require_fused(b >= 1, "fused shard: kernel does not fit an SM");
    return sm_count();
  }();
  void* args[] = {&a};
  coop_launch((const void*)k_fused_run, dim3(grid), dim3(kFT), args, 0, s);
  CYC_LAUNCHED();
  CYC_CUDA(cudaMemcpyAsync(hres, dres.p, 7 * 8, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  for (int k = 0; k < 6; ++k) res[k] = hres[k];
  final_cur = (int)hres[5];
  barriers_done = hres[6];
}

void FusedShard::final_vector(uint32_t* out, cudaStream_t s) const {
  const uint32_t* src =
      reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(base) + (final_cur ? off_x1 : off_x0));
  CYC_CUDA(cudaMemcpyAsync(out, src, (size_t)gath->n * 4, cudaMemcpyDefault, s));
  CYC_CUDA(cudaStreamSynchronize(s));
}

}  // namespace cyc
