// owcty.cu — OWCTY (One-Way-Catch-Them-Young) on the device: the paper's
// comparison algorithm (reference owcty.cpp:14-87), an independent accepting-
// cycle verdict on the same device snapshot.
//
// approx := V; repeat { approx := reach(approx); approx := elim(approx) }
// until approx is empty or unchanged. reach keeps the vertices of approx
// properly reachable (path length >= 1 through approx) from accepting vertices
// of approx (owcty.cpp:14-33); elim removes vertices with no predecessor in
// the set until none is left (owcty.cpp:35-54). Both are closures, so the
// device computes them with monotone dense passes (any order gives the same
// fixpoint); rows longer than the heavy threshold are split into warp chunks.
// Survivors non-empty <=> accepting cycle; witness = min accepting survivor.
#include <chrono>

#include "frontier.cuh"
#include "owcty.cuh"

namespace cyc {

namespace {

constexpr int kT = 256;

__device__ __forceinline__ bool accw(const uint64_t* acc, uint32_t v) {
  return (acc[v >> 6] >> (v & 63u)) & 1ull;
}

// reach (owcty.cpp:14-33) on the frontier engine: seeds = accepting members
// of the set (not marked: a source counts only if re-reached), push along
// the snapshot rows, only set members are marked.
struct OpReachIn {
  uint32_t* mark;
  const uint8_t* set;
  __device__ uint32_t token(uint32_t) const { return 0u; }
  __device__ bool relax(uint32_t, uint32_t, uint32_t w, uint32_t) const {
    return set[w] && test_and_set_bit(mark, w);
  }
};
struct SeedAccIn {
  const uint64_t* acc;
  const uint8_t* set;
  __device__ bool operator()(uint32_t v) const { return set[v] && accw(acc, v); }
};

__global__ void k_ow_take(uint32_t n, const uint32_t* __restrict__ r, uint8_t* set) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    set[v] = (r[v >> 5] >> (v & 31u)) & 1u;
}

// elim: drop set members without a predecessor in the set (in place, monotone)
__global__ void k_ow_elim(uint32_t n, const uint32_t* __restrict__ goff, const uint32_t* __restrict__ gcol,
                          uint32_t heavy, uint8_t* set, uint32_t* flag) {
  bool ch = false;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    if (!set[c] || goff[c + 1] - goff[c] > heavy) continue;
    bool any = false;
    for (uint32_t i = goff[c]; i < goff[c + 1] && !any; ++i) any = ((volatile uint8_t*)set)[gcol[i]] != 0;
    if (!any) {
      set[c] = 0;
      ch = true;
    }
  }
  if (ch) *flag = 1;
}

// heavy rows: a chunk with a live predecessor marks its row alive for this pass
__global__ void k_ow_elim_chunks(const uint4* __restrict__ chunks, uint32_t nch,
                                 const uint32_t* __restrict__ gcol, const uint8_t* set, uint8_t* alive) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t k = gw; k < nch; k += nw) {
    const uint4 ch = chunks[k];
    if (!set[ch.x]) continue;
    bool hit = false;
    for (uint32_t i = ch.y + lane; i < ch.z; i += 32u) hit |= ((volatile const uint8_t*)set)[gcol[i]] != 0;
    if (__any_sync(kFull, hit) && lane == 0) alive[ch.x] = 1;
  }
}

__global__ void k_ow_elim_heavy_apply(uint32_t n, const uint32_t* __restrict__ goff, uint32_t heavy,
                                      uint8_t* set, uint8_t* alive, uint32_t* flag) {
  bool ch = false;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    if (goff[c + 1] - goff[c] <= heavy) continue;
    if (set[c] && !alive[c]) {
      set[c] = 0;
      ch = true;
    }
    alive[c] = 0;
  }
  if (ch) *flag = 1;
}

// set := r; counts |set| and |set xor before|, min accepting member
__global__ void k_ow_commit(uint32_t n, uint8_t* set, uint8_t* before,
                            const uint64_t* __restrict__ acc, unsigned long long* cnt, uint32_t* minacc) {
  unsigned long long live = 0, diff = 0;
  uint32_t mn = kNone;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint8_t x = set[v];
    live += x;
    diff += x != before[v];
    before[v] = x;
    if (x && accw(acc, v)) mn = min(mn, v);
  }
  for (int o = 16; o > 0; o >>= 1) {
    live += __shfl_xor_sync(kFull, live, o);
    diff += __shfl_xor_sync(kFull, diff, o);
    mn = min(mn, __shfl_xor_sync(kFull, mn, o));
  }
  if ((threadIdx.x & 31u) == 0) {
    if (live) atomicAdd(cnt, live);
    if (diff) atomicAdd(cnt + 1, diff);
    if (mn != kNone) atomicMin(minacc, mn);
  }
}

__global__ void k_fill(uint32_t n, uint8_t* p, uint8_t v) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}

template <class F>
void until_stable(uint32_t* dflag, cudaStream_t s, F&& pass) {
  for (;;) {
    uint32_t h = 0;
    CYC_CUDA(cudaMemsetAsync(dflag, 0, 4, s));
    pass();
    CYC_CUDA(cudaMemcpyAsync(&h, dflag, 4, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
    if (!h) break;
  }
}

}  // namespace

OwctyResult run_owcty_device(const DevCsr& snap, const DevCsr& gath, const uint64_t* acc, cudaStream_t s) {
  using clk = std::chrono::steady_clock;
  auto ms = [](clk::time_point a) { return std::chrono::duration<double, std::milli>(clk::now() - a).count(); };
  OwctyResult out;
  const uint32_t n = gath.n;
  if (n == 0) return out;
  const size_t words = (size_t)n / 32 + 2;
  DevBuf set((size_t)n + 1, s), r(words * 4, s), before((size_t)n + 1, s), alive((size_t)n + 1, s);
  DevBuf ctl(64, s);
  uint32_t* flag = ctl.as<uint32_t>();
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(ctl.as<uint8_t>() + 16);
  uint32_t* minacc = reinterpret_cast<uint32_t*>(ctl.as<uint8_t>() + 32);
  const uint32_t grid = grid_for(n, kT, 8), cgrid = sm_count() * 8;
  const uint32_t hv = gath.heavy_deg ? gath.heavy_deg : kNone;
  FrontierWs fws;
  const FrontierBufs fb = fws.bufs(n, (uint64_t)snap.m, s);
  k_fill<<<grid, kT, 0, s>>>(n, set.as<uint8_t>(), 1);
  CYC_LAUNCHED();
  k_fill<<<grid, kT, 0, s>>>(n, before.as<uint8_t>(), 1);
  CYC_LAUNCHED();
  CYC_CUDA(cudaMemsetAsync(alive.p, 0, (size_t)n + 1, s));
  for (;;) {
    // reach (into r), then set := r
    auto t0 = clk::now();
    CYC_CUDA(cudaMemsetAsync(r.p, 0, words * 4, s));
    seed_frontier(n, SeedAccIn{acc, set.as<uint8_t>()}, fb, nullptr, s);
    run_frontier(snap.o(), snap.c(), fb, OpReachIn{r.as<uint32_t>(), set.as<uint8_t>()}, s);
    k_ow_take<<<grid, kT, 0, s>>>(n, r.as<uint32_t>(), set.as<uint8_t>());
    CYC_LAUNCHED();
    CYC_CUDA(cudaStreamSynchronize(s));
    out.reach_ms += ms(t0);
    auto t1 = clk::now();
    until_stable(flag, s, [&] {
      k_ow_elim<<<grid, kT, 0, s>>>(n, gath.o(), gath.c(), hv, set.as<uint8_t>(), flag);
      CYC_LAUNCHED();
      if (gath.n_heavy_chunks) {
        k_ow_elim_chunks<<<cgrid, kT, 0, s>>>(gath.heavy.as<uint4>(), gath.n_heavy_chunks, gath.c(),
                                              set.as<uint8_t>(), alive.as<uint8_t>());
        CYC_LAUNCHED();
        k_ow_elim_heavy_apply<<<grid, kT, 0, s>>>(n, gath.o(), hv, set.as<uint8_t>(), alive.as<uint8_t>(),
                                                  flag);
        CYC_LAUNCHED();
      }
    });
    out.elim_ms += ms(t1);
    CYC_CUDA(cudaMemsetAsync(cnt, 0, 16, s));
    CYC_CUDA(cudaMemsetAsync(minacc, 0xFF, 4, s));
    k_ow_commit<<<grid, kT, 0, s>>>(n, set.as<uint8_t>(), before.as<uint8_t>(), acc, cnt, minacc);
    CYC_LAUNCHED();
    unsigned long long hc[2];
    uint32_t hm = kNone;
    CYC_CUDA(cudaMemcpyAsync(hc, cnt, 16, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaMemcpyAsync(&hm, minacc, 4, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
    ++out.outer_iterations;
    if (hc[0] == 0 || hc[1] == 0) {
      out.final_size = hc[0];
      if (hc[0]) {
        out.cycle = true;
        out.witness = hm;
      }
      return out;
    }
  }
}

}  // namespace cyc
