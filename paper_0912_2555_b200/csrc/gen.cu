// gen.cu — device generator for the C4 product graph (include/cyc_gen.h):
// vertex ids in BFS discovery order from the initial state, exactly the
// sequential queue order of cyc_prod_generate_host, computed level by level.
//
// Level frontier = the id range [a, b) (ids are handed out level by level,
// in order). Sequential BFS gives an undiscovered successor the id of its
// FIRST discovery in (parent id, successor index) order, so per level:
//   claim:  every candidate (t = (i-a)*6 + j) atomicMin's its key into
//           claim[state] when the state has no id yet;
//   flag:   the candidate holding the minimum is the discoverer;
//   scan:   exclusive scan of the flags in t order = new ids b + rank.
// Then the log is emitted per source id in successor order, as on the host.
#include "gen.cuh"

namespace cyc {

namespace {

constexpr int kT = 256;
constexpr uint32_t kSlots = 6;  // max successors of a product state

__global__ void k_prod_init(uint32_t n, uint32_t* id_of_key, uint32_t* claim) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    id_of_key[k] = k == 0 ? 0u : kNone;
    claim[k] = kNone;
  }
}

__global__ void k_prod_claim(cyc_gen_params p, uint32_t a, uint32_t cand, const uint32_t* __restrict__ key_of_id,
                             const uint32_t* __restrict__ id_of_key, uint32_t* claim) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < cand; t += gridDim.x * blockDim.x) {
    uint32_t succ[kSlots];
    const uint32_t c = cyc_prod_succ(&p, key_of_id[a + t / kSlots], succ);
    const uint32_t j = t % kSlots;
    if (j < c && id_of_key[succ[j]] == kNone) atomicMin(&claim[succ[j]], t);
  }
}

__global__ void k_prod_flag(cyc_gen_params p, uint32_t a, uint32_t cand, const uint32_t* __restrict__ key_of_id,
                            const uint32_t* __restrict__ id_of_key, const uint32_t* __restrict__ claim,
                            uint32_t* flag) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < cand; t += gridDim.x * blockDim.x) {
    uint32_t succ[kSlots];
    const uint32_t c = cyc_prod_succ(&p, key_of_id[a + t / kSlots], succ);
    const uint32_t j = t % kSlots;
    flag[t] = j < c && id_of_key[succ[j]] == kNone && claim[succ[j]] == t;
  }
}

__global__ void k_prod_assign(cyc_gen_params p, uint32_t a, uint32_t b, uint32_t cand,
                              uint32_t* __restrict__ key_of_id, uint32_t* __restrict__ id_of_key,
                              const uint32_t* __restrict__ flag, const uint32_t* __restrict__ rank) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < cand; t += gridDim.x * blockDim.x) {
    if (!flag[t]) continue;
    uint32_t succ[kSlots];
    cyc_prod_succ(&p, key_of_id[a + t / kSlots], succ);
    const uint32_t key = succ[t % kSlots], id = b + rank[t];
    id_of_key[key] = id;
    key_of_id[id] = key;
  }
}

__global__ void k_prod_degree(cyc_gen_params p, const uint32_t* __restrict__ key_of_id, uint32_t* deg) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < p.n; v += gridDim.x * blockDim.x) {
    uint32_t succ[kSlots];
    deg[v] = cyc_prod_succ(&p, key_of_id[v], succ);
  }
}

__global__ void k_prod_emit(cyc_gen_params p, const uint32_t* __restrict__ key_of_id,
                            const uint32_t* __restrict__ id_of_key, const uint32_t* __restrict__ pos,
                            uint2* edges, uint64_t* acc) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < p.n; v += gridDim.x * blockDim.x) {
    uint32_t succ[kSlots];
    const uint32_t key = key_of_id[v];
    const uint32_t c = cyc_prod_succ(&p, key, succ);
    if (edges)
      for (uint32_t j = 0; j < c; ++j) edges[(uint64_t)pos[v] + j] = make_uint2(v, id_of_key[succ[j]]);
    if (acc) {
      const unsigned bal = __ballot_sync(__activemask(), cyc_prod_accepting_key(&p, key));
      // v..v+31 of a full warp cover half of one u64 word (grid stride is a multiple of 64)
      if ((threadIdx.x & 31u) == 0) {
        uint32_t* w32 = reinterpret_cast<uint32_t*>(acc);
        w32[v >> 5] = bal;
      }
    }
  }
}

}  // namespace

void gen_product_device(const cyc_gen_params& p, uint32_t* edges, uint64_t* acc, cudaStream_t s) {
  const uint32_t n = p.n;
  require_gen(p.kind == CYC_GEN_PRODUCT && n > 0 && (n & 63u) == 0, "product generator: bad params");
  DevBuf key_of_id((size_t)n * 4, s), id_of_key((size_t)n * 4, s), claim((size_t)n * 4, s);
  DevBuf flag, rank, scratch, tot(8, s);
  k_prod_init<<<grid_for(n, kT, 8), kT, 0, s>>>(n, id_of_key.as<uint32_t>(), claim.as<uint32_t>());
  CYC_LAUNCHED();
  CYC_CUDA(cudaMemsetAsync(key_of_id.p, 0, 4, s));
  uint32_t a = 0, b = 1;
  size_t cap = 0;
  while (a < b) {
    const uint64_t cand64 = (uint64_t)(b - a) * kSlots;
    require_gen(cand64 < 0xFFFFFFFFull, "product generator: frontier too large");
    const uint32_t cand = (uint32_t)cand64;
    if (cand > cap) {
      cap = (size_t)cand * 2;
      flag.alloc(cap * 4 + 4, s);
      rank.alloc(cap * 4 + 4, s);
    }
    const uint32_t g = grid_for(cand, kT, 8);
    k_prod_claim<<<g, kT, 0, s>>>(p, a, cand, key_of_id.as<uint32_t>(), id_of_key.as<uint32_t>(),
                                  claim.as<uint32_t>());
    CYC_LAUNCHED();
    k_prod_flag<<<g, kT, 0, s>>>(p, a, cand, key_of_id.as<uint32_t>(), id_of_key.as<uint32_t>(),
                                 claim.as<uint32_t>(), flag.as<uint32_t>());
    CYC_LAUNCHED();
    exclusive_scan(flag.as<uint32_t>(), rank.as<uint32_t>(), cand, tot.as<uint32_t>(), s, scratch);
    k_prod_assign<<<g, kT, 0, s>>>(p, a, b, cand, key_of_id.as<uint32_t>(), id_of_key.as<uint32_t>(),
                                   flag.as<uint32_t>(), rank.as<uint32_t>());
    CYC_LAUNCHED();
    uint32_t found = 0;
    CYC_CUDA(cudaMemcpyAsync(&found, tot.p, 4, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
    a = b;
    b += found;
  }
  require_gen(b == n, "product generator: unreachable states");
  // the log: per source id, successors in canonical order
  DevBuf deg((size_t)n * 4, s), pos((size_t)n * 4 + 4, s);
  const uint32_t gv = grid_for(n, kT, 8);
  k_prod_degree<<<gv, kT, 0, s>>>(p, key_of_id.as<uint32_t>(), deg.as<uint32_t>());
  CYC_LAUNCHED();
  exclusive_scan(deg.as<uint32_t>(), pos.as<uint32_t>(), n, tot.as<uint32_t>(), s, scratch);
  k_prod_emit<<<gv, kT, 0, s>>>(p, key_of_id.as<uint32_t>(), id_of_key.as<uint32_t>(), pos.as<uint32_t>(),
                                reinterpret_cast<uint2*>(edges), acc);
  CYC_LAUNCHED();
}

}  // namespace cyc
