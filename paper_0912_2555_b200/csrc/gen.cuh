// gen.cuh — device generation of synthetic inputs that are not a pure
// function of the edge index (C4: BFS-ordered product state space).
#pragma once

#include "../../include/cyc_gen.h"
#include "build.cuh"

namespace cyc {

inline void require_gen(bool ok, const char* msg) {
  if (!ok) throw Error(CYC_E_CONTRACT, msg);
}

// Fills edges (2*p.m u32, device, nullable) and acc (ceil(n/64) u64, device,
// nullable) exactly as cyc_prod_generate_host does.
void gen_product_device(const cyc_gen_params& p, uint32_t* edges, uint64_t* acc, cudaStream_t s);

}  // namespace cyc
