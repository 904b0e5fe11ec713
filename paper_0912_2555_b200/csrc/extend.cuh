// extend.cuh — incremental snapshot support: row-wise sorted union of CSRs.
#pragma once

#include "build.cuh"

namespace cyc {

// out (n rows) = row-wise sorted, duplicate-free union of a (a.n <= n rows;
// missing rows empty) and b (n rows). Both inputs have sorted unique rows.
void merge_csr(const DevCsr& a, const DevCsr& b, uint32_t n, cudaStream_t s, DevCsr& out);

}  // namespace cyc
