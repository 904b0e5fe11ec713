// owcty.cuh — OWCTY verdict on the device (reference owcty.hpp / owcty.cpp).
#pragma once

#include "build.cuh"

namespace cyc {

struct OwctyResult {
  bool cycle = false;
  uint32_t witness = kNone;
  uint64_t outer_iterations = 0;
  uint64_t final_size = 0;
  double reach_ms = 0.0;
  double elim_ms = 0.0;
};

// run_owcty (owcty.cpp:56-87) over the relation of `snap` (row u = successors
// of u), `gath` its reverse; acc = u64 accepting words.
OwctyResult run_owcty_device(const DevCsr& snap, const DevCsr& gath, const uint64_t* acc, cudaStream_t s);

}  // namespace cyc
