// scc.cuh — K2: restriction of a snapshot to its cyclic accepting SCCs.
#pragma once

#include "build.cuh"

namespace cyc {

// restrict_to_accepting_sccs (reference graph.cpp:190-221) on device CSRs.
// snap/gath are the snapshot relation and its reverse; acc = u64 words.
void restrict_graph(const DevCsr& snap, const DevCsr& gath, const uint64_t* acc, cudaStream_t s,
                    DevCsr& out_snap, DevCsr& out_gath, DevBuf& out_acc, DevBuf& out_kept);

// keep mask only (u8 per vertex), for tests and the device SCC verdict.
void scc_keep_mask(const DevCsr& snap, const DevCsr& gath, const uint64_t* acc, cudaStream_t s,
                   uint8_t* keep);

// Accepting vertices of cyclic SCCs, ascending (scc_verdict, oracle.cpp:32-98).
uint32_t scc_cyclic_accepting(const DevCsr& snap, const DevCsr& gath, const uint64_t* acc,
                              cudaStream_t s, DevBuf& list);

}  // namespace cyc
