// ingest.cuh — explicit-graph text and binary ingestion on the device.
#pragma once

#include <string>

#include "build.cuh"

namespace cyc {

// DiagCode values of the reference (errors.hpp:21-28) that the format uses.
constexpr int kDiagSyntax = 0;
constexpr int kDiagRange = 5;

// cycheck::ParseError (errors.hpp:32-45): code, 1-based line and column.
struct ParseFailure : std::runtime_error {
  int code, line, col;
  ParseFailure(int c, int l, int k, const std::string& m) : std::runtime_error(m), code(c), line(l), col(k) {}
};

inline void require_ingest(bool ok, const char* msg) {
  if (!ok) throw Error(CYC_E_RESOURCE, msg);
}

// ExplicitGraph (graph.hpp:140-144) on the device.
struct ExplicitDev {
  uint32_t n = 0;
  uint64_t n_acc = 0;  // accepting ids in file order (duplicates kept)
  uint64_t m = 0;
  DevBuf edges;        // uint2 (src, dst), file order
  DevBuf acc_ids;      // u32[n_acc]
  DevBuf acc_words;    // binary format: u64 words of n bits
  bool has_words = false;
};

// parse_explicit_graph (graph.cpp:259-297) over device text (16-byte aligned);
// throws ParseFailure exactly where and as the reference throws ParseError.
void parse_explicit_device(const uint8_t* dtext, uint64_t len, cudaStream_t s, ExplicitDev& out);
// fill_log's accepting bitset (graph.cpp:305-310) as u64 words.
void explicit_acc_words(const ExplicitDev& g, cudaStream_t s, DevBuf& words);
// accepting ids (ascending) of a graph loaded from the binary format.
void explicit_acc_ids_from_words(ExplicitDev& g, cudaStream_t s);

}  // namespace cyc
