// plan.cuh — storage layout of the MAP loop's map vector and CSRs.
//
// The reference gathers x[u] for every edge of every row in vertex-id order
// (map_engine.cpp:56-63). On a power-law graph whose ids are a random
// permutation (config 3: R-MAT 2^26 with a seeded vertex permutation) the
// gathered columns are spread over the whole 268 MB map vector, so every 32 B
// L2 sector holds one hot word and seven cold ones and the vector cannot stay
// in the 126 MB L2 (measured: 40 % L2 hit, ~30 GB DRAM per dense step for
// 9.3 GB of algorithmic bytes).
//
// A plan stores vertex v at position perm[v], positions ordered by how often
// the vertex is gathered (its in-degree in the gather relation = its row
// length in the snapshot relation), descending. The hottest words then share
// sectors and the hot prefix fits L2. Only storage moves: map VALUES stay
// original ids + 1, so max, the self-witness and the demotion set are the
// reference's, and every id that leaves the kernel (witness, iteration hash,
// final vector, used set) is mapped back through orig[]/perm[].
#pragma once

#include "build.cuh"

namespace cyc {

enum PlanLayout { kLayoutAuto = 0, kLayoutIdentity = 1, kLayoutDegree = 2 };

struct MapPlan {
  bool decided = false;
  bool relabel = false;   // storage order differs from vertex ids
  int layout = -1;        // layout the decision was made for
  DevCsr gath, snap;      // storage-space gather index and snapshot relation (relabel only)
  DevBuf orig;            // u32[n_pad + 1]: storage position -> vertex id (identity on padding)
  DevBuf perm;            // u32[n]: vertex id -> storage position
  // sliced ELL of the storage gather rows of at most kHeavyDeg edges: slice s =
  // rows [32s, 32s+32) padded to its widest row, column-major (sell[(off+j)*32
  // + lane]); sdesc[s] = {off, width, mask of heavy rows, 0}; absent entries
  // hold n_pad (the always-NIL map slot). Longer rows: gath's heavy chunks.
  DevBuf sell, sdesc;
  uint64_t sell_words = 0;
  // rows longer than kHeavyDeg as kHeavyChunk-column chunks: chunk c = hcol[c *
  // kHeavyChunk ..] (padded with n_pad), row hrow[c]; a row's chunks consecutive
  DevBuf hcol, hrow;
  uint32_t n_hchunks = 0;
  double hot_share = 0;   // share of gathers hitting the n/8 most-gathered vertices
  float build_ms = 0;
};

// Decides the layout (kLayoutAuto: relabel when the map vector is larger than
// ~1/3 of L2 and the n/8 hottest vertices take >= half of all gathers) and
// builds the storage-space CSRs with their heavy chunks and HYB slab.
// Returns false when the graph's plan for this layout was already built.
bool build_plan(const DevCsr& snap, const DevCsr& gath, int layout, MapPlan& plan, cudaStream_t s);

// Storage order by descending key (row lengths of key_off, n+1 offsets):
// orig[p] = vertex at position p (identity on the padding up to n_pad), perm = inverse.
void degree_order(const uint32_t* key_off, const uint32_t* tie_off, uint32_t n, uint32_t* orig, uint32_t* perm,
                  cudaStream_t s);
// `in` with rows and columns relabelled to storage order (out[perm[v]] = in[v]
// with columns mapped through perm); needs in's heavy-chunk list.
void relayout(const DevCsr& in, const uint32_t* orig, const uint32_t* perm, DevCsr& out, DevBuf& scratch,
              cudaStream_t s);
// Rows of g longer than kHeavyDeg as padded kHeavyChunk-column chunks (+ their rows).
void build_hslab(DevCsr& g, uint32_t np, DevBuf& hcol, DevBuf& hrow, uint32_t& n_hchunks, cudaStream_t s);
// Sliced ELL of g's rows [row_lo, row_hi) (multiples of 32) of at most
// kHeavyDeg edges; returns the slab's words.
uint64_t build_sell(const DevCsr& g, uint32_t row_lo, uint32_t row_hi, uint32_t np, DevBuf& sell, DevBuf& sdesc,
                    cudaStream_t s);

// dst bit p = src bit orig[p] for p < n (u32 words, dst has n_words words).
void permute_bits(const uint32_t* src, const uint32_t* orig, uint32_t n, uint32_t* dst, cudaStream_t s);

}  // namespace cyc
