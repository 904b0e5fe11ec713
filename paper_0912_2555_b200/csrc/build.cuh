// build.cuh — device CSR layout and the K1 build entry points.
#pragma once

#include "common.cuh"

namespace cyc {

constexpr uint32_t kRowPad = 256;  // row padding of map buffers and the HYB slab
constexpr uint32_t kHeavyDeg = 64;     // rows longer than this are split into chunks
constexpr uint32_t kHeavyChunk = 128;  // edges per heavy chunk (one warp, 4 per lane)

// One CSR on the device. Row offsets are u32 (n+1), columns u32 (m).
struct DevCsr {
  uint32_t n = 0;
  uint32_t m = 0;
  DevBuf off, col;
  DevBuf heavy;                 // uint4 {row, beg, end, 0} chunks of rows with deg > heavy_deg
  uint32_t n_heavy_chunks = 0;
  uint32_t heavy_deg = 0;
  uint32_t max_degree = 0;
  // HYB slab (gather side): the first ell_k columns of every row, column-major
  // (ell[k*n + v], kNone padded), and bit v of ovf = row v has more than ell_k.
  // Rows are padded to ell_n (a multiple of kRowPad); padding columns and
  // absent entries hold the sentinel ell_n, an always-NIL map slot.
  DevBuf ell, ovf;
  uint32_t ell_k = 0, ell_n = 0;
  const uint32_t* o() const { return off.as<uint32_t>(); }
  const uint32_t* c() const { return col.as<uint32_t>(); }
};

// Grow-only build temporaries owned by a context and reused by every build
// (pool allocations of several GB per build cost up to ~1 s of mapping).
struct BuildArena {
  DevBuf tmp, tmp2, raw, roff, ucnt, lists, counts, bcnt, bbase, bcur, scratch;
  DevBuf sp_row, sp_sub, sp_desc, sp_tmp;  // long-row split sort
  template <class T>
  T* get(DevBuf& b, size_t bytes, cudaStream_t s) {
    if (b.bytes < bytes) b.alloc(bytes + bytes / 8, s);
    return b.as<T>();
  }
};

int sm_count();
uint32_t grid_for(uint64_t items, int threads, int per_sm);
void exclusive_scan(const uint32_t* in, uint32_t* out, uint32_t n, uint32_t* total,
                    cudaStream_t s, DevBuf& scratch);
void build_csr(const uint32_t* d_edges, uint64_t m_log, uint32_t n, int key_dst, cudaStream_t s,
               DevCsr& out, uint32_t* d_err, BuildArena& ar);
// col_blocks > 1: chunks split at column-block boundaries and grouped by block
// (pull gathers stay within an L2-sized slice of the map vector).
void build_heavy(DevCsr& g, uint32_t heavy, uint32_t chunk, cudaStream_t s, uint32_t col_blocks = 1);
// Column blocks for the pull side of an n-vertex graph (1 when the map fits L2).
uint32_t pull_col_blocks(uint32_t n);
// Chooses ell_k in {1,2,4,8} minimising per-step pull bytes and builds the slab.
void build_ell(DevCsr& g, cudaStream_t s);

}  // namespace cyc
