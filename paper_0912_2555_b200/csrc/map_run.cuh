// map_run.cuh — workspace and launch interface of the persistent MAP loop.
#pragma once

#include "build.cuh"

namespace cyc {

// Frontier vertices whose push degree exceeds kBigDeg are expanded as chunks
// of kChunk edges by whole warps; the rest lane by lane from the bitmap.
constexpr uint32_t kBigDeg = 32;
constexpr uint32_t kChunk = 128;

// Per-step counters.
struct alignas(64) SlotCtl {
  unsigned long long fedges;  // push degrees of the vertices first raised in the step
  unsigned int nraised;       // vertices raised
  unsigned int changed;
  unsigned int nchunk;        // big-vertex chunks enlisted for the next step; bit 31: a CTA's list
                              // overflowed, the next push step re-chunks the frontier (kChunkOver)
  unsigned int cand_cnt;      // self-witness candidates
  unsigned int wit;           // exact min self-witness (pull rows)
  unsigned int wl_count;      // frontier words listed for the next push step
  unsigned int wl_over;       // the list is incomplete: scan the bitmap instead
  unsigned int light_next;    // pull steps on a plan: next unclaimed light slice (dynamic distribution)
  unsigned int heavy_next;    // ... and heavy-slab chunks claimed beyond every warp's first unit
};
constexpr unsigned int kChunkOver = 0x80000000u;

// Control block of one k_map_run launch. Per-step counters rotate over three
// slots (step g writes slot g%3, reads slot (g-1)%3, and clears slot (g+1)%3),
// per-iteration counters over two.
struct RunCtl {
  SlotCtl slot[3];
  unsigned long long it_hash[2];
  unsigned int it_finwit[2];
  unsigned int it_dcount[2];
  unsigned long long it_fsize[2];
  unsigned int it_vmax[2];        // per fixpoint (parity): max over F of id+1, the largest possible map value
  unsigned long long res[16];
};

enum RunRes {
  kResCycle = 0, kResWitness, kResIterations, kResKernelCalls, kResDemoted, kResStepsLast,
  kResPullSteps, kResPushSteps, kResEdges, kResRows, kResBytes, kResCur, kResTag, kResBars, kResRaised
};

// Row-sharded runs (world > 1, shard.cu): every rank keeps the whole map vector
// and frontier bitmaps replicated, computes the rows [row_lo, row_hi) of each
// step and stores the changed ones straight into every peer's buffers (NVLink
// peer pointers); per-step records are reduced by every rank after a
// cross-rank barrier, so all ranks take the same decisions.
constexpr int kMaxWorld = 8;

struct alignas(32) ShardRec {
  unsigned long long fedges;  // push degrees of the rank's newly raised vertices (local push rows)
  unsigned int nraised, changed, wit, pad;
};

struct RunArgs {
  uint32_t n, m;
  const uint32_t* goff;  // gather index (pull): row v = sources flowing into v
  const uint32_t* gcol;
  const uint32_t* poff;  // snapshot relation (push): row u = targets u flows into
  const uint32_t* pcol;
  const uint32_t* bigm;  // bit v: push degree of v > kBigDeg
  const uint32_t* ell;   // HYB slab of the gather index (column-major, ell_k wide)
  const uint32_t* ovf;   // bit v: gather row v is longer than ell_k (or heavy)
  uint32_t ell_k;
  const uint4* sdesc;    // sliced ELL of a degree-ordered plan: {off/32, width, heavy rows mask, 0} per 32 rows
  const uint32_t* sell;  //   (null: HYB slab above)
  const uint32_t* hcol;  // heavy rows of a plan as padded 128-column chunks (null: `heavy` below)
  const uint32_t* hrow;  //   row of each chunk
  uint32_t n_hchunks;
  uint32_t hot_k;        // positions [0, hot_k) whose frontier bits pull steps stage in shared memory
  uint32_t n_pad;        // rows padded to kRowPad; P[n_pad] is the NIL sentinel slot
  const uint4* heavy;    // gather rows longer than heavy_deg, split into chunks
  uint32_t n_heavy, heavy_deg;
  uint32_t* P[2];                  // packed map words: accepting<<31 | code
  uint32_t* FB[2];                 // frontier bitmaps: vertices changed in the step
  uint32_t* WL[2];                 // frontier word lists (non-zero FB words of the step)
  uint32_t wl_cap;
  uint4* BC[2];                    // frontier chunks {v, beg, end} of big-degree vertices
  uint32_t* C[2];                  // self-witness candidates
  uint32_t* F;                     // accepting set, u32 words (demoted in place)
  uint32_t* used;                  // scratch bitmap, zero between iterations
  const uint32_t* orig;            // storage position -> vertex id (null: identity layout, plan.cuh)
  const uint32_t* perm;            // vertex id -> storage position (null: identity)
  uint32_t nwords, nwords_pad;     // FB words for n and for the padded rows
  uint32_t chunk_cap;
  uint32_t cand_cap;               // capacity of C[k]
  RunCtl* ctl;
  unsigned long long* iter_hash;
  unsigned long long* iter_steps;
  unsigned long long cap;
  unsigned long long max_iterations, max_steps;
  unsigned long long* trace;       // optional per-step record {mode|step, edges, raised, clock}
  uint32_t trace_cap;
  uint32_t alpha;
  int early_exit, mode;
  // -- this rank's part of the grid and of the rows (single GPU: the whole grid, all rows)
  uint32_t blk0, nblk;
  int world, rank, emulated;       // emulated: all ranks share one grid on one GPU (tests)
  uint32_t row_lo, row_hi;
  uint32_t* peerP[kMaxWorld][2];
  uint32_t* peerFB[kMaxWorld][2];
  ShardRec* rec;                   // [2][kMaxWorld]: step records written by every rank
  ShardRec* peerRec[kMaxWorld];
  unsigned long long* bar;         // cross-rank barrier counter, incremented by every rank
  unsigned long long* peerBar[kMaxWorld];
  unsigned long long bar_base;     // barriers completed by earlier runs
};

struct RunWs {
  uint32_t n = 0, m = 0, n_pad = 0;
  DevBuf P[2], FB[2], WL[2], BC[2], C[2], F, used, bigm, ctl, hist, trace;
  uint32_t wl_cap = 0;
  uint32_t chunk_cap = 0;
  uint32_t trace_len = 0;
  const uint32_t* orig = nullptr;  // layout of the last run (plan.cuh); strip_codes maps back
  const uint32_t* bigm_src = nullptr;  // push offsets bigm was computed from
  void ensure(uint32_t n, uint32_t m, const uint32_t* poff, cudaStream_t s);
};

struct RunOut {
  unsigned long long res[16];
  float ms;
  uint32_t grid, block;
  double plan_ms = 0;
  int layout = 1;
};

// Runs the device-resident MAP loop. F must already hold the accepting words.
// snap/gath are in storage order; orig/perm describe it (null: identity).
void launch_map_run(const DevCsr& snap, const DevCsr& gath, const uint32_t* orig, const uint32_t* perm,
                    const uint4* sdesc, const uint32_t* sell, const uint32_t* hcol, const uint32_t* hrow,
                    uint32_t n_hchunks, RunWs& ws, int early_exit, int mode,
                    unsigned long long max_iterations, unsigned long long max_steps,
                    uint32_t alpha, unsigned long long cap, uint32_t trace_cap, cudaStream_t s,
                    cudaEvent_t e0, cudaEvent_t e1, RunOut& out);

// One rank of a sharded run as seen by the launcher (shard.cu fills it).
struct ShardRunIn {
  int device;
  cudaStream_t s;
  const DevCsr* push;  // push rows restricted to this rank's targets
  const DevCsr* gath;  // this rank's gather rows
  const uint32_t* orig;
  const uint32_t* perm;
  const uint4* sdesc;
  const uint32_t* sell;
  const uint32_t* hcol;
  const uint32_t* hrow;
  uint32_t n_hchunks;
  RunWs* ws;
  uint32_t* P[2];
  uint32_t* FB[2];
  const uint32_t* bigm;  // push degree > kBigDeg over this rank's push rows
  uint32_t n;
  uint64_t m_global;
  int world, rank;
  uint32_t row_lo, row_hi;
  uint32_t* peerP[kMaxWorld][2];
  uint32_t* peerFB[kMaxWorld][2];
  ShardRec* rec;
  ShardRec* peerRec[kMaxWorld];
  unsigned long long* bar;
  unsigned long long* peerBar[kMaxWorld];
  unsigned long long bar_base;
};

// Runs the k ranks of this process: one cooperative grid per device (they
// meet at system-scope barriers), or, emulated, all k ranks in one grid on one
// device (tests). outs[i].res[kResBars] = barriers completed (next bar_base).
void launch_map_run_shards(ShardRunIn* in, int k, bool emulated, int early_exit, int mode,
                           unsigned long long max_iterations, unsigned long long max_steps, uint32_t alpha,
                           unsigned long long cap, RunOut* outs);

// Writes the codes (flag bit stripped) of workspace buffer `cur` into dst,
// in vertex-id order (ws.orig set: dst[orig[p]] = code of position p).
void strip_codes(const RunWs& ws, int cur, uint32_t n, uint32_t* dst, cudaStream_t s);

// Dense single Jacobi step (MaxPropagation::step) on plain codes.
void launch_step_pull(const DevCsr& gath, const uint32_t* x, const uint32_t* accw, uint32_t* out,
                      uint32_t* flags, cudaStream_t s);

// Dense step over rows [lo, hi) only (sharded runs): rec = {changed,
// UINT32_MAX - min witness} as int64 (MAX-reducible); no-op when state[0].
void launch_step_range(const DevCsr& gath, uint32_t lo, uint32_t hi, const uint32_t* x,
                       const uint32_t* accw, uint32_t* out, long long* rec, const long long* state,
                       int first_only, cudaStream_t s);
// Sparse exchange: changed rows of [lo, hi) into sp (sp[0] = count) and the
// post step applying every rank's changes (or flagging overflow).
void launch_shard_collect(uint32_t lo, uint32_t hi, const uint32_t* x, const uint32_t* out, uint32_t cap,
                          uint2* sp, const long long* state, int list_mode, const uint32_t* rlist,
                          const uint32_t* rcnt, uint32_t* rbits, const uint32_t* accw, long long* rec,
                          cudaStream_t s);
void launch_shard_push(const uint2* sp_all, int world, uint32_t cap, const DevCsr& snap, uint32_t lo, uint32_t hi,
                       const uint32_t* accw, uint32_t* out, uint32_t* rbits, uint32_t* rlist, uint32_t* rcnt,
                       const long long* state, cudaStream_t s);
void launch_shard_post_sparse(const long long* rec, long long* state, const uint2* sp_all, int world,
                              uint32_t cap, uint32_t* x, cudaStream_t s);
// Unpads the gathered slices into x and advances the sharded fixpoint state.
void launch_shard_post(const long long* rec, long long* state, const uint32_t* x_pad,
                       const uint32_t* bounds, int world, uint32_t maxrows, uint32_t* x, cudaStream_t s);
// Device-only demotion for sharded runs: counts[0] = |D|, counts[1] = |F'|.
void launch_demote_async(const uint32_t* x, uint32_t n, const uint32_t* accw, uint32_t* remaining,
                         unsigned long long* counts, uint32_t* used_scratch, cudaStream_t s);

// demote(): remaining = F & ~used(x); demoted ascending; returns |D| on host.
uint64_t run_demote(const uint32_t* x, uint32_t n, const uint32_t* accw, uint32_t* remaining,
                    uint32_t* demoted, cudaStream_t s);

}  // namespace cyc
