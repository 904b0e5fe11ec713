/*
 * cycheck_b200.h — C ABI of the B200-native MAP accepting-cycle engine.
 *
 * Drop-in boundary for the reference's MAP hot path
 * (/root/reference/proj/include/cycheck/{graph,map_engine}.hpp). The
 * reference exposes a C++ value API with exceptions; this ABI uses opaque
 * handles, plain pointers, sizes and status codes. Every pointer argument
 * may be host memory (pageable or pinned) or device memory of the context's
 * GPU; the library detects which and copies host data inside the call.
 *
 * Status codes map onto the reference's exceptions (errors.hpp:10-22):
 *   CYC_E_CONTRACT  -> cycheck::ContractError      (precondition broken)
 *   CYC_E_RESOURCE  -> cycheck::ResourceLimitError (capacity / device OOM)
 *   CYC_E_CUDA      -> runtime failure (CUDA / NCCL error)
 *   CYC_E_PARSE     -> cycheck::ParseError (message = ParseError::what(),
 *                      code/line/col via cyc_last_parse_error)
 * cyc_last_error() returns the calling thread's last message.
 *
 * Conventions (reference types.hpp:9, map_engine.hpp:16-29, bitset.hpp:12-72):
 *   vertex ids are uint32_t; map values are codes id+1 with 0 = NIL;
 *   vertex sets are uint64_t words, bit v in word v>>6, tail bits zero.
 *   Limits of this engine: n < 2^31, snapshot edges m < 2^32.
 */
#ifndef CYCHECK_B200_H
#define CYCHECK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum cyc_status {
  CYC_OK = 0,
  CYC_E_CONTRACT = 1,
  CYC_E_RESOURCE = 2,
  CYC_E_CUDA = 3,
  CYC_E_INVALID = 4,
  CYC_E_PARSE = 5
} cyc_status;

/* reference types.hpp:12 `enum class Orientation { forward, transposed }` */
enum { CYC_FORWARD = 0, CYC_TRANSPOSED = 1 };

/* Propagation step selection inside the device loop. */
enum { CYC_MODE_AUTO = 0, CYC_MODE_PULL = 1, CYC_MODE_PUSH = 2 };

typedef struct cyc_ctx cyc_ctx;
typedef struct cyc_graph cyc_graph;

/* reference map_engine.hpp:33-36 MapOptions {workers, early_exit}; `workers`
 * has no meaning on the GPU (results are worker-count invariant). */
typedef struct cyc_map_options {
  int32_t early_exit;      /* default 1 */
  int32_t mode;            /* CYC_MODE_* (default AUTO) */
  uint64_t max_iterations; /* 0 = run to verdict (run_map); 1 = one fixpoint */
  uint64_t max_steps;      /* 0 = unbounded; else stop the first fixpoint after k steps */
  uint32_t push_alpha;     /* push when frontier edges * alpha < m (0 = default 16) */
  uint32_t trace_cap;      /* > 0: record up to this many steps (cyc_map_trace) */
  int32_t layout;          /* CYC_LAYOUT_*: storage order of the map vector (default AUTO) */
  int32_t reserved;
} cyc_map_options;

/* Storage order of the map vector and CSRs inside run_map (results are the
 * same in every layout). DEGREE stores vertices by descending gather count so
 * the hot words of a power-law graph share L2 sectors; AUTO picks it when the
 * vector is larger than ~1/3 of L2 and the n/8 most-gathered vertices take at
 * least half of the gathers. The plan is built once per graph and layout. */
#define CYC_LAYOUT_AUTO 0
#define CYC_LAYOUT_IDENTITY 1
#define CYC_LAYOUT_DEGREE 2

/* reference map_engine.hpp:101-106 MapStats + types.hpp:18-27 Verdict, plus
 * device-side evidence for the roofline. */
typedef struct cyc_map_stats {
  int32_t cycle_found;
  uint32_t witness;            /* valid iff cycle_found; cyc_check maps it back to the
                                  log's ids when it restricted (explore.cpp:117-118) */
  uint64_t iterations;
  uint64_t kernel_calls;
  uint64_t demoted_total;
  uint64_t steps_last;         /* steps of the last fixpoint */
  uint64_t pull_steps, push_steps;
  uint64_t edges_touched;      /* sum over steps of edges read */
  uint64_t rows_touched;       /* sum over steps of rows processed */
  uint64_t algorithmic_bytes;  /* sum over steps of 8*E_s + 12*V_s */
  double loop_ms;              /* device time of the loop kernel(s), CUDA events */
  uint32_t grid_blocks, block_threads;
  double plan_ms;              /* host time building the storage plan in this call (0: cached) */
  int32_t layout;              /* CYC_LAYOUT_IDENTITY or CYC_LAYOUT_DEGREE: the layout that ran */
  int32_t world;               /* ranks of a sharded run (1: one device) */
  uint64_t exchanged_rows;     /* sharded: rows every rank stored into each peer, over all steps */
} cyc_map_stats;

/* ---- context ------------------------------------------------------------ */
cyc_status cyc_ctx_create(int device, cyc_ctx** out);
void cyc_ctx_destroy(cyc_ctx* ctx);
const char* cyc_last_error(void);
/* Number of kernels this process has launched through the library. */
uint64_t cyc_launch_count(void);
cyc_status cyc_ctx_synchronize(cyc_ctx* ctx);
/* The CUDA stream (cudaStream_t) every call of this context is ordered on. */
void* cyc_ctx_stream(cyc_ctx* ctx);
/* external != 0: order the context on `stream` (e.g. the stream NCCL / torch
 * work is issued on; 0 is the legacy default stream); external == 0 restores
 * the context's own stream. */
cyc_status cyc_ctx_set_stream(cyc_ctx* ctx, void* stream, int external);
/* Allocate the device memory a build_snapshot (+ storage plan) of a log of
 * up to m_log edges over n vertices uses, now: first touch of device memory
 * runs at ~150 GB/s, ~0.4 s of a 2^30-edge log's first call. background != 0:
 * on a library thread, while the caller loads its log; the next build (or
 * reserve, or destroy) waits for it. Not a limit: builds still allocate what
 * they need; memory the reserve cannot get is simply not reserved. */
cyc_status cyc_ctx_reserve(cyc_ctx* ctx, uint64_t m_log, uint32_t n, int background);

/* ---- graph (reference graph.hpp:27-42 CsrSnapshot) ---------------------- */
/* build_snapshot (graph.hpp:97-98, graph.cpp:63-105): edges = 2*m_log u32
 * (src,dst) pairs of the logged prefix; acc_words = accepting flags of the n
 * vertices (EdgeLog::accepting_prefix, graph.cpp:206-213), may be NULL.
 * Duplicates are removed and rows sorted. Builds both the snapshot relation
 * and its reverse (the MaxPropagation gather index, map_engine.cpp:9-19). */
cyc_status cyc_graph_build(cyc_ctx* ctx, const uint32_t* edges, uint64_t m_log, uint32_t n,
                           const uint64_t* acc_words, int orientation, cyc_graph** out);
/* Device copy of an already-built snapshot (reference CsrSnapshot layout:
 * row_offsets n+1 u64, col_indices m u32 sorted per row, accepting words):
 * the entry point for callers that hold a CsrSnapshot (run_map takes one,
 * map_engine.hpp:111). The gather index is derived on the device. */
cyc_status cyc_graph_from_csr(cyc_ctx* ctx, const uint64_t* row_offsets, const uint32_t* col_indices,
                              uint32_t n, uint64_t m, const uint64_t* acc_words, int orientation,
                              cyc_graph** out);
/* Incremental snapshot: the snapshot of the log prefix
 * (m_prev + m_new edges, n vertices) from `prev` — the snapshot of the prefix
 * (m_prev, prev n) — and only the new edges new_edges[0 .. 2*m_new) (log
 * order, host or device). Equal, bit for bit, to cyc_graph_build on the whole
 * prefix (graph.cpp:63-105), which the explorer's detector does every round
 * (explore.cpp:71-124). n >= prev's n; acc_words = accepting prefix of n
 * (NULL: prev's bits, new vertices not accepting). prev must not be
 * restricted; orientation is prev's. */
cyc_status cyc_graph_extend(cyc_ctx* ctx, const cyc_graph* prev, const uint32_t* new_edges, uint64_t m_new,
                            uint32_t n, const uint64_t* acc_words, cyc_graph** out);
/* Logged-edge prefix length a snapshot was built from (m_prev for extend). */
cyc_status cyc_graph_log_prefix(const cyc_graph* g, uint64_t* m_log);
/* restrict_to_accepting_sccs (graph.hpp:103-114, graph.cpp:190-221). */
cyc_status cyc_graph_restrict(cyc_ctx* ctx, const cyc_graph* in, cyc_graph** out);
void cyc_graph_destroy(cyc_graph* g);
cyc_status cyc_graph_info(const cyc_graph* g, uint32_t* n, uint64_t* m, int* orientation,
                          int* restricted);
/* Copies out the snapshot CSR: row_offsets (n+1 u64), col_indices (m u32),
 * accepting (ceil(n/64) u64), kept (n u32, restricted graphs only). Any
 * pointer may be NULL. */
cyc_status cyc_graph_export(const cyc_graph* g, uint64_t* row_offsets, uint32_t* col_indices,
                            uint64_t* acc_words, uint32_t* kept);
/* Copies out the gather index (reverse relation) in the same layout. */
cyc_status cyc_graph_export_gather(const cyc_graph* g, uint64_t* row_offsets,
                                   uint32_t* col_indices);

/* ---- map engine (reference map_engine.hpp:50-112) ----------------------- */
/* MaxPropagation::step (map_engine.cpp:21-79): out = step(x); witness =
 * UINT32_MAX when none. acc_words NULL = the snapshot's accepting set. */
cyc_status cyc_map_step(cyc_ctx* ctx, const cyc_graph* g, const uint64_t* acc_words,
                        const uint32_t* x, uint32_t* out, int32_t* changed, uint32_t* witness);
/* fixpoint (map_engine.cpp:94-121). values: n codes (nullable). */
cyc_status cyc_fixpoint(cyc_ctx* ctx, const cyc_graph* g, const uint64_t* acc_words,
                        const cyc_map_options* opt, uint32_t* values, uint64_t* steps,
                        uint32_t* witness);
/* demote (map_engine.cpp:123-137): remaining = F \ D (words), demoted = D
 * ascending (capacity n, nullable); returns |D| in n_demoted. */
cyc_status cyc_demote(cyc_ctx* ctx, const uint32_t* values, uint32_t n,
                      const uint64_t* acc_words, uint64_t* remaining, uint32_t* demoted,
                      uint64_t* n_demoted);
/* run_map (map_engine.cpp:139-162). final_values (n codes, nullable) = the
 * last fixpoint vector; iter_hash / iter_steps (nullable, capacity cap) =
 * per-iteration vector hash (sum of splitmix64((v<<32)|x[v])) and steps. */
cyc_status cyc_map_run(cyc_ctx* ctx, const cyc_graph* g, const uint64_t* acc_words,
                       const cyc_map_options* opt, cyc_map_stats* stats, uint32_t* final_values,
                       uint64_t* iter_hash, uint64_t* iter_steps, uint64_t cap);

/* Per-step record of the graph's last loop run with trace_cap > 0: 64 u64 per
 * step (index = step tag - 2): [0] = mode << 60 | input chunks << 24 | step in
 * fixpoint, [1] frontier edges, [2] raised, [3] t_start, [7] t_end, [16..64)
 * = 16 spread slots each of t_phase0, t_phase1, t_flags (globaltimer ns, the
 * latest any warp reached that point; take the max over the slots). */
cyc_status cyc_map_trace(const cyc_graph* g, uint64_t* out, uint32_t cap, uint32_t* len);

/* scc_verdict (reference oracle.cpp:32-98) on the device: cycle iff some
 * accepting vertex lies in a cyclic SCC; cyclic_accepting (nullable,
 * capacity n) receives those vertices ascending, witness the smallest. An
 * independent verdict at scales the reference's Tarjan cannot reach. */
cyc_status cyc_scc_verdict(cyc_ctx* ctx, const cyc_graph* g, int32_t* cycle, uint32_t* witness,
                           uint32_t* cyclic_accepting, uint64_t* count);

/* run_owcty (reference owcty.hpp:12-31, owcty.cpp:56-87) on the device over
 * the snapshot relation (the reference runs it on a forward snapshot,
 * cycheck_main.cpp:98-106): alternate proper reachability from accepting
 * vertices and in-degree-0 elimination until the set is empty or unchanged.
 * witness = min accepting survivor (UINT32_MAX when none). acc_words NULL =
 * the snapshot's accepting set. */
typedef struct cyc_owcty_stats {
  uint64_t outer_iterations;
  uint64_t final_size;
  double reach_ms;
  double elim_ms;
} cyc_owcty_stats;
cyc_status cyc_owcty(cyc_ctx* ctx, const cyc_graph* g, const uint64_t* acc_words, int32_t* cycle,
                     uint32_t* witness, cyc_owcty_stats* stats);

/* ---- explicit-graph ingestion ---------------------------- */
/* ExplicitGraph (graph.hpp:136-150) on the device. */
typedef struct cyc_explicit cyc_explicit;
/* parse_explicit_graph (graph.cpp:259-297) of `len` bytes of text (host or
 * device): "graph <n>", "accepting <id>...", "edge <src> <dst>" lines, '#'
 * comments. On malformed input returns CYC_E_PARSE with the reference's
 * ParseError text ("<line>:<col>: error[syntax|range]: ...") for the same
 * first offending line. */
cyc_status cyc_explicit_parse(cyc_ctx* ctx, const char* text, uint64_t len, cyc_explicit** out);
/* Binary edge list: "CYCGRAPH", u32 version = 1, u32 n, u64 m, u64 accepting
 * words[ceil(n/64)], u32 edges[2m] (log order) — one file feeds the reference
 * (oracle/ref_driver.cpp) and the device without text parsing. */
cyc_status cyc_explicit_load_binary(cyc_ctx* ctx, const void* data, uint64_t len, cyc_explicit** out);
/* DiagCode (errors.hpp:21-28), line, column of the last CYC_E_PARSE. */
cyc_status cyc_last_parse_error(int* code, int* line, int* col);
cyc_status cyc_explicit_info(const cyc_explicit* g, uint32_t* n, uint64_t* n_accepting, uint64_t* m);
/* accepting ids (file order; ascending for binary input) and edges (2m u32). */
cyc_status cyc_explicit_export(const cyc_explicit* g, uint32_t* accepting, uint32_t* edges);
/* fill_log (graph.cpp:305-310) + build_snapshot on the device. */
cyc_status cyc_explicit_snapshot(cyc_ctx* ctx, const cyc_explicit* g, int orientation, cyc_graph** out);
void cyc_explicit_destroy(cyc_explicit* g);

/* ---- one-call pipeline: edge log -> verdict ----------------------------- */
/* cycheck graph / explore final round (cycheck_main.cpp:88-97,
 * explore.cpp:71-124): build_snapshot [+ restrict] + run_map. Timings in
 * ms_out[4] = {h2d+build, restrict, loop, total} (nullable). */
cyc_status cyc_check(cyc_ctx* ctx, const uint32_t* edges, uint64_t m_log, uint32_t n,
                     const uint64_t* acc_words, int orientation, int scc_restrict,
                     const cyc_map_options* opt, cyc_map_stats* stats, double* ms_out);

/* ---- row-sharded run_map over several GPUs ----------------- */
/* A shard is one rank's part of a graph: from the whole edge log it keeps
 * the gather rows of an edge-balanced contiguous row range (the reference's
 * worker partition, map_engine.cpp:35-43) and the push rows that target them,
 * so a rank's edge memory is ~1/world. The map vector is replicated; in every
 * step each rank stores the rows it changed straight into every peer's vector
 * (NVLink peer memory) and the ranks meet at a system-scope barrier inside
 * one persistent kernel each. Results equal run_map on the whole graph.
 * Ranks in different processes connect by exchanging cyc_shard_handle()
 * blobs (e.g. an allgather); ranks in one process with cyc_shard_connect_local
 * (one context per device; ranks that share a device run as one grid, for
 * tests). layout: CYC_LAYOUT_* as in cyc_map_options. */
typedef struct cyc_shard cyc_shard;
#define CYC_SHARD_HANDLE_BYTES 512
cyc_status cyc_shard_build(cyc_ctx* ctx, const uint32_t* edges, uint64_t m_log, uint32_t n,
                           const uint64_t* acc_words, int orientation, int layout, int world, int rank,
                           cyc_shard** out);
/* rows [row_lo, row_hi) in storage order; local snapshot edges; device bytes
 * of the rank's graph structures (edges ~1/world, vectors replicated). */
cyc_status cyc_shard_info(const cyc_shard* sh, uint32_t* row_lo, uint32_t* row_hi, uint64_t* local_edges,
                          uint64_t* device_bytes);
cyc_status cyc_shard_handle(const cyc_shard* sh, void* out);
/* handles: world blobs of CYC_SHARD_HANDLE_BYTES, in rank order */
cyc_status cyc_shard_connect(cyc_shard* sh, const void* handles);
cyc_status cyc_shard_connect_local(cyc_shard* const* shards, int world);
/* run_map (map_engine.cpp:139-162) on the `count` ranks this process holds
 * (1 per process, or all of them after cyc_shard_connect_local); every rank's
 * stats are the whole graph's; final_values / iter_* from shards[0]'s replica. */
cyc_status cyc_shard_run_map(cyc_shard* const* shards, int count, const uint64_t* acc_words,
                             const cyc_map_options* opt, cyc_map_stats* stats, uint32_t* final_values,
                             uint64_t* iter_hash, uint64_t* iter_steps, uint64_t cap);
void cyc_shard_destroy(cyc_shard* sh);

/* ---- synthetic inputs and buffers (bench / tests) ----------------------- */
/* Generates a cyc_gen.h configuration's edge log and accepting words into
 * device or host buffers (edges: 2*m u32, acc: ceil(n/64) u64). */
cyc_status cyc_gen_fill(cyc_ctx* ctx, const void* gen_params, uint32_t* edges,
                        uint64_t* acc_words);
cyc_status cyc_gen_preset(int index, void* gen_params);
cyc_status cyc_gen_prepare(void* gen_params);
cyc_status cyc_host_alloc(size_t bytes, void** out);      /* pinned */
void cyc_host_free(void* p);
cyc_status cyc_device_alloc(cyc_ctx* ctx, size_t bytes, void** out);
void cyc_device_free(cyc_ctx* ctx, void* p);
/* Copy ordered on the context's stream, returns without waiting (pair with
 * cyc_ctx_synchronize); either side may be host (pinned for overlap) or device. */
cyc_status cyc_memcpy_async(cyc_ctx* ctx, void* dst, const void* src, size_t bytes);
cyc_status cyc_memcpy(cyc_ctx* ctx, void* dst, const void* src, size_t bytes);
/* Writes `bytes` of a scratch buffer to evict L2 (timing hygiene). */
cyc_status cyc_flush_l2(cyc_ctx* ctx, size_t bytes);

/* ---- multi-GPU row sharding (one process per GPU) ------------------------ */
/* Device-side state of one sharded fixpoint (int64[8], device memory):
 * [0] done, [1] steps taken, [2] witness (UINT32_MAX = none), [3] early_exit,
 * [4] blocked by a sparse step that overflowed, [5] largest per-rank change
 * count seen, [6..7] that step's reduced record (for its dense completion).
 * Every rank holds an identical copy; all updates happen on the device from
 * all-reduced records, so ranks stay in lockstep without host syncs. */
/* One Jacobi step (MaxPropagation::step) restricted to rows [lo, hi) of the
 * gather index: out[v - lo] for v in the range, from the full replicated
 * vector x (n codes, device) and accepting words (device). rec (device
 * int64[2]) receives {changed, UINT32_MAX - min self-witness} (MAX-reducible;
 * 0 = no witness). A no-op when state[0] (done) or state[4] (blocked) is
 * set, and with first_only (sparse protocol) after the fixpoint's first step,
 * which cyc_shard_push then takes. Asynchronous on the context's stream (no
 * host sync), for use between collectives. */
cyc_status cyc_shard_step(cyc_ctx* ctx, const cyc_graph* g, uint32_t lo, uint32_t hi,
                          const uint32_t* x, const uint64_t* acc_words, uint32_t* out,
                          int64_t* rec, const int64_t* state, int first_only);
/* After the all-gather of the padded slices (x_pad: world * maxrows codes)
 * and the MAX all-reduce of rec: x[bounds[r] + i] = x_pad[r*maxrows + i]
 * (bounds: device u32[world+1]) and, unless done, state advances: steps++,
 * and the fixpoint ends (done, witness) on a witness with early_exit or on
 * no change (map_engine.cpp:94-121). Asynchronous. */
cyc_status cyc_shard_post(cyc_ctx* ctx, const int64_t* rec, int64_t* state, const uint32_t* x_pad,
                          const uint32_t* bounds, int world, uint32_t maxrows, uint32_t* x);
/* Sparse (changed-only) exchange: after cyc_shard_step, the
 * rank's changed rows (out[v-lo] != x[v]) as (v, value) pairs into sp
 * (uint2[cap+1], sp[0] = {count, 0}); after an all-gather of every rank's sp
 * (sp_all = world x (cap+1) uint2) and the MAX all-reduce of rec,
 * cyc_shard_post_sparse applies all changes and advances state, or — if some
 * rank changed more than cap rows — blocks the rest of the batch (state[4])
 * so the host completes that step with the dense exchange. */
cyc_status cyc_shard_collect(cyc_ctx* ctx, uint32_t lo, uint32_t hi, const uint32_t* x, const uint32_t* out,
                             uint32_t cap, uint32_t* sp, const int64_t* state, int list_mode,
                             const uint32_t* rlist, const uint32_t* rcnt, uint32_t* rbits,
                             const uint64_t* acc_words, int64_t* rec);
/* Frontier (push) step of the sparse protocol, steps after the first: from
 * every rank's changes of the previous step (sp_all, already applied to x),
 * raise this rank's targets in out (= x's slice) along the snapshot rows;
 * raised rows go to rlist (local indices, count rcnt, dedup bitmap rbits of
 * (hi-lo)/32+1 words, all device memory) for cyc_shard_collect(list_mode=1),
 * which also produces the step record. Early-exit runs only. */
cyc_status cyc_shard_push(cyc_ctx* ctx, const cyc_graph* g, uint32_t lo, uint32_t hi, const uint32_t* sp_all,
                          int world, uint32_t cap, const uint64_t* acc_words, uint32_t* out, uint32_t* rbits,
                          uint32_t* rlist, uint32_t* rcnt, const int64_t* state);
cyc_status cyc_shard_post_sparse(cyc_ctx* ctx, const int64_t* rec, int64_t* state, const uint32_t* sp_all,
                                 int world, uint32_t cap, uint32_t* x);
/* used-bitmap demotion on a full replicated vector, entirely on device:
 * remaining = F \ D (words, device), counts[0] = |D|, counts[1] = |F'|
 * (device u64[2]); asynchronous. */
cyc_status cyc_shard_demote(cyc_ctx* ctx, const uint32_t* x, uint32_t n, const uint64_t* acc_words,
                            uint64_t* remaining, uint64_t* counts);
/* Fused exchange: one persistent kernel per rank runs the whole
 * run_map for rows [lo, hi) and stores every new row value straight into all
 * ranks' replicated vectors over peer memory (CUDA IPC / NVLink) as it is
 * computed; a system-scope barrier per step replaces the collectives.
 * open: allocates the rank's shared block, writes its 64-byte IPC handle;
 * connect: all ranks' handles in rank order (world x 64 bytes); run: every
 * rank calls it with the same accepting words and early_exit; stats and the
 * final vector (n codes, nullable) equal run_map's. */
typedef struct cyc_fused cyc_fused;
cyc_status cyc_fused_open(cyc_ctx* ctx, const cyc_graph* g, uint32_t lo, uint32_t hi, int rank, int world,
                          cyc_fused** out, void* handle_out);
cyc_status cyc_fused_connect(cyc_fused* f, const void* handles);
cyc_status cyc_fused_run(cyc_fused* f, const uint64_t* acc_words, int early_exit, cyc_map_stats* st,
                         uint32_t* final_values);
void cyc_fused_close(cyc_fused* f);
/* Edge-balanced contiguous row ranges, the reference's worker partition rule
 * (map_engine.cpp:35-43): bounds[r] for r in [0, parts], computed on the
 * host from gather row offsets (n+1 u64). */
cyc_status cyc_shard_bounds(const uint64_t* row_offsets, uint32_t n, int parts, uint32_t* bounds);

#ifdef __cplusplus
}
#endif

#endif /* CYCHECK_B200_H */
