/*
 * cyc_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the reference's MAP hot path
 * (/root/reference/proj/src/graph.cpp, src/map_engine.cpp). It is the checker
 * for the B200 library: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it. The product path never links or calls it.
 *
 * Pinned against (a) the SPEC.md [OP] known-answer examples and (b) the
 * reference itself, compiled from /root/reference by oracle/Makefile into
 * oracle/_ref/ (tests/test_oracle.py, tests/golden/).
 *
 * Conventions (reference types.hpp, map_engine.hpp:16-29, bitset.hpp):
 *   VertexId = uint32_t; map codes are id+1 with 0 = NIL;
 *   accepting sets are uint64_t words, bit v of word v>>6, tail bits zero.
 */
#ifndef CYC_ORACLE_H
#define CYC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cyo_csr {
  uint32_t n;
  uint64_t m;
  uint64_t* off; /* n + 1 */
  uint32_t* col; /* m */
} cyo_csr;

typedef struct cyo_map_stats {
  int cycle_found;
  uint32_t witness; /* valid iff cycle_found */
  uint64_t iterations;
  uint64_t kernel_calls;
  uint64_t demoted_total;
} cyo_map_stats;

void cyo_csr_free(cyo_csr* g);

/* build_snapshot (graph.cpp:63-105). edges = 2*m_log u32 (src,dst). Returns
 * -1 when an endpoint is >= n. */
int cyo_build_snapshot(const uint32_t* edges, uint64_t m_log, uint32_t n, int transposed,
                       cyo_csr* out);

/* Gather index of MaxPropagation (map_engine.cpp:9-19): the reverse relation. */
int cyo_transpose(const cyo_csr* g, cyo_csr* out);

/* Vertices of cyclic SCCs holding an accepting vertex (graph.cpp:125-196). */
void cyo_scc_keep_mask(const cyo_csr* g, const uint64_t* acc, uint8_t* keep);

/* restrict_to_accepting_sccs (graph.cpp:190-221). kept must hold n entries;
 * out_acc must hold (n+63)/64 words. */
int cyo_restrict(const cyo_csr* g, const uint64_t* acc, cyo_csr* out, uint64_t* out_acc,
                 uint32_t* kept, uint32_t* n_kept);

/* MaxPropagation::step (map_engine.cpp:21-79) on the gather index.
 * witness = UINT32_MAX when none. */
void cyo_step(const cyo_csr* gather, const uint32_t* x, const uint64_t* acc, uint32_t* out,
              int* changed, uint32_t* witness);

/* fixpoint (map_engine.cpp:94-121): values written to x (n entries), scratch
 * is n entries. Returns the step count. */
uint64_t cyo_fixpoint(const cyo_csr* gather, const uint64_t* acc, int early_exit, uint32_t* x,
                      uint32_t* scratch, uint32_t* witness);

/* demote (map_engine.cpp:123-137). remaining = (n+63)/64 words, demoted
 * receives |D| ascending ids (capacity n). Returns |D|. */
uint64_t cyo_demote(const uint32_t* x, uint32_t n, const uint64_t* acc, uint64_t* remaining,
                    uint32_t* demoted);

/* run_map (map_engine.cpp:139-162) plus the per-iteration evidence the
 * reference does not return: final_x (n entries, nullable) is the last
 * fixpoint vector, iter_hash[k] = cyo_vector_hash of iteration k's fixpoint
 * vector, iter_steps[k] its step count (both nullable, capacity cap). */
void cyo_run_map(const cyo_csr* gather, const uint64_t* acc, int early_exit, cyo_map_stats* st,
                 uint32_t* final_x, uint64_t* iter_hash, uint64_t* iter_steps, uint64_t cap);

/* owcty.cpp:14-87 — OWCTY over the rows of g (row u = successors of u):
 * approx = V; repeat { reach; elim } until empty or unchanged. witness =
 * min accepting survivor (0xFFFFFFFF when none), final_size = |approx|. */
void cyo_run_owcty(const cyo_csr* g, const uint64_t* acc, int* cycle, uint32_t* witness,
                   uint64_t* outer_iterations, uint64_t* final_size);

/* Order-independent 64-bit hash of a map vector (sum of mixed (v, x[v])). */
uint64_t cyo_vector_hash(const uint32_t* x, uint32_t n);

/* Edge log of a cyc_gen.h configuration (2*m entries) and its accepting words. */
int cyo_generate(const void* gen_params, uint32_t* edges, uint64_t* acc_words);
int cyo_gen_preset(int index, void* gen_params);
int cyo_gen_prepare(void* gen_params);

#ifdef __cplusplus
}
#endif

#endif
