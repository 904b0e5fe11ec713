/*
 * cyc_oracle.c — TEST INFRASTRUCTURE ONLY (see cyc_oracle.h).
 *
 * Plain-C restatement of the reference MAP path. Each function cites the
 * reference lines it follows; the algorithms are restated, not transcribed.
 */
#include "cyc_oracle.h"

#include <stdlib.h>
#include <string.h>

#include "../include/cyc_gen.h"

static int acc_test(const uint64_t* acc, uint32_t v) { return (int)((acc[v >> 6] >> (v & 63)) & 1u); }

void cyo_csr_free(cyo_csr* g) {
  if (!g) return;
  free(g->off);
  free(g->col);
  g->off = NULL;
  g->col = NULL;
  g->n = 0;
  g->m = 0;
}

static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

/* graph.cpp:63-105 — counting sort of the logged prefix by row key (dst for
 * the transposed orientation, src for forward), then every row sorted
 * ascending with adjacent duplicates dropped. */
int cyo_build_snapshot(const uint32_t* edges, uint64_t m_log, uint32_t n, int transposed,
                       cyo_csr* out) {
  memset(out, 0, sizeof *out);
  for (uint64_t i = 0; i < 2 * m_log; ++i)
    if (edges[i] >= n) return -1;
  uint64_t* start = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  uint32_t* bucket = (uint32_t*)malloc((m_log ? m_log : 1) * sizeof(uint32_t));
  uint64_t* fill = (uint64_t*)malloc(((size_t)n + 1) * sizeof(uint64_t));
  const int key = transposed ? 1 : 0; /* which half of the pair is the row */
  for (uint64_t i = 0; i < m_log; ++i) start[edges[2 * i + key] + 1]++;
  for (uint32_t v = 0; v < n; ++v) start[v + 1] += start[v];
  memcpy(fill, start, ((size_t)n + 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < m_log; ++i) bucket[fill[edges[2 * i + key]]++] = edges[2 * i + (1 - key)];
  out->n = n;
  out->off = (uint64_t*)malloc(((size_t)n + 1) * sizeof(uint64_t));
  out->col = (uint32_t*)malloc((m_log ? m_log : 1) * sizeof(uint32_t));
  uint64_t w = 0;
  out->off[0] = 0;
  for (uint32_t v = 0; v < n; ++v) {
    uint64_t b = start[v], e = start[v + 1];
    if (e - b > 1) qsort(bucket + b, (size_t)(e - b), sizeof(uint32_t), cmp_u32);
    for (uint64_t k = b; k < e; ++k)
      if (k == b || bucket[k] != bucket[k - 1]) out->col[w++] = bucket[k];
    out->off[v + 1] = w;
  }
  out->m = w;
  free(start);
  free(bucket);
  free(fill);
  return 0;
}

/* map_engine.cpp:9-19 — gather index: entry (u -> c) of g becomes u in row c.
 * Rows come out ascending because u is visited in increasing order. */
int cyo_transpose(const cyo_csr* g, cyo_csr* out) {
  memset(out, 0, sizeof *out);
  uint32_t n = g->n;
  out->n = n;
  out->m = g->m;
  out->off = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  out->col = (uint32_t*)malloc((g->m ? g->m : 1) * sizeof(uint32_t));
  for (uint64_t k = 0; k < g->m; ++k) out->off[g->col[k] + 1]++;
  for (uint32_t v = 0; v < n; ++v) out->off[v + 1] += out->off[v];
  uint64_t* pos = (uint64_t*)malloc(((size_t)n + 1) * sizeof(uint64_t));
  memcpy(pos, out->off, ((size_t)n + 1) * sizeof(uint64_t));
  for (uint32_t u = 0; u < n; ++u)
    for (uint64_t k = g->off[u]; k < g->off[u + 1]; ++k) out->col[pos[g->col[k]]++] = u;
  free(pos);
  return 0;
}

/* graph.cpp:125-196 — SCC decomposition (here: iterative Tarjan with an
 * explicit call stack) and the keep rule: a component is kept iff it is
 * cyclic (>= 2 vertices or a self-loop) and holds an accepting vertex. */
void cyo_scc_keep_mask(const cyo_csr* g, const uint64_t* acc, uint8_t* keep) {
  const uint32_t n = g->n;
  const uint32_t NONE = 0xFFFFFFFFu;
  uint32_t* idx = (uint32_t*)malloc(((size_t)n + 1) * sizeof(uint32_t));
  uint32_t* low = (uint32_t*)malloc(((size_t)n + 1) * sizeof(uint32_t));
  uint32_t* comp = (uint32_t*)malloc(((size_t)n + 1) * sizeof(uint32_t));
  uint8_t* onstk = (uint8_t*)calloc((size_t)n + 1, 1);
  uint8_t* loop = (uint8_t*)calloc((size_t)n + 1, 1);
  uint32_t* stk = (uint32_t*)malloc(((size_t)n + 1) * sizeof(uint32_t));
  uint32_t* cs_v = (uint32_t*)malloc(((size_t)n + 1) * sizeof(uint32_t));
  uint64_t* cs_e = (uint64_t*)malloc(((size_t)n + 1) * sizeof(uint64_t));
  /* per component: size and flags, at most n components */
  uint32_t* csize = (uint32_t*)calloc((size_t)n + 1, sizeof(uint32_t));
  uint8_t* cflag = (uint8_t*)calloc((size_t)n + 1, 1); /* bit0 self-loop, bit1 accepting */
  for (uint32_t v = 0; v < n; ++v) idx[v] = NONE;
  uint32_t counter = 0, sp = 0, ncomp = 0;
  for (uint32_t r = 0; r < n; ++r) {
    if (idx[r] != NONE) continue;
    uint32_t depth = 0;
    cs_v[0] = r;
    cs_e[0] = g->off[r];
    idx[r] = low[r] = counter++;
    stk[sp++] = r;
    onstk[r] = 1;
    depth = 1;
    while (depth) {
      uint32_t v = cs_v[depth - 1];
      if (cs_e[depth - 1] < g->off[v + 1]) {
        uint32_t w = g->col[cs_e[depth - 1]++];
        if (w == v) loop[v] = 1;
        if (idx[w] == NONE) {
          idx[w] = low[w] = counter++;
          stk[sp++] = w;
          onstk[w] = 1;
          cs_v[depth] = w;
          cs_e[depth] = g->off[w];
          ++depth;
        } else if (onstk[w] && idx[w] < low[v]) {
          low[v] = idx[w];
        }
        continue;
      }
      --depth;
      if (depth && low[v] < low[cs_v[depth - 1]]) low[cs_v[depth - 1]] = low[v];
      if (low[v] == idx[v]) {
        uint32_t c = ncomp++;
        uint32_t w;
        do {
          w = stk[--sp];
          onstk[w] = 0;
          comp[w] = c;
          csize[c]++;
          if (loop[w]) cflag[c] |= 1;
          if (acc_test(acc, w)) cflag[c] |= 2;
        } while (w != v);
      }
    }
  }
  for (uint32_t v = 0; v < n; ++v) {
    uint32_t c = comp[v];
    int cyclic = csize[c] >= 2 || (cflag[c] & 1);
    keep[v] = (uint8_t)(cyclic && (cflag[c] & 2));
  }
  free(idx); free(low); free(comp); free(onstk); free(loop); free(stk);
  free(cs_v); free(cs_e); free(csize); free(cflag);
}

/* graph.cpp:197-221 — order-preserving renumbering of kept vertices; every
 * edge with both endpoints kept survives (cross-SCC edges included). */
int cyo_restrict(const cyo_csr* g, const uint64_t* acc, cyo_csr* out, uint64_t* out_acc,
                 uint32_t* kept, uint32_t* n_kept) {
  const uint32_t n = g->n;
  uint8_t* keep = (uint8_t*)malloc((size_t)n + 1);
  uint32_t* nid = (uint32_t*)malloc(((size_t)n + 1) * sizeof(uint32_t));
  cyo_scc_keep_mask(g, acc, keep);
  uint32_t k = 0;
  for (uint32_t v = 0; v < n; ++v) {
    nid[v] = keep[v] ? k : 0xFFFFFFFFu;
    if (keep[v]) kept[k++] = v;
  }
  *n_kept = k;
  memset(out, 0, sizeof *out);
  out->n = k;
  out->off = (uint64_t*)malloc(((size_t)k + 1) * sizeof(uint64_t));
  out->col = (uint32_t*)malloc((g->m ? g->m : 1) * sizeof(uint32_t));
  memset(out_acc, 0, (((size_t)k + 63) / 64) * sizeof(uint64_t));
  uint64_t w = 0;
  out->off[0] = 0;
  for (uint32_t a = 0; a < k; ++a) {
    uint32_t v = kept[a];
    if (acc_test(acc, v)) out_acc[a >> 6] |= 1ull << (a & 63);
    for (uint64_t e = g->off[v]; e < g->off[v + 1]; ++e)
      if (nid[g->col[e]] != 0xFFFFFFFFu) out->col[w++] = nid[g->col[e]];
    out->off[a + 1] = w;
  }
  out->m = w;
  free(keep);
  free(nid);
  return 0;
}

/* map_engine.cpp:21-79 — one Jacobi step. Row v of the gather index lists
 * the sources u whose candidate max(x[u], u+1 if accepting) flows into v. */
void cyo_step(const cyo_csr* gather, const uint32_t* x, const uint64_t* acc, uint32_t* out,
              int* changed, uint32_t* witness) {
  int ch = 0;
  uint32_t wit = 0xFFFFFFFFu;
  for (uint32_t v = 0; v < gather->n; ++v) {
    uint32_t best = x[v];
    for (uint64_t e = gather->off[v]; e < gather->off[v + 1]; ++e) {
      uint32_t u = gather->col[e];
      uint32_t cand = x[u];
      if (acc_test(acc, u) && u + 1 > cand) cand = u + 1;
      if (cand > best) best = cand;
    }
    out[v] = best;
    if (best != x[v]) ch = 1;
    if (best == v + 1 && acc_test(acc, v) && v < wit) wit = v;
  }
  *changed = ch;
  *witness = wit;
}

/* map_engine.cpp:94-121 — all-NIL start; every step counts, including the
 * final unchanged one; with early_exit the first witness ends the run. */
uint64_t cyo_fixpoint(const cyo_csr* gather, const uint64_t* acc, int early_exit, uint32_t* x,
                      uint32_t* scratch, uint32_t* witness) {
  uint32_t n = gather->n;
  memset(x, 0, (size_t)n * sizeof(uint32_t));
  uint64_t steps = 0;
  for (;;) {
    int ch;
    uint32_t w;
    cyo_step(gather, x, acc, scratch, &ch, &w);
    ++steps;
    memcpy(x, scratch, (size_t)n * sizeof(uint32_t));
    if ((w != 0xFFFFFFFFu && early_exit) || !ch) {
      *witness = w;
      return steps;
    }
  }
}

/* map_engine.cpp:123-137 — D = accepting vertices that are somebody's value. */
uint64_t cyo_demote(const uint32_t* x, uint32_t n, const uint64_t* acc, uint64_t* remaining,
                    uint32_t* demoted) {
  size_t words = ((size_t)n + 63) / 64;
  uint64_t* used = (uint64_t*)calloc(words ? words : 1, sizeof(uint64_t));
  for (uint32_t v = 0; v < n; ++v)
    if (x[v] != 0 && x[v] - 1 < n) used[(x[v] - 1) >> 6] |= 1ull << ((x[v] - 1) & 63);
  uint64_t nd = 0;
  for (size_t i = 0; i < words; ++i) {
    uint64_t d = acc[i] & used[i];
    remaining[i] = acc[i] & ~used[i];
    while (d) {
      int b = __builtin_ctzll(d);
      demoted[nd++] = (uint32_t)(i * 64 + (size_t)b);
      d &= d - 1;
    }
  }
  free(used);
  return nd;
}

uint64_t cyo_vector_hash(const uint32_t* x, uint32_t n) {
  uint64_t h = 0;
  for (uint32_t v = 0; v < n; ++v) h += cyc_splitmix64(((uint64_t)v << 32) | x[v]);
  return h;
}

/* map_engine.cpp:139-162 — MAP loop: fixpoint, witness => cycle, else demote;
 * an empty D or an empty accepting set ends the run without a cycle. */
void cyo_run_map(const cyo_csr* gather, const uint64_t* acc, int early_exit, cyo_map_stats* st,
                 uint32_t* final_x, uint64_t* iter_hash, uint64_t* iter_steps, uint64_t cap) {
  const uint32_t n = gather->n;
  size_t words = ((size_t)n + 63) / 64;
  memset(st, 0, sizeof *st);
  uint64_t* front = (uint64_t*)malloc((words ? words : 1) * sizeof(uint64_t));
  uint64_t* rem = (uint64_t*)malloc((words ? words : 1) * sizeof(uint64_t));
  uint32_t* x = (uint32_t*)calloc((size_t)n + 1, sizeof(uint32_t));
  uint32_t* tmp = (uint32_t*)malloc(((size_t)n + 1) * sizeof(uint32_t));
  uint32_t* dem = (uint32_t*)malloc(((size_t)n + 1) * sizeof(uint32_t));
  memcpy(front, acc, words * sizeof(uint64_t));
  for (;;) {
    int any = 0;
    for (size_t i = 0; i < words; ++i) any |= front[i] != 0;
    if (!any) break;
    uint32_t w;
    uint64_t steps = cyo_fixpoint(gather, front, early_exit, x, tmp, &w);
    if (st->iterations < cap) {
      if (iter_hash) iter_hash[st->iterations] = cyo_vector_hash(x, n);
      if (iter_steps) iter_steps[st->iterations] = steps;
    }
    st->iterations++;
    st->kernel_calls += steps;
    if (w != 0xFFFFFFFFu) {
      st->cycle_found = 1;
      st->witness = w;
      break;
    }
    uint64_t nd = cyo_demote(x, n, front, rem, dem);
    st->demoted_total += nd;
    if (nd == 0) break;
    memcpy(front, rem, words * sizeof(uint64_t));
  }
  if (final_x) memcpy(final_x, x, (size_t)n * sizeof(uint32_t));
  free(front); free(rem); free(x); free(tmp); free(dem);
}

int cyo_generate(const void* gen_params, uint32_t* edges, uint64_t* acc_words) {
  const cyc_gen_params* p = (const cyc_gen_params*)gen_params;
  if (p->kind == CYC_GEN_PRODUCT) {
    uint32_t* a = (uint32_t*)malloc(((size_t)p->n + 1) * 4);
    uint32_t* b = (uint32_t*)malloc(((size_t)p->n + 1) * 4);
    int rc = a && b ? cyc_prod_generate_host(p, a, b, edges, acc_words) : -1;
    free(a);
    free(b);
    return rc;
  }
  for (uint64_t i = 0; i < p->m; ++i) cyc_gen_edge(p, i, &edges[2 * i], &edges[2 * i + 1]);
  size_t words = ((size_t)p->n + 63) / 64;
  memset(acc_words, 0, words * sizeof(uint64_t));
  for (uint32_t v = 0; v < p->n; ++v)
    if (cyc_gen_accepting(p, v)) acc_words[v >> 6] |= 1ull << (v & 63);
  return 0;
}

int cyo_gen_preset(int index, void* gen_params) {
  return cyc_gen_config((cyc_gen_params*)gen_params, index);
}

int cyo_gen_prepare(void* gen_params) { return cyc_gen_init((cyc_gen_params*)gen_params); }

/* owcty.cpp:14-33 — vertices of `in` reachable by >= 1 edge, through `in`,
 * from an accepting member of `in` (explicit stack, any visiting order). */
static void owcty_reach(const cyo_csr* g, const uint8_t* in, const uint64_t* acc, uint8_t* out,
                        uint32_t* stack) {
  const uint32_t n = g->n;
  size_t top = 0;
  memset(out, 0, n);
  for (uint32_t v = 0; v < n; ++v)
    if (in[v] && ((acc[v >> 6] >> (v & 63)) & 1)) stack[top++] = v;
  /* sources are expanded once even if never re-reached */
  while (top) {
    const uint32_t u = stack[--top];
    for (uint64_t i = g->off[u]; i < g->off[u + 1]; ++i) {
      const uint32_t c = g->col[i];
      if (in[c] && !out[c]) {
        out[c] = 1;
        if (!((acc[c >> 6] >> (c & 63)) & 1)) stack[top++] = c; /* accepting c already seeded */
      }
    }
  }
}

/* owcty.cpp:35-54 — drop members without a predecessor in the set, repeatedly. */
static void owcty_elim(const cyo_csr* g, uint8_t* set, uint32_t* indeg, uint32_t* queue) {
  const uint32_t n = g->n;
  size_t head = 0, tail = 0;
  memset(indeg, 0, (size_t)n * 4);
  for (uint32_t u = 0; u < n; ++u)
    if (set[u])
      for (uint64_t i = g->off[u]; i < g->off[u + 1]; ++i)
        if (set[g->col[i]]) indeg[g->col[i]]++;
  for (uint32_t v = 0; v < n; ++v)
    if (set[v] && !indeg[v]) queue[tail++] = v;
  while (head < tail) {
    const uint32_t v = queue[head++];
    set[v] = 0;
    for (uint64_t i = g->off[v]; i < g->off[v + 1]; ++i) {
      const uint32_t c = g->col[i];
      if (set[c] && --indeg[c] == 0) queue[tail++] = c;
    }
  }
}

void cyo_run_owcty(const cyo_csr* g, const uint64_t* acc, int* cycle, uint32_t* witness,
                   uint64_t* outer_iterations, uint64_t* final_size) {
  const uint32_t n = g->n;
  *cycle = 0;
  *witness = 0xFFFFFFFFu;
  *outer_iterations = 0;
  *final_size = 0;
  if (n == 0) return;
  uint8_t* set = (uint8_t*)malloc(n);
  uint8_t* nxt = (uint8_t*)malloc(n);
  uint32_t* a = (uint32_t*)malloc((size_t)n * 4);
  uint32_t* b = (uint32_t*)malloc((size_t)n * 4);
  memset(set, 1, n);
  uint64_t live = n;
  for (;;) {
    /* a vertex may sit on the reach stack at most twice (seed + reached) */
    uint32_t* stack = (uint32_t*)malloc((size_t)n * 8);
    owcty_reach(g, set, acc, nxt, stack);
    free(stack);
    owcty_elim(g, nxt, a, b);
    ++*outer_iterations;
    uint64_t cnt = 0;
    int same = 1;
    for (uint32_t v = 0; v < n; ++v) {
      cnt += nxt[v];
      same &= nxt[v] == set[v];
    }
    memcpy(set, nxt, n);
    live = cnt;
    if (cnt == 0 || same) break;
  }
  *final_size = live;
  for (uint32_t v = 0; v < n && live; ++v)
    if (set[v] && ((acc[v >> 6] >> (v & 63)) & 1)) {
      *cycle = 1;
      *witness = v;
      break;
    }
  free(set);
  free(nxt);
  free(a);
  free(b);
}
