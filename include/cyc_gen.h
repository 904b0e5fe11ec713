/*
 * cyc_gen.h — seeded synthetic graph generators shared, bit-for-bit, by the
 * B200 library (device-side generation for the bench), the CPU oracle
 * restatement (oracle/), and the reference driver (oracle/ref_driver.cpp).
 *
 * Every edge is a pure function of (params, edge index), so a host run and a
 * device run produce identical logs without shipping the edge list around.
 * Configs follow SURVEY.md §8(d) (seed 0x09122555 + config index):
 *   C1  uniform random digraph, n = 2^16, out-degree 4, 5 % accepting
 *   C2  layered DAG of SCCs (accepting connectors c_0..c_L, W rings of S per
 *       layer, every ring member -> c_{l+1}); iterations = L+1,
 *       kernel_calls = (L+1)^2
 *   C3  R-MAT (Graph500 a,b,c = .57,.19,.19), seeded vertex permutation
 *   C4  product state space: a token on a 2^g x 2^g torus (moves +x, +y)
 *       times a 4-state Buechi automaton, planted accepting cycle in one
 *       region; ids in BFS discovery order from the initial state (the
 *       explorer's interner order, reference graph.cpp:223-230)
 *   C5  chain of small SCCs (C2 layout, only the sink connector accepting,
 *       ring exit from member S/2)
 * Vertex ids are VertexId = uint32_t (reference types.hpp:9); the log is the
 * reference EdgeLog's {src,dst} pair sequence (graph.hpp:80-82).
 *
 * Header-only C; compiles as C99, C++ and CUDA (host+device).
 */
#ifndef CYC_GEN_H
#define CYC_GEN_H

#include <stdint.h>

#if defined(__CUDACC__)
#define CYC_HD __host__ __device__ __forceinline__
#else
#define CYC_HD static inline
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define CYC_SEED_BASE 0x09122555ull

enum cyc_gen_kind {
  CYC_GEN_UNIFORM = 1, /* C1 */
  CYC_GEN_LAYERED = 2, /* C2 (exit_all = 1, acc_all = 1), C5 (exit_all = 0, acc_all = 0) */
  CYC_GEN_RMAT = 3,    /* C3 */
  CYC_GEN_PRODUCT = 4  /* C4 */
};

typedef struct cyc_gen_params {
  int32_t kind;
  uint32_t n;          /* derived by cyc_gen_init */
  uint64_t m;          /* logged edges, derived by cyc_gen_init */
  uint64_t seed;
  /* uniform */
  uint32_t deg;
  /* accepting threshold: v accepting iff hash(seed^salt, v) < acc_thr */
  uint64_t acc_thr;
  /* layered */
  uint32_t L, W, S;
  uint32_t exit_all;   /* 1: every ring member -> c_{l+1}; 0: member S/2 only */
  uint32_t acc_all;    /* 1: every connector accepting; 0: only c_L */
  /* rmat */
  uint32_t scale, edgefactor;
  uint64_t thr_a, thr_ab, thr_abc;
  uint64_t perm_mul1, perm_mul2; /* odd multipliers of the vertex permutation */
  /* product (C4) */
  uint32_t grid_bits;  /* torus side G = 2^grid_bits, n = 4 G^2 */
  uint32_t region;     /* side of the square region R (clamped to G/2) */
  uint32_t plant;      /* 1: reset move from R's far corner back to its near corner */
  uint32_t reserved;
} cyc_gen_params;

CYC_HD uint64_t cyc_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* Counter-based stream: value i of stream `seed`. */
CYC_HD uint64_t cyc_hash2(uint64_t seed, uint64_t i) {
  return cyc_splitmix64(cyc_splitmix64(seed) ^ (i * 0xD1B54A32D192ED03ull));
}

/* Threshold for a fraction given in basis points (1/10000). */
CYC_HD uint64_t cyc_bp_threshold(uint32_t bp) {
  return (uint64_t)bp * (0xFFFFFFFFFFFFFFFFull / 10000ull);
}

#define CYC_ACC_SALT 0xACCE97ull

/* Maps a 64-bit hash uniformly onto [0, n). */
CYC_HD uint32_t cyc_range(uint64_t h, uint32_t n) {
  return (uint32_t)(((h >> 32) * (uint64_t)n) >> 32);
}

/* Bijection on [0, 2^bits): odd multiply and xor-shift rounds. */
CYC_HD uint32_t cyc_permute_bits(uint32_t v, uint32_t bits, uint64_t mul1, uint64_t mul2) {
  uint64_t mask = (bits >= 64) ? ~0ull : ((1ull << bits) - 1ull);
  uint64_t x = v;
  uint32_t half = bits / 2 ? bits / 2 : 1;
  x = (x * mul1) & mask;
  x ^= x >> half;
  x = (x * mul2) & mask;
  x ^= x >> half;
  x = (x * mul1) & mask;
  return (uint32_t)x;
}

/* Layered graphs: connector c_l has id l*(W*S+1); ring r member j of layer l
 * has id l*(W*S+1) + 1 + r*S + j; sink c_L = L*(W*S+1). */
CYC_HD uint32_t cyc_layer_stride(const cyc_gen_params* p) { return p->W * p->S + 1u; }
CYC_HD uint32_t cyc_layer_exits(const cyc_gen_params* p) { return p->exit_all ? p->S : 1u; }

/* ---- C4 product graph ------------------------------------------------------
 * System state (x, y) on a G x G torus; moves E: x+1, N: y+1 (mod G), plus,
 * when planted, a reset move from R's far corner (rx+k-1, ry+k-1) to its near
 * corner (rx, ry); R = [rx, rx+k) x [ry, ry+k), rx = ry = G/4.
 * Automaton (q2 accepting), guards read the source state's label inR:
 *   q0 -true-> q0, q0 -true-> q1, q1 -true-> q1, q1 -true-> q2,
 *   q2 -inR-> q2, q2 -!inR-> q3, q3 -true-> q3.
 * Product move (s,q) -> (s',q') for each system move s -> s' and each enabled
 * automaton transition q -> q', in that nesting order. Accepting cycles exist
 * only inside R x {q2}, and only through the planted reset. Every one of the
 * 4 G^2 product states is reachable from (0,0,q0) (k < G).
 * State key = q << 2g | y << g | x; vertex id = BFS discovery index. */
CYC_HD uint32_t cyc_prod_side(const cyc_gen_params* p) { return 1u << p->grid_bits; }
CYC_HD uint32_t cyc_prod_k(const cyc_gen_params* p) {
  uint32_t half = cyc_prod_side(p) / 2u;
  return p->region < 1u ? 1u : (p->region > half ? half : p->region);
}
/* Successors of `key` in canonical order into out[0..5]; returns the count. */
CYC_HD uint32_t cyc_prod_succ(const cyc_gen_params* p, uint32_t key, uint32_t* out) {
  const uint32_t g = p->grid_bits, G = 1u << g, mask = G - 1u;
  const uint32_t x = key & mask, y = (key >> g) & mask, q = key >> (2u * g);
  const uint32_t k = cyc_prod_k(p), r0 = G / 4u;
  const int in_r = x >= r0 && x < r0 + k && y >= r0 && y < r0 + k;
  uint32_t qs[2], nq = 0;
  if (q == 0u) { qs[0] = 0u; qs[1] = 1u; nq = 2u; }
  else if (q == 1u) { qs[0] = 1u; qs[1] = 2u; nq = 2u; }
  else if (q == 2u) { qs[0] = in_r ? 2u : 3u; nq = 1u; }
  else { qs[0] = 3u; nq = 1u; }
  uint32_t mv[3], nm = 0;
  mv[nm++] = (y << g) | ((x + 1u) & mask);
  mv[nm++] = (((y + 1u) & mask) << g) | x;
  if (p->plant && x == r0 + k - 1u && y == r0 + k - 1u) mv[nm++] = (r0 << g) | r0;
  uint32_t c = 0;
  for (uint32_t a = 0; a < nm; ++a)
    for (uint32_t b = 0; b < nq; ++b) out[c++] = (qs[b] << (2u * g)) | mv[a];
  return c;
}
CYC_HD int cyc_prod_accepting_key(const cyc_gen_params* p, uint32_t key) {
  return (key >> (2u * p->grid_bits)) == 2u;
}

/* Edge i of the log (index-addressable kinds; C4 needs the BFS order, see
 * cyc_prod_generate_host and the library's device generator). */
CYC_HD void cyc_gen_edge(const cyc_gen_params* p, uint64_t i, uint32_t* src, uint32_t* dst) {
  if (p->kind == CYC_GEN_UNIFORM) {
    *src = (uint32_t)(i / p->deg);
    *dst = cyc_range(cyc_hash2(p->seed, i), p->n);
  } else if (p->kind == CYC_GEN_LAYERED) {
    uint64_t per_ring = 1ull + p->S + cyc_layer_exits(p);
    uint64_t per_layer = (uint64_t)p->W * per_ring;
    uint32_t l = (uint32_t)(i / per_layer);
    uint64_t rem = i % per_layer;
    uint32_t r = (uint32_t)(rem / per_ring);
    uint32_t k = (uint32_t)(rem % per_ring);
    uint32_t base = l * cyc_layer_stride(p);
    uint32_t ring = base + 1u + r * p->S;
    if (k == 0) {                       /* c_l -> ring entry */
      *src = base;
      *dst = ring;
    } else if (k <= p->S) {             /* ring cycle member k-1 -> member k mod S */
      *src = ring + (k - 1u);
      *dst = ring + (k % p->S);
    } else {                            /* exit -> c_{l+1} */
      uint32_t member = p->exit_all ? (k - p->S - 1u) : (p->S / 2u);
      *src = ring + member;
      *dst = base + cyc_layer_stride(p);
    }
  } else { /* R-MAT */
    uint32_t s = 0, d = 0;
    for (uint32_t lev = 0; lev < p->scale; ++lev) {
      uint64_t r = cyc_hash2(p->seed, i * (uint64_t)p->scale + lev);
      uint32_t sb = 0, db = 0;
      if (r < p->thr_a) {
      } else if (r < p->thr_ab) {
        db = 1;
      } else if (r < p->thr_abc) {
        sb = 1;
      } else {
        sb = 1;
        db = 1;
      }
      s = (s << 1) | sb;
      d = (d << 1) | db;
    }
    *src = cyc_permute_bits(s, p->scale, p->perm_mul1, p->perm_mul2);
    *dst = cyc_permute_bits(d, p->scale, p->perm_mul1, p->perm_mul2);
  }
}

CYC_HD int cyc_gen_accepting(const cyc_gen_params* p, uint32_t v) {
  if (p->kind == CYC_GEN_LAYERED) {
    uint32_t stride = cyc_layer_stride(p);
    if (v % stride != 0) return 0;
    return p->acc_all ? 1 : (v == p->L * stride);
  }
  return cyc_hash2(p->seed ^ CYC_ACC_SALT, v) < p->acc_thr;
}

/* Fills derived fields (n, m). Returns 0 on success, -1 on bad params. */
CYC_HD int cyc_gen_init(cyc_gen_params* p) {
  if (p->kind == CYC_GEN_UNIFORM) {
    if (p->n == 0 || p->deg == 0) { p->m = 0; return p->n == 0 ? 0 : -1; }
    p->m = (uint64_t)p->n * p->deg;
    return 0;
  }
  if (p->kind == CYC_GEN_LAYERED) {
    if (p->W == 0 || p->S == 0) return -1;
    uint64_t n = (uint64_t)p->L * ((uint64_t)p->W * p->S + 1ull) + 1ull;
    if (n >= 0x80000000ull) return -1;
    p->n = (uint32_t)n;
    p->m = (uint64_t)p->L * p->W * (1ull + p->S + cyc_layer_exits(p));
    return 0;
  }
  if (p->kind == CYC_GEN_PRODUCT) {
    if (p->grid_bits < 2 || p->grid_bits > 14) return -1;
    const uint64_t G = 1ull << p->grid_bits;
    p->n = (uint32_t)(4ull * G * G);
    p->m = 12ull * G * G + (p->plant ? 6ull : 0ull);
    return 0;
  }
  if (p->kind == CYC_GEN_RMAT) {
    if (p->scale == 0 || p->scale > 30) return -1;
    p->n = 1u << p->scale;
    p->m = (uint64_t)p->n * p->edgefactor;
    p->perm_mul1 = cyc_splitmix64(p->seed ^ 0x5151ull) | 1ull;
    p->perm_mul2 = cyc_splitmix64(p->seed ^ 0xA2A2ull) | 1ull;
    if (p->thr_abc == 0) { /* Graph500 defaults a,b,c,d = .57,.19,.19,.05 */
      p->thr_a = cyc_bp_threshold(5700);
      p->thr_ab = cyc_bp_threshold(7600);
      p->thr_abc = cyc_bp_threshold(9500);
    }
    return 0;
  }
  return -1;
}

/* Canonical configurations. `index` is the config number
 * 1..5; size knobs may be overridden afterwards, then cyc_gen_init again. */
CYC_HD int cyc_gen_config(cyc_gen_params* p, int index) {
  cyc_gen_params z;
  {
    unsigned char* b = (unsigned char*)&z;
    for (unsigned k = 0; k < sizeof z; ++k) b[k] = 0;
  }
  *p = z;
  p->seed = CYC_SEED_BASE + (uint64_t)index;
  switch (index) {
    case 1:
      p->kind = CYC_GEN_UNIFORM; p->n = 1u << 16; p->deg = 4; p->acc_thr = cyc_bp_threshold(500);
      break;
    case 2:
      p->kind = CYC_GEN_LAYERED; p->L = 64; p->W = 4096; p->S = 16; p->exit_all = 1; p->acc_all = 1;
      break;
    case 3:
      p->kind = CYC_GEN_RMAT; p->scale = 26; p->edgefactor = 16; p->acc_thr = cyc_bp_threshold(100);
      break;
    case 4:
      p->kind = CYC_GEN_PRODUCT; p->grid_bits = 13; p->region = 64; p->plant = 1;
      break;
    case 5:
      p->kind = CYC_GEN_LAYERED; p->L = 64; p->W = 512; p->S = 512; p->exit_all = 0; p->acc_all = 0;
      break;
    default:
      return -1;
  }
  return cyc_gen_init(p);
}

/* Host generation of C4 (sequential BFS queue = the interner's discovery
 * order): key_of_id / id_of_key are caller arrays of p->n entries; edges
 * (2 p->m) and acc_words (ceil(n/64)) may be NULL. Returns 0, or -1 if some
 * state is unreachable. */
#ifndef __CUDA_ARCH__
static inline int cyc_prod_generate_host(const cyc_gen_params* p, uint32_t* key_of_id,
                                         uint32_t* id_of_key, uint32_t* edges, uint64_t* acc_words) {
  const uint32_t n = p->n;
  uint32_t succ[6];
  uint64_t tail = 1, e = 0;
  for (uint32_t k = 0; k < n; ++k) id_of_key[k] = 0xFFFFFFFFu;
  key_of_id[0] = 0u;
  id_of_key[0] = 0u;
  for (uint64_t head = 0; head < tail; ++head) {
    const uint32_t c = cyc_prod_succ(p, key_of_id[head], succ);
    for (uint32_t j = 0; j < c; ++j)
      if (id_of_key[succ[j]] == 0xFFFFFFFFu) {
        id_of_key[succ[j]] = (uint32_t)tail;
        key_of_id[tail++] = succ[j];
      }
  }
  if (tail != n) return -1;
  for (uint32_t v = 0; v < n; ++v) {
    const uint32_t c = cyc_prod_succ(p, key_of_id[v], succ);
    for (uint32_t j = 0; j < c && edges; ++j, ++e) {
      edges[2 * e] = v;
      edges[2 * e + 1] = id_of_key[succ[j]];
    }
  }
  if (acc_words) {
    for (uint64_t w = 0; w < ((uint64_t)n + 63u) / 64u; ++w) acc_words[w] = 0;
    for (uint32_t v = 0; v < n; ++v)
      if (cyc_prod_accepting_key(p, key_of_id[v])) acc_words[v >> 6] |= 1ull << (v & 63u);
  }
  return 0;
}
#endif

#ifdef __cplusplus
}
#endif

#endif /* CYC_GEN_H */
