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
  CYC_GEN_RMAT = 3     /* C3 */
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

/* Edge i of the log. */
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
    case 5:
      p->kind = CYC_GEN_LAYERED; p->L = 64; p->W = 512; p->S = 512; p->exit_all = 0; p->acc_all = 0;
      break;
    default:
      return -1;
  }
  return cyc_gen_init(p);
}

#ifdef __cplusplus
}
#endif

#endif /* CYC_GEN_H */
