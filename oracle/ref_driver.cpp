// ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference implementation (compiled from
// /root/reference/proj/src/{graph,map_engine,parallel,errors,oracle}.cpp by
// oracle/Makefile into oracle/_ref/libcycheck_ref.so). It drives only the
// reference's public API (proj/include/cycheck/*.hpp) so that tests and the
// bench's CPU arm can run the reference on the same seeded inputs as the GPU.
//
// run_map does not return the map vector (map_engine.cpp:139-162), so
// ref_run_map replays its loop with the public fixpoint()/demote() and checks
// the replica's MapStats against run_map's own before reporting.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "cycheck/errors.hpp"
#include "cycheck/graph.hpp"
#include "cycheck/map_engine.hpp"
#include "cycheck/oracle.hpp"
#include "cycheck/owcty.hpp"
#include "cycheck/parallel.hpp"
#include "../include/cyc_gen.h"

using namespace cycheck;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

struct Snap {
  CsrSnapshot snap;
  std::vector<VertexId> kept;  // only for restricted snapshots
  // the reference's MaxPropagation of this snapshot (its gather-index build,
  // map_engine.cpp:9-19), made once by ref_time_steps and reused
  std::unique_ptr<MaxPropagation> prop;
  double prop_s = 0;
};

Bitset bitset_from(const uint64_t* words, uint32_t n) {
  Bitset b(n);
  if (words) {
    for (size_t i = 0; i < b.words().size(); ++i) b.words()[i] = words[i];
    b.trim();
  }
  return b;
}

uint64_t vec_hash(const MapVector& x) {
  uint64_t h = 0;
  for (uint32_t v = 0; v < x.size(); ++v) h += cyc_splitmix64((uint64_t(v) << 32) | x[v].code);
  return h;
}

MapVector to_vec(const uint32_t* x, uint32_t n) {
  MapVector out(n);
  for (uint32_t v = 0; v < n; ++v) out[v].code = x[v];
  return out;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Status codes: 0 ok, 1 ContractError, 2 ResourceLimitError, 3 other.
#define REF_TRY try {
#define REF_CATCH                                  \
  }                                                \
  catch (const ContractError& e) { return fail(e, 1); } \
  catch (const ResourceLimitError& e) { return fail(e, 2); } \
  catch (const ParseError& e) { return fail(e, 5); } \
  catch (const std::exception& e) { return fail(e, 3); }

// EdgeLog + build_snapshot (graph.cpp:63-111). edges: 2*m u32 pairs.
int ref_snapshot_new(const uint32_t* edges, uint64_t m, uint32_t n, const uint64_t* acc,
                     int transposed, void** out) {
  REF_TRY
  EdgeLog::Limits lim;
  lim.max_vertices = n > 0 ? n : 1;
  lim.max_edges = m > 0 ? m : 1;
  EdgeLog log(lim);
  for (uint32_t v = 0; v < n; ++v) log.add_vertex(acc && ((acc[v >> 6] >> (v & 63)) & 1u));
  for (uint64_t i = 0; i < m; ++i) log.append_edge(edges[2 * i], edges[2 * i + 1]);
  auto* s = new Snap;
  s->snap = build_snapshot(log, transposed ? Orientation::transposed : Orientation::forward);
  *out = s;
  return 0;
  REF_CATCH
}

}  // extern "C"

// Appends a generated configuration to the reference's own EdgeLog.
static void fill_log(const cyc_gen_params* p, EdgeLog& log) {
  if (p->kind == CYC_GEN_PRODUCT) {  // BFS-ordered product graph (cyc_gen.h)
    std::vector<uint32_t> a(p->n), b(p->n), e(2 * p->m);
    std::vector<uint64_t> w((p->n + 63) / 64);
    if (cyc_prod_generate_host(p, a.data(), b.data(), e.data(), w.data()) != 0)
      throw std::runtime_error("product generator: unreachable states");
    for (uint32_t v = 0; v < p->n; ++v) log.add_vertex((w[v >> 6] >> (v & 63)) & 1);
    for (uint64_t i = 0; i < p->m; ++i) log.append_edge(e[2 * i], e[2 * i + 1]);
    return;
  }
  for (uint32_t v = 0; v < p->n; ++v) log.add_vertex(cyc_gen_accepting(p, v) != 0);
  for (uint64_t i = 0; i < p->m; ++i) {
    uint32_t s, d;
    cyc_gen_edge(p, i, &s, &d);
    log.append_edge(s, d);
  }
}

extern "C" {

int ref_snapshot_gen(const void* params, int transposed, void** out) {
  REF_TRY
  const auto* p = static_cast<const cyc_gen_params*>(params);
  EdgeLog::Limits lim;
  lim.max_vertices = p->n > 0 ? p->n : 1;
  lim.max_edges = p->m > 0 ? p->m : 1;
  EdgeLog log(lim);
  fill_log(p, log);
  auto* s = new Snap;
  s->snap = build_snapshot(log, transposed ? Orientation::transposed : Orientation::forward);
  *out = s;
  return 0;
  REF_CATCH
}

void ref_snapshot_free(void* h) { delete static_cast<Snap*>(h); }

void ref_snapshot_info(void* h, uint32_t* n, uint64_t* m) {
  auto* s = static_cast<Snap*>(h);
  *n = s->snap.n;
  *m = s->snap.m;
}

void ref_snapshot_export(void* h, uint64_t* off, uint32_t* col, uint64_t* acc, uint32_t* kept) {
  auto* s = static_cast<Snap*>(h);
  if (off) std::memcpy(off, s->snap.row_offsets.data(), (s->snap.n + 1ull) * 8);
  if (col && s->snap.m) std::memcpy(col, s->snap.col_indices.data(), s->snap.m * 4);
  if (acc && !s->snap.accepting.words().empty())
    std::memcpy(acc, s->snap.accepting.words().data(), s->snap.accepting.words().size() * 8);
  if (kept && !s->kept.empty()) std::memcpy(kept, s->kept.data(), s->kept.size() * 4);
}

// restrict_to_accepting_sccs (graph.cpp:190-221).
int ref_restrict(void* h, void** out) {
  REF_TRY
  auto* s = static_cast<Snap*>(h);
  SccRestriction r = restrict_to_accepting_sccs(s->snap);
  auto* o = new Snap;
  o->snap = std::move(r.snapshot);
  o->kept = std::move(r.kept);
  *out = o;
  return 0;
  REF_CATCH
}

// MaxPropagation::step (map_engine.cpp:21-79). witness = UINT32_MAX if none.
int ref_step(void* h, const uint32_t* x, const uint64_t* acc, int workers, uint32_t* out,
             int* changed, uint32_t* witness) {
  REF_TRY
  auto* s = static_cast<Snap*>(h);
  MaxPropagation k(s->snap);
  WorkerPool pool(workers);
  MapVector xv = to_vec(x, s->snap.n), ov;
  StepResult r = k.step(xv, acc ? bitset_from(acc, s->snap.n) : s->snap.accepting, ov, pool);
  for (uint32_t v = 0; v < s->snap.n; ++v) out[v] = ov[v].code;
  *changed = r.changed;
  *witness = r.self_witness ? *r.self_witness : 0xFFFFFFFFu;
  return 0;
  REF_CATCH
}

// fixpoint (map_engine.cpp:94-121).
int ref_fixpoint(void* h, const uint64_t* acc, int early_exit, int workers, uint32_t* values,
                 uint64_t* steps, uint32_t* witness) {
  REF_TRY
  auto* s = static_cast<Snap*>(h);
  MapOptions o;
  o.workers = workers;
  o.early_exit = early_exit != 0;
  FixpointResult fr = fixpoint(s->snap, acc ? bitset_from(acc, s->snap.n) : s->snap.accepting, o);
  for (uint32_t v = 0; v < s->snap.n; ++v) values[v] = fr.values[v].code;
  *steps = fr.steps;
  *witness = fr.witness ? *fr.witness : 0xFFFFFFFFu;
  return 0;
  REF_CATCH
}

// demote (map_engine.cpp:123-137).
int ref_demote(const uint32_t* x, uint32_t n, const uint64_t* acc, uint64_t* remaining,
               uint32_t* demoted, uint64_t* n_demoted) {
  REF_TRY
  DemoteResult d = demote(to_vec(x, n), bitset_from(acc, n));
  std::memcpy(remaining, d.remaining.words().data(), d.remaining.words().size() * 8);
  for (size_t i = 0; i < d.demoted.size(); ++i) demoted[i] = d.demoted[i];
  *n_demoted = d.demoted.size();
  return 0;
  REF_CATCH
}

// run_map (map_engine.cpp:139-162), replayed through public fixpoint/demote to
// expose the vectors; stats[] = {cycle, witness, iterations, kernel_calls,
// demoted_total}. Returns 4 if the replica disagrees with run_map itself.
int ref_run_map(void* h, const uint64_t* acc, int early_exit, int workers, uint64_t* stats,
                uint32_t* final_x, uint64_t* iter_hash, uint64_t* iter_steps, uint64_t cap,
                int check_run_map) {
  REF_TRY
  auto* s = static_cast<Snap*>(h);
  const CsrSnapshot& snap = s->snap;
  Bitset front = acc ? bitset_from(acc, snap.n) : snap.accepting;
  MapOptions o;
  o.workers = workers;
  o.early_exit = early_exit != 0;
  MaxPropagation kernel(snap);
  WorkerPool pool(workers);
  MapStats st;
  MapVector last(snap.n, MapValue::nil());
  bool cycle = false;
  uint32_t wit = 0xFFFFFFFFu;
  while (front.any()) {
    FixpointResult fr = fixpoint(kernel, front, o, pool);
    if (st.iterations < cap) {
      if (iter_hash) iter_hash[st.iterations] = vec_hash(fr.values);
      if (iter_steps) iter_steps[st.iterations] = fr.steps;
    }
    ++st.iterations;
    st.kernel_calls += fr.steps;
    last = fr.values;
    if (fr.witness) {
      cycle = true;
      wit = *fr.witness;
      break;
    }
    DemoteResult dr = demote(fr.values, front);
    st.demoted_total += dr.demoted.size();
    if (dr.demoted.empty()) break;
    front = std::move(dr.remaining);
  }
  if (check_run_map) {
    auto [verdict, rs] = run_map(snap, acc ? bitset_from(acc, snap.n) : snap.accepting, o);
    bool same = verdict.cycle_found() == cycle && rs.iterations == st.iterations &&
                rs.kernel_calls == st.kernel_calls && rs.demoted_total == st.demoted_total &&
                (!cycle || (verdict.witness && *verdict.witness == wit));
    if (!same) {
      g_err = "replica disagrees with run_map";
      return 4;
    }
  }
  stats[0] = cycle;
  stats[1] = wit;
  stats[2] = st.iterations;
  stats[3] = st.kernel_calls;
  stats[4] = st.demoted_total;
  if (final_x)
    for (uint32_t v = 0; v < snap.n; ++v) final_x[v] = last[v].code;
  return 0;
  REF_CATCH
}

// scc_verdict (oracle.cpp:32-98) on the snapshot's own edge relation.
int ref_scc_verdict(void* h, int* cycle) {
  REF_TRY
  auto* s = static_cast<Snap*>(h);
  auto edges = s->snap.edge_list();
  OracleVerdict ov = scc_verdict(edges, s->snap.n, s->snap.accepting, ~0ull);
  *cycle = ov.verdict.cycle_found();
  return 0;
  REF_CATCH
}

// run_owcty (owcty.cpp:56-87) on the snapshot: out = {cycle, witness,
// outer_iterations, final_size}.
int ref_run_owcty(void* h, const uint64_t* acc, uint64_t* out) {
  REF_TRY
  auto* s = static_cast<Snap*>(h);
  Bitset a = acc ? bitset_from(acc, s->snap.n) : s->snap.accepting;
  auto [v, st] = run_owcty(s->snap, a);
  out[0] = v.cycle_found();
  out[1] = v.witness ? *v.witness : 0xFFFFFFFFull;
  out[2] = st.outer_iterations;
  out[3] = st.final_size;
  return 0;
  REF_CATCH
}

// parse_explicit_graph (graph.cpp:259-297) of an in-memory text; *out owns the
// ExplicitGraph. Status 5 = ParseError (message = what()).
int ref_explicit_parse(const char* text, uint64_t len, void** out) {
  REF_TRY
  std::istringstream in(std::string(text, len));
  *out = new ExplicitGraph(parse_explicit_graph(in));
  return 0;
  REF_CATCH
}

void ref_explicit_info(void* h, uint32_t* n, uint64_t* n_acc, uint64_t* m) {
  auto* g = static_cast<ExplicitGraph*>(h);
  *n = g->n;
  *n_acc = g->accepting.size();
  *m = g->edges.size();
}

void ref_explicit_export(void* h, uint32_t* acc, uint32_t* edges) {
  auto* g = static_cast<ExplicitGraph*>(h);
  for (size_t i = 0; i < g->accepting.size(); ++i) acc[i] = g->accepting[i];
  for (size_t i = 0; i < g->edges.size(); ++i) {
    edges[2 * i] = g->edges[i].first;
    edges[2 * i + 1] = g->edges[i].second;
  }
}

void ref_explicit_free(void* h) { delete static_cast<ExplicitGraph*>(h); }

// fill_log (graph.cpp:305-310) + build_snapshot of a parsed explicit graph.
int ref_explicit_snapshot(void* h, int transposed, void** out) {
  REF_TRY
  auto* g = static_cast<ExplicitGraph*>(h);
  EdgeLog::Limits lim;
  lim.max_vertices = g->n > 0 ? g->n : 1;
  lim.max_edges = g->edges.size() > 0 ? g->edges.size() : 1;
  EdgeLog log(lim);
  fill_log(*g, log);
  auto* s = new Snap;
  s->snap = build_snapshot(log, transposed ? Orientation::transposed : Orientation::forward);
  *out = s;
  return 0;
  REF_CATCH
}

// CPU baseline timing: times[] = {gather_build_s, steps_s}; runs Jacobi steps
// of the first MAP fixpoint from all-NIL with `workers` threads until the
// fixpoint, `max_steps`, or `max_seconds` elapses. Returns steps done.
int ref_time_steps(void* h, int workers, uint64_t max_steps, double max_seconds, double* times,
                   uint64_t* steps_done) {
  REF_TRY
  using clk = std::chrono::steady_clock;
  auto* s = static_cast<Snap*>(h);
  if (!s->prop) {
    auto t0 = clk::now();
    s->prop = std::make_unique<MaxPropagation>(s->snap);
    s->prop_s = std::chrono::duration<double>(clk::now() - t0).count();
  }
  const MaxPropagation& kernel = *s->prop;
  WorkerPool pool(workers);
  MapVector x(s->snap.n, MapValue::nil()), nx(s->snap.n, MapValue::nil());
  uint64_t k = 0;
  auto t2 = clk::now();
  while (k < max_steps) {
    StepResult r = kernel.step(x, s->snap.accepting, nx, pool);
    ++k;
    x.swap(nx);
    if (!r.changed) {  // restart the fixpoint so the sample keeps doing full steps
      std::fill(x.begin(), x.end(), MapValue::nil());
    }
    if (std::chrono::duration<double>(clk::now() - t2).count() > max_seconds) break;
  }
  auto t3 = clk::now();
  times[0] = s->prop_s;  // the gather-index build (first call of this snapshot)
  times[1] = std::chrono::duration<double>(t3 - t2).count();
  *steps_done = k;
  return 0;
  REF_CATCH
}

// Times build_snapshot on a generated log (seconds). Log fill is excluded.
int ref_time_build(const void* params, int transposed, double* seconds) {
  REF_TRY
  const auto* p = static_cast<const cyc_gen_params*>(params);
  EdgeLog::Limits lim;
  lim.max_vertices = p->n > 0 ? p->n : 1;
  lim.max_edges = p->m > 0 ? p->m : 1;
  EdgeLog log(lim);
  fill_log(p, log);
  auto t0 = std::chrono::steady_clock::now();
  CsrSnapshot snap = build_snapshot(log, transposed ? Orientation::transposed : Orientation::forward);
  *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return snap.m > 0 ? 0 : 0;
  REF_CATCH
}

int ref_hw_threads() { return (int)std::thread::hardware_concurrency(); }

// SETUP ONLY (not timed, not the reference's code): the CsrSnapshot that
// build_snapshot (graph.cpp:63-105) produces for a generated config, built
// with `threads` threads so that the bench's CPU arm can time the reference's
// own MaxPropagation on config 3 without first spending minutes in the
// single-threaded reference build. Same content: rows keyed by dst
// (transposed) or src, columns ascending and deduplicated, accepting frozen.
// tests/test_oracle.py checks it against build_snapshot itself.
int ref_snapshot_gen_fast(const void* params, int transposed, int threads, void** out) {
  REF_TRY
  const auto* p = static_cast<const cyc_gen_params*>(params);
  if (p->kind == CYC_GEN_PRODUCT) return ref_snapshot_gen(params, transposed, out);
  const uint32_t n = p->n;
  const uint64_t m = p->m;
  const int T = threads > 0 ? threads : 1;
  auto par = [&](auto&& body) {  // body(thread index, begin, end) over [0, m)
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] { body(t, m * t / T, m * (t + 1) / T); });
    for (auto& x : th) x.join();
  };
  std::vector<std::vector<uint32_t>> cnt(T, std::vector<uint32_t>(n + 1, 0));
  par([&](int t, uint64_t b, uint64_t e) {
    for (uint64_t i = b; i < e; ++i) {
      uint32_t sv, dv;
      cyc_gen_edge(p, i, &sv, &dv);
      ++cnt[t][transposed ? dv : sv];
    }
  });
  // raw offsets: row-major, thread-minor (each thread's slice of a row contiguous)
  std::vector<uint64_t> roff(n + 1, 0);
  {
    uint64_t acc = 0;
    for (uint32_t v = 0; v < n; ++v) {
      roff[v] = acc;
      for (int t = 0; t < T; ++t) {
        const uint32_t c = cnt[t][v];
        cnt[t][v] = (uint32_t)acc;  // becomes the thread's cursor (relative base fits: see below)
        acc += c;
      }
    }
    roff[n] = acc;
  }
  std::vector<uint32_t> raw(m ? m : 1);
  // cursors may exceed 2^32 for m >= 2^32; the device limit is m < 2^32 anyway
  par([&](int t, uint64_t b, uint64_t e) {
    for (uint64_t i = b; i < e; ++i) {
      uint32_t sv, dv;
      cyc_gen_edge(p, i, &sv, &dv);
      const uint32_t r = transposed ? dv : sv;
      raw[cnt[t][r]++] = transposed ? sv : dv;
    }
  });
  cnt.clear();
  cnt.shrink_to_fit();
  std::vector<uint32_t> ucnt(n, 0);
  {  // sort + dedup each row in place, rows split over threads
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        for (uint64_t v = t; v < n; v += T) {
          uint32_t* b = raw.data() + roff[v];
          uint32_t* e = raw.data() + roff[v + 1];
          std::sort(b, e);
          ucnt[v] = (uint32_t)(std::unique(b, e) - b);
        }
      });
    for (auto& x : th) x.join();
  }
  auto* s = new Snap;
  CsrSnapshot& sn = s->snap;
  sn.orientation = transposed ? Orientation::transposed : Orientation::forward;
  sn.n = n;
  sn.row_offsets.assign(n + 1ull, 0);
  for (uint32_t v = 0; v < n; ++v) sn.row_offsets[v + 1] = sn.row_offsets[v] + ucnt[v];
  sn.m = sn.row_offsets[n];
  sn.col_indices.resize(sn.m);
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        for (uint64_t v = t; v < n; v += T)
          std::copy(raw.data() + roff[v], raw.data() + roff[v] + ucnt[v], sn.col_indices.data() + sn.row_offsets[v]);
      });
    for (auto& x : th) x.join();
  }
  sn.accepting = Bitset(n);
  for (uint32_t v = 0; v < n; ++v)
    if (cyc_gen_accepting(p, v)) sn.accepting.set(v);
  *out = s;
  return 0;
  REF_CATCH
}

// CPU time to verdict of the reference, phase by phase, the way
// cycheck_main.cpp:88-97 splits it (csr_ms = build_snapshot, kernel_ms =
// run_map) and explore.cpp:93-101 adds the final-round restriction:
//   t[0] log fill (EdgeLog::append_edge for every generated edge, not the
//        reference's work but its input), t[1] build_snapshot,
//   t[2] restrict_to_accepting_sccs (0 if restrict_ == 0),
//   t[3 + i] run_map with MapOptions{workers[i], early_exit} (includes the
//        MaxPropagation gather-index build, map_engine.cpp:144).
// stats[5 i ..] = {cycle, witness (in the log's ids), iterations, kernel_calls,
// demoted_total} of run i.
int ref_ttv(const void* params, int transposed, int restrict_, int early, const int* workers, int nw,
            double* t, uint64_t* stats) {
  REF_TRY
  using clk = std::chrono::steady_clock;
  auto secs = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
  const auto* p = static_cast<const cyc_gen_params*>(params);
  EdgeLog::Limits lim;
  lim.max_vertices = p->n > 0 ? p->n : 1;
  lim.max_edges = p->m > 0 ? p->m : 1;
  auto t0 = clk::now();
  EdgeLog log(lim);
  fill_log(p, log);
  auto t1 = clk::now();
  CsrSnapshot snap = build_snapshot(log, transposed ? Orientation::transposed : Orientation::forward);
  auto t2 = clk::now();
  t[0] = secs(t0, t1);
  t[1] = secs(t1, t2);
  t[2] = 0;
  SccRestriction r;
  const CsrSnapshot* run_on = &snap;
  if (restrict_) {
    auto t3 = clk::now();
    r = restrict_to_accepting_sccs(snap);
    t[2] = secs(t3, clk::now());
    run_on = &r.snapshot;
  }
  for (int i = 0; i < nw; ++i) {
    MapOptions o;
    o.workers = workers[i];
    o.early_exit = early != 0;
    auto t4 = clk::now();
    auto [verdict, st] = run_map(*run_on, run_on->accepting, o);
    t[3 + i] = secs(t4, clk::now());
    uint64_t* out = stats + 5 * i;
    out[0] = verdict.cycle_found();
    out[1] = verdict.witness ? (restrict_ ? r.kept[*verdict.witness] : *verdict.witness) : 0xFFFFFFFFull;
    out[2] = st.iterations;
    out[3] = st.kernel_calls;
    out[4] = st.demoted_total;
  }
  return 0;
  REF_CATCH
}

}  // extern "C"
