// dropin_test.cpp — TEST INFRASTRUCTURE ONLY.
//
// Builds against the reference's own headers and sources (oracle/Makefile,
// target `dropin`) and checks that the C++ drop-in (include/cycheck_b200.hpp)
// returns what the reference returns when a reference call site switches to
// it: same Verdict, witness and MapStats from cycheck::run_map, the same CSR
// from build_snapshot, the same restriction. Runs on a GPU box (the binary is
// prebuilt into oracle/_ref/ and shipped); exits non-zero on any mismatch.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>

#include "cycheck/graph.hpp"
#include "cycheck/map_engine.hpp"
#include "cycheck/oracle.hpp"
#include "cycheck/owcty.hpp"
#include "../include/cycheck_b200.hpp"
#include "../include/cyc_gen.h"

using namespace cycheck;

// `dropin_test time <scale>`: the cycheck_main.cpp:88-97 path (build_snapshot
// from the reference's EdgeLog + run_map) through the drop-in, timed against
// cyc_check from a contiguous pinned copy of the same log (R-MAT, config 3's
// generator at the given scale). Prints one JSON line.
static int time_dropin(int scale) {
  using clk = std::chrono::steady_clock;
  auto ms = [](clk::time_point a) { return std::chrono::duration<double, std::milli>(clk::now() - a).count(); };
  cyc_gen_params p;
  cyc_gen_config(&p, 3);
  p.scale = (uint32_t)scale;
  cyc_gen_init(&p);
  b200::Engine gpu(0);
  EdgeLog log({p.n, p.m});
  auto t0 = clk::now();
  for (uint32_t v = 0; v < p.n; ++v) log.add_vertex(cyc_gen_accepting(&p, v) != 0);
  for (uint64_t i = 0; i < p.m; ++i) {
    uint32_t s, d;
    cyc_gen_edge(&p, i, &s, &d);
    log.append_edge(s, d);
  }
  const double fill_ms = ms(t0);
  // contiguous pinned copy of the same edges
  void* pin = nullptr;
  b200::check(cyc_host_alloc(p.m * 8, &pin));
  for (uint64_t i = 0; i < p.m; ++i) {
    auto e = log.edge(i);
    static_cast<uint32_t*>(pin)[2 * i] = e.first;
    static_cast<uint32_t*>(pin)[2 * i + 1] = e.second;
  }
  const Bitset acc = log.accepting_prefix(p.n);
  // DROPIN_VARIANTS="log2:threads,...": DeviceLog staging block / fill threads sweep
  if (const char* vs = std::getenv("DROPIN_VARIANTS")) {
    std::string all(vs);
    size_t pos = 0;
    while (pos < all.size()) {
      size_t q = all.find(',', pos);
      if (q == std::string::npos) q = all.size();
      const std::string item = all.substr(pos, q - pos);
      pos = q + 1;
      const size_t c = item.find(':');
      setenv("CYC_STAGE_LOG2", item.substr(0, c).c_str(), 1);
      setenv("CYC_STAGE_THREADS", item.substr(c + 1).c_str(), 1);
      double best = 1e30;
      for (int rep = 0; rep < 3; ++rep) {
        auto tb = clk::now();
        b200::DeviceLog dl(gpu, log, 0, p.m);
        best = std::min(best, ms(tb));
      }
      std::printf("{\"variant\": \"%s\", \"device_log_ms\": %.2f}\n", item.c_str(), best);
    }
    unsetenv("CYC_STAGE_LOG2");
    unsetenv("CYC_STAGE_THREADS");
  }
  double best_drop = 1e30, best_pin = 1e30, csr_ms = 0, kernel_ms = 0;
  bool same = true;
  for (int rep = 0; rep < 3; ++rep) {
    auto tb = clk::now();
    auto snap = b200::build_snapshot(gpu, log, Orientation::transposed);
    const double c = ms(tb);
    auto tk = clk::now();
    auto [v, st] = b200::run_map<Verdict, MapStats>(snap, log.accepting_prefix(snap.n()), MapOptions{});
    const double k = ms(tk);
    if (c + k < best_drop) {
      best_drop = c + k;
      csr_ms = c;
      kernel_ms = k;
    }
    cyc_map_options o{};
    o.early_exit = 1;
    cyc_map_stats cs{};
    auto tp = clk::now();
    b200::check(cyc_check(gpu.get(), static_cast<const uint32_t*>(pin), p.m, p.n, acc.words().data(),
                          CYC_TRANSPOSED, 0, &o, &cs, nullptr));
    best_pin = std::min(best_pin, ms(tp));
    same = same && cs.cycle_found == (int)v.cycle_found() && cs.kernel_calls == st.kernel_calls;
  }
  cyc_host_free(pin);
  std::printf("{\"scale\": %d, \"m_log\": %llu, \"log_fill_ms\": %.1f, \"dropin_ms\": %.2f, \"csr_ms\": %.2f, "
              "\"kernel_ms\": %.2f, \"pinned_cyc_check_ms\": %.2f, \"ratio\": %.3f, \"same_verdict\": %s}\n",
              scale, (unsigned long long)p.m, fill_ms, best_drop, csr_ms, kernel_ms, best_pin, best_drop / best_pin,
              same ? "true" : "false");
  return same ? 0 : 1;
}

int main(int argc, char** argv) {
  if (argc > 2 && std::strcmp(argv[1], "time") == 0) return time_dropin(std::atoi(argv[2]));
  const int trials = argc > 1 ? std::atoi(argv[1]) : 200;
  b200::Engine gpu(0);
  std::mt19937_64 rng(0x0912255);
  int bad = 0;
  for (int t = 0; t < trials; ++t) {
    const uint32_t n = 1 + rng() % 400;
    const uint64_t m = rng() % (4 * n + 1);
    EdgeLog log({n, m ? m : 1});
    for (uint32_t v = 0; v < n; ++v) log.add_vertex(rng() % 100 < (t % 2 ? 5u : 30u));
    for (uint64_t i = 0; i < m; ++i) log.append_edge(rng() % n, rng() % n);
    for (Orientation o : {Orientation::transposed, Orientation::forward}) {
      if (std::getenv("DROPIN_TRACE")) std::fprintf(stderr, "trial %d orient %d n %u m %llu\n", t, (int)o, n,
                                                    (unsigned long long)m);
      CsrSnapshot ref = build_snapshot(log, o);
      b200::Snapshot dev = b200::build_snapshot(gpu, log, o);
      CsrSnapshot back;
      dev.export_to(back);
      if (back.row_offsets != ref.row_offsets || back.col_indices != ref.col_indices ||
          !(back.accepting == ref.accepting)) {
        std::printf("trial %d: build_snapshot differs\n", t);
        ++bad;
      }
      b200::Snapshot up = b200::upload(gpu, ref);
      // incremental: snapshot of a prefix (vertex prefix = just enough for
      // its edges), extended to the whole log
      {
        const uint64_t mh = m / 2;
        uint32_t nh = 0;
        for (uint64_t i = 0; i < mh; ++i) {
          auto e = log.edge(i);
          nh = std::max(nh, std::max(e.first, e.second) + 1);
        }
        b200::Snapshot half = b200::build_snapshot(gpu, log, o, mh, nh);
        b200::Snapshot ext = b200::extend_snapshot(half, log, m, n);
        CsrSnapshot eb;
        ext.export_to(eb);
        if (eb.row_offsets != ref.row_offsets || eb.col_indices != ref.col_indices ||
            !(eb.accepting == ref.accepting)) {
          std::printf("trial %d: extend_snapshot differs\n", t);
          ++bad;
        }
      }
      for (bool early : {true, false}) {
        MapOptions opts;
        opts.early_exit = early;
        auto [rv, rs] = run_map(ref, ref.accepting, opts);
        auto [gv, gs] = b200::run_map<Verdict, MapStats>(dev, ref.accepting, opts);
        auto [uv, us] = b200::run_map<Verdict, MapStats>(up, ref.accepting, opts);
        for (auto* p : {&gv, &uv}) {
          if (!(*p == rv)) {
            std::printf("trial %d: verdict differs\n", t);
            ++bad;
          }
        }
        for (auto* p : {&gs, &us}) {
          if (p->iterations != rs.iterations || p->kernel_calls != rs.kernel_calls ||
              p->demoted_total != rs.demoted_total || p->cycle_witness != rs.cycle_witness) {
            std::printf("trial %d: stats differ (%llu/%llu vs %llu/%llu)\n", t,
                        (unsigned long long)p->iterations, (unsigned long long)p->kernel_calls,
                        (unsigned long long)rs.iterations, (unsigned long long)rs.kernel_calls);
            ++bad;
          }
        }
      }
      if (std::getenv("DROPIN_TRACE")) std::fprintf(stderr, "  run_map done\n");
      // explore.cpp-style caller on a row-sharded graph (ranks emulated on this GPU)
      if (t % 8 == 0) {
        std::vector<b200::Engine> engines = {gpu, gpu, gpu};
        b200::ShardedGraph sg(engines, log, o, m, n);
        for (bool early : {true, false}) {
          MapOptions mo;
          mo.early_exit = early;
          auto [rv, rs] = run_map(ref, ref.accepting, mo);
          auto [sv, ss] = sg.run_map<Verdict, MapStats>(ref.accepting, mo);
          if (!(sv == rv) || ss.iterations != rs.iterations || ss.kernel_calls != rs.kernel_calls ||
              ss.demoted_total != rs.demoted_total) {
            std::printf("trial %d: sharded run_map differs\n", t);
            ++bad;
          }
        }
      }
      // OWCTY and the SCC verdict through the drop-in (owcty.hpp, oracle.hpp)
      auto [ov, os] = run_owcty(ref, ref.accepting);
      auto [gov, gos] = b200::run_owcty<Verdict, OwctyStats>(dev, ref.accepting);
      if (!(gov == ov) || gos.outer_iterations != os.outer_iterations || gos.final_size != os.final_size) {
        std::printf("trial %d: run_owcty differs\n", t);
        ++bad;
      }
      const Verdict sv = scc_verdict(ref.edge_list(), ref.n, ref.accepting, ~0ull).verdict;
      if (b200::scc_verdict<Verdict>(dev).cycle_found() != sv.cycle_found()) {
        std::printf("trial %d: scc_verdict differs\n", t);
        ++bad;
      }
      if (std::getenv("DROPIN_TRACE")) std::fprintf(stderr, "  owcty+scc done\n");
      SccRestriction rr = restrict_to_accepting_sccs(ref);
      auto [gr, kept] = b200::restrict_to_accepting_sccs(dev);
      CsrSnapshot grb;
      gr.export_to(grb);
      if (kept != rr.kept || grb.row_offsets != rr.snapshot.row_offsets ||
          grb.col_indices != rr.snapshot.col_indices) {
        std::printf("trial %d: restriction differs\n", t);
        ++bad;
      }
    }
  }
  std::printf("dropin_test: %d trials, %d mismatches\n", trials, bad);
  return bad ? 1 : 0;
}
