// dropin_test.cpp — TEST INFRASTRUCTURE ONLY.
//
// Builds against the reference's own headers and sources (oracle/Makefile,
// target `dropin`) and checks that the C++ drop-in (include/cycheck_b200.hpp)
// returns what the reference returns when a reference call site switches to
// it: same Verdict, witness and MapStats from cycheck::run_map, the same CSR
// from build_snapshot, the same restriction. Runs on a GPU box (the binary is
// prebuilt into oracle/_ref/ and shipped); exits non-zero on any mismatch.
#include <algorithm>
#include <cstdio>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "cycheck/graph.hpp"
#include "cycheck/map_engine.hpp"
#include "cycheck/oracle.hpp"
#include "cycheck/owcty.hpp"
#include "../include/cycheck_b200.hpp"

using namespace cycheck;

int main(int argc, char** argv) {
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
