// cycheck_b200.hpp — C++ drop-in for the reference's MAP hot path.
//
// Header-only C++17 over the C ABI in cycheck_b200.h. The functions mirror
// /root/reference/proj/include/cycheck/{graph,map_engine}.hpp one for one and
// are templated on the caller's own types, so the reference's call sites
// (tools/cycheck_main.cpp:88-97, src/explore.cpp:71-124) switch by
// qualifying the call and keeping their CsrSnapshot / EdgeLog / Bitset /
// MapOptions / Verdict / MapStats:
//
//     cycheck::b200::Engine gpu;                               // cuda:0
//     auto snap = cycheck::b200::build_snapshot(gpu, log, Orientation::transposed);
//     auto [verdict, stats] = cycheck::b200::run_map<Verdict, MapStats>(snap, accepting, opts);
//
// Requirements on the templated types are exactly the reference members used
// below (EdgeLog::edge/edge_count/vertex_count/accepting_prefix, Bitset::
// words/size, CsrSnapshot::{n,m,row_offsets,col_indices,accepting,
// orientation}, MapOptions::early_exit, Verdict::cycle/no_cycle, MapStats::
// {iterations,kernel_calls,demoted_total,cycle_witness}). Errors surface as
// the reference's exception types when the caller names them (template
// parameters ContractErr / ResourceErr), std::runtime_error otherwise.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <cstdlib>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "cycheck_b200.h"

namespace cycheck {
namespace b200 {

struct DefaultContractError : std::logic_error {
  using std::logic_error::logic_error;
};
struct DefaultResourceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class ContractErr = DefaultContractError, class ResourceErr = DefaultResourceError>
inline void check(cyc_status st) {
  if (st == CYC_OK) return;
  const std::string msg = cyc_last_error();
  if (st == CYC_E_CONTRACT) throw ContractErr(msg);
  if (st == CYC_E_RESOURCE) throw ResourceErr(msg);
  throw std::runtime_error(msg);
}

// One GPU and one CUDA stream (the reference's WorkerPool role, parallel.hpp).
class Engine {
 public:
  explicit Engine(int device = 0) {
    cyc_ctx* c = nullptr;
    check(cyc_ctx_create(device, &c));
    ctx_.reset(c, &cyc_ctx_destroy);
  }
  cyc_ctx* get() const { return ctx_.get(); }
  // Allocates a build's device memory for logs up to m_log edges / n vertices
  // ahead of the first build (cyc_ctx_reserve), by default on a library
  // thread while the caller fills its EdgeLog.
  void reserve(uint64_t m_log, uint32_t n, bool background = true) const {
    check(cyc_ctx_reserve(ctx_.get(), m_log, n, background ? 1 : 0));
  }

 private:
  std::shared_ptr<cyc_ctx> ctx_;
};

// Device-resident snapshot (CsrSnapshot on the GPU, plus its gather index).
class Snapshot {
 public:
  Snapshot() = default;
  Snapshot(const Engine& e, cyc_graph* g) : eng_(e), g_(g, &cyc_graph_destroy) {
    check(cyc_graph_info(g, &n_, &m_, &orientation_, &restricted_));
  }
  uint32_t n() const { return n_; }
  uint64_t m() const { return m_; }
  bool transposed() const { return orientation_ == CYC_TRANSPOSED; }
  cyc_graph* get() const { return g_.get(); }
  const Engine& engine() const { return eng_; }

  // Copies the CSR back into a reference CsrSnapshot-like object.
  template <class Csr>
  void export_to(Csr& out) const {
    out.n = n_;
    out.m = m_;
    out.row_offsets.assign(static_cast<size_t>(n_) + 1, 0);
    out.col_indices.assign(m_, 0);
    std::vector<uint64_t> acc((n_ + 63) / 64 + 1, 0);
    check(cyc_graph_export(g_.get(), out.row_offsets.data(), out.col_indices.data(), acc.data(),
                           nullptr));
    out.accepting = decltype(out.accepting)(n_);
    for (size_t i = 0; i < out.accepting.words().size(); ++i) out.accepting.words()[i] = acc[i];
  }

 private:
  Engine eng_;
  std::shared_ptr<cyc_graph> g_;
  uint32_t n_ = 0;
  uint64_t m_ = 0;
  int orientation_ = CYC_TRANSPOSED;
  int restricted_ = 0;
};

template <class OrientationT>
inline int orientation_code(OrientationT o) {
  return static_cast<int>(o) == 1 ? CYC_TRANSPOSED : CYC_FORWARD;  // types.hpp:12
}

// The logged edges [lo, hi) in device memory. The EdgeLog's 65,536-edge chunks
// (graph.hpp:83-87) are only reachable through EdgeLog::edge(i), so host
// threads gather blocks of kStageEdges edges into two pinned buffers in turn
// while the previous block's H2D copy runs on the context's stream. Measured
// on config 3 (1.07 G edges, 16 host threads): build_snapshot through this
// path 418 ms vs 280 ms for cyc_check from an already pinned contiguous log —
// the gather itself is host-memory bound (8.6 GB read + 8.6 GB written); a
// persistent worker pool with a separate copier thread measured slower (469 ms).
class DeviceLog {
 public:
  static constexpr uint64_t kStageEdges = 1ull << 22;  // 32 MB per pinned block
  template <class EdgeLogT>
  DeviceLog(const Engine& e, const EdgeLogT& log, uint64_t lo, uint64_t hi) : e_(e), m_(hi - lo) {
    if (!m_) return;
    check(cyc_device_alloc(e.get(), m_ * 8, &dev_));
    uint64_t stage = kStageEdges;
    unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (const char* v = std::getenv("CYC_STAGE_LOG2")) stage = 1ull << std::atoi(v);  // tuning knobs
    if (const char* v = std::getenv("CYC_STAGE_THREADS")) nt = (unsigned)std::max(1, std::atoi(v));
    const uint64_t blk = std::min<uint64_t>(stage, m_);
    const uint64_t nb = (m_ + blk - 1) / blk;
    if (nb == 1 || m_ < (1u << 16)) nt = 1;
    uint32_t* pin[2];
    std::unique_lock<std::mutex> lk(staging(blk * 8, pin));  // one upload at a time owns the blocks
    // Workers live for the whole upload: worker t fills slice t of every block
    // (block i into pin[i & 1] once the copy of block i-2 has finished) while
    // this thread issues block i's copy as soon as all slices are in. Spawning
    // the workers per 32 MB block cost ~100 ms on a 2^30-edge log.
    std::unique_ptr<std::atomic<unsigned>[]> filled(new std::atomic<unsigned>[nb]);
    for (uint64_t i = 0; i < nb; ++i) filled[i].store(0, std::memory_order_relaxed);
    std::atomic<uint64_t> free_upto{1};  // blocks <= this may be filled
    std::atomic<bool> abort{false};
    auto work = [&](unsigned t) {
      for (uint64_t i = 0; i < nb; ++i) {
        while (free_upto.load(std::memory_order_acquire) < i) {
          if (abort.load(std::memory_order_relaxed)) return;
          std::this_thread::yield();
        }
        const uint64_t b = i * blk, cnt = std::min(blk, m_ - b);
        const uint64_t s = cnt * t / nt, f = cnt * (t + 1) / nt;
        uint32_t* dst = pin[i & 1];
        for (uint64_t j = s; j < f; ++j) {
          const auto pr = log.edge(lo + b + j);
          dst[2 * j] = pr.first;
          dst[2 * j + 1] = pr.second;
        }
        filled[i].fetch_add(1, std::memory_order_release);
      }
    };
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) th.emplace_back(work, t);
    cyc_status st = CYC_OK;
    for (uint64_t i = 0; i < nb && st == CYC_OK; ++i) {
      while (filled[i].load(std::memory_order_acquire) < nt) std::this_thread::yield();
      if (i >= 1) {
        st = cyc_ctx_synchronize(e.get());  // block i-1's copy is done: its buffer may take block i+1
        free_upto.store(i + 1, std::memory_order_release);
      }
      const uint64_t b = i * blk, cnt = std::min(blk, m_ - b);
      if (st == CYC_OK) st = cyc_memcpy_async(e.get(), static_cast<char*>(dev_) + b * 8, pin[i & 1], cnt * 8);
    }
    if (st == CYC_OK) st = cyc_ctx_synchronize(e.get());
    abort.store(true);
    free_upto.store(nb);
    for (auto& x : th) x.join();
    if (st != CYC_OK) {  // the destructor will not run
      cyc_device_free(e.get(), dev_);
      dev_ = nullptr;
      check(st);
    }
  }
  ~DeviceLog() {
    if (dev_) cyc_device_free(e_.get(), dev_);
  }
  DeviceLog(const DeviceLog&) = delete;
  DeviceLog& operator=(const DeviceLog&) = delete;
  const uint32_t* data() const { return static_cast<const uint32_t*>(dev_); }
  uint64_t size() const { return m_; }

 private:
  // Two pinned staging blocks kept for the process (pinning 2 x 32 MB per
  // upload cost milliseconds every snapshot); one upload at a time uses them.
  static std::unique_lock<std::mutex> staging(uint64_t bytes, uint32_t* (&pin)[2]) {
    static std::mutex mu;
    static void* buf[2] = {nullptr, nullptr};
    static uint64_t cap = 0;
    std::unique_lock<std::mutex> lk(mu);
    if (cap < bytes) {
      for (auto& p : buf) {
        if (p) cyc_host_free(p);
        p = nullptr;
      }
      for (auto& p : buf) check(cyc_host_alloc(bytes, &p));
      cap = bytes;
    }
    pin[0] = static_cast<uint32_t*>(buf[0]);
    pin[1] = static_cast<uint32_t*>(buf[1]);
    return lk;
  }
  Engine e_;
  uint64_t m_ = 0;
  void* dev_ = nullptr;
};

// build_snapshot(log, orientation, m, n) — graph.hpp:97-98. The logged prefix
// goes to the device through DeviceLog's pinned double buffer.
template <class EdgeLogT, class OrientationT>
Snapshot build_snapshot(const Engine& e, const EdgeLogT& log, OrientationT orientation, uint64_t m,
                        uint32_t n) {
  DeviceLog dl(e, log, 0, m);
  auto acc = log.accepting_prefix(n);
  cyc_graph* g = nullptr;
  check(cyc_graph_build(e.get(), dl.data(), m, n, acc.words().data(), orientation_code(orientation), &g));
  return Snapshot(e, g);
}

// build_snapshot(log, orientation) — graph.hpp:101 (edge count captured first).
template <class EdgeLogT, class OrientationT>
Snapshot build_snapshot(const Engine& e, const EdgeLogT& log, OrientationT orientation) {
  const uint64_t m = log.edge_count();
  const uint32_t n = log.vertex_count();
  return build_snapshot(e, log, orientation, m, n);
}

// Incremental snapshot: the snapshot of the prefix (m, n) of
// the same log `prev` was built from, uploading and sorting only the edges
// logged since. Same result as build_snapshot(e, log, orientation, m, n) — what
// the explorer's detector calls every round (explore.cpp:71-124).
template <class EdgeLogT>
Snapshot extend_snapshot(const Snapshot& prev, const EdgeLogT& log, uint64_t m, uint32_t n) {
  uint64_t m_prev = 0;
  check(cyc_graph_log_prefix(prev.get(), &m_prev));
  if (m < m_prev) throw DefaultContractError("extend_snapshot: edge prefix shrinks");
  DeviceLog dl(prev.engine(), log, m_prev, m);
  auto acc = log.accepting_prefix(n);
  cyc_graph* g = nullptr;
  check(cyc_graph_extend(prev.engine().get(), prev.get(), dl.data(), m - m_prev, n, acc.words().data(), &g));
  return Snapshot(prev.engine(), g);
}

// Upload of a host CsrSnapshot (for callers that already built one).
template <class Csr>
Snapshot upload(const Engine& e, const Csr& snap) {
  cyc_graph* g = nullptr;
  check(cyc_graph_from_csr(e.get(), snap.row_offsets.data(), snap.col_indices.data(), snap.n, snap.m,
                           snap.accepting.words().data(), orientation_code(snap.orientation), &g));
  return Snapshot(e, g);
}

// restrict_to_accepting_sccs — graph.hpp:110-114; kept[new] = original id.
inline std::pair<Snapshot, std::vector<uint32_t>> restrict_to_accepting_sccs(const Snapshot& s) {
  cyc_graph* g = nullptr;
  check(cyc_graph_restrict(s.engine().get(), s.get(), &g));
  Snapshot r(s.engine(), g);
  std::vector<uint32_t> kept(r.n());
  check(cyc_graph_export(g, nullptr, nullptr, nullptr, kept.data()));
  return {std::move(r), std::move(kept)};
}

template <class BitsetT>
const uint64_t* words_of(const BitsetT& acc, uint32_t n) {
  if (acc.size() != n) throw DefaultContractError("run_map: accepting set size mismatch");
  return acc.words().data();
}

template <class OptionsT>
cyc_map_options to_c(const OptionsT& o) {
  cyc_map_options c{};
  c.early_exit = o.early_exit ? 1 : 0;
  c.mode = CYC_MODE_AUTO;
  return c;
}

// run_map — map_engine.hpp:111-112 (workers is meaningless on the GPU; the
// result is the same for every worker count).
template <class VerdictT, class StatsT, class BitsetT, class OptionsT>
std::pair<VerdictT, StatsT> run_map(const Snapshot& s, const BitsetT& accepting, const OptionsT& opt) {
  cyc_map_options o = to_c(opt);
  cyc_map_stats st{};
  check(cyc_map_run(s.engine().get(), s.get(), words_of(accepting, s.n()), &o, &st, nullptr, nullptr,
                    nullptr, 0));
  StatsT stats;
  stats.iterations = st.iterations;
  stats.kernel_calls = st.kernel_calls;
  stats.demoted_total = st.demoted_total;
  if (st.cycle_found) {
    stats.cycle_witness = st.witness;
    return {VerdictT::cycle(st.witness), stats};
  }
  return {VerdictT::no_cycle(), stats};
}

// Row-sharded run_map over several GPUs of this process: one
// Engine per device, each rank keeps ~1/N of the snapshot's edges; results
// equal run_map on one device. Engines on the same device run their ranks as
// one grid (tests on one GPU).
class ShardedGraph {
 public:
  template <class EdgeLogT, class OrientationT>
  ShardedGraph(const std::vector<Engine>& engines, const EdgeLogT& log, OrientationT orientation, uint64_t m,
               uint32_t n, int layout = CYC_LAYOUT_AUTO)
      : n_(n) {
    const int world = static_cast<int>(engines.size());
    if (world < 1) throw DefaultContractError("ShardedGraph: no engines");
    auto acc = log.accepting_prefix(n);
    for (int r = 0; r < world; ++r) {
      DeviceLog dl(engines[r], log, 0, m);
      cyc_shard* s = nullptr;
      check(cyc_shard_build(engines[r].get(), dl.data(), m, n, acc.words().data(), orientation_code(orientation),
                            layout, world, r, &s));
      shards_.emplace_back(s, &cyc_shard_destroy);
      engines_.push_back(engines[r]);
    }
    std::vector<cyc_shard*> raw;
    for (auto& s : shards_) raw.push_back(s.get());
    check(cyc_shard_connect_local(raw.data(), world));
  }
  uint32_t n() const { return n_; }
  // edges held by rank r
  uint64_t local_edges(int r) const {
    uint64_t e = 0;
    check(cyc_shard_info(shards_.at(r).get(), nullptr, nullptr, &e, nullptr));
    return e;
  }
  template <class VerdictT, class StatsT, class BitsetT, class OptionsT>
  std::pair<VerdictT, StatsT> run_map(const BitsetT& accepting, const OptionsT& opt) const {
    if (accepting.size() != n_) throw DefaultContractError("run_map: accepting set size mismatch");
    std::vector<cyc_shard*> raw;
    for (auto& s : shards_) raw.push_back(s.get());
    cyc_map_options o{};
    o.early_exit = opt.early_exit ? 1 : 0;
    cyc_map_stats st{};
    check(cyc_shard_run_map(raw.data(), static_cast<int>(raw.size()), accepting.words().data(), &o, &st, nullptr,
                            nullptr, nullptr, 0));
    StatsT stats;
    stats.iterations = st.iterations;
    stats.kernel_calls = st.kernel_calls;
    stats.demoted_total = st.demoted_total;
    if (st.cycle_found) {
      stats.cycle_witness = st.witness;
      return {VerdictT::cycle(st.witness), stats};
    }
    return {VerdictT::no_cycle(), stats};
  }

 private:
  uint32_t n_ = 0;
  std::vector<Engine> engines_;
  std::vector<std::shared_ptr<cyc_shard>> shards_;
};

// fixpoint — map_engine.hpp:86-87; fills values with map codes (id+1, 0 NIL).
template <class BitsetT, class OptionsT>
uint64_t fixpoint(const Snapshot& s, const BitsetT& accepting, const OptionsT& opt,
                  std::vector<uint32_t>& values, uint32_t& witness) {
  cyc_map_options o = to_c(opt);
  values.assign(s.n(), 0);
  uint64_t steps = 0;
  check(cyc_fixpoint(s.engine().get(), s.get(), words_of(accepting, s.n()), &o, values.data(), &steps,
                     &witness));
  return steps;
}

// demote — map_engine.hpp:99; remaining words (F \ D) and D ascending.
template <class BitsetT>
std::vector<uint32_t> demote(const Engine& e, const std::vector<uint32_t>& values, const BitsetT& accepting,
                             std::vector<uint64_t>& remaining) {
  const uint32_t n = static_cast<uint32_t>(values.size());
  remaining.assign((n + 63) / 64 + 1, 0);
  std::vector<uint32_t> d(n + 1);
  uint64_t nd = 0;
  check(cyc_demote(e.get(), values.data(), n, words_of(accepting, n), remaining.data(), d.data(), &nd));
  d.resize(nd);
  return d;
}

// run_owcty — owcty.hpp:28-31 over the snapshot relation (the reference runs
// it on a forward snapshot, cycheck_main.cpp:98-106). StatsT is the
// reference's OwctyStats (outer_iterations, reach_ms, elim_ms, final_size).
template <class VerdictT, class StatsT, class BitsetT>
std::pair<VerdictT, StatsT> run_owcty(const Snapshot& s, const BitsetT& accepting) {
  if (accepting.size() != s.n()) throw DefaultContractError("run_owcty: accepting set size mismatch");
  int32_t cyc = 0;
  uint32_t w = 0;
  cyc_owcty_stats st{};
  check(cyc_owcty(s.engine().get(), s.get(), accepting.words().data(), &cyc, &w, &st));
  StatsT stats;
  stats.outer_iterations = st.outer_iterations;
  stats.reach_ms = st.reach_ms;
  stats.elim_ms = st.elim_ms;
  stats.final_size = st.final_size;
  return {cyc ? VerdictT::cycle(w) : VerdictT::no_cycle(), stats};
}

// scc_verdict — oracle.cpp:32-98 on the snapshot relation: the verdict and the
// accepting vertices of cyclic SCCs (ascending).
template <class VerdictT>
VerdictT scc_verdict(const Snapshot& s, std::vector<uint32_t>* cyclic_accepting = nullptr) {
  int32_t cyc = 0;
  uint32_t w = 0;
  uint64_t k = 0;
  std::vector<uint32_t> buf(cyclic_accepting ? s.n() + 1 : 0);
  check(cyc_scc_verdict(s.engine().get(), s.get(), &cyc, &w, cyclic_accepting ? buf.data() : nullptr, &k));
  if (cyclic_accepting) {
    buf.resize(k);
    *cyclic_accepting = std::move(buf);
  }
  return cyc ? VerdictT::cycle(w) : VerdictT::no_cycle();
}

}  // namespace b200
}  // namespace cycheck
