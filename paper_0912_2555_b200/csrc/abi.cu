// abi.cu — the extern "C" boundary (include/cycheck_b200.h).
//
// Each entry point mirrors one reference operation (cited per function),
// stages host inputs onto the context's stream, runs the device kernels and
// copies results back. C++ exceptions never cross the ABI: they become
// status codes plus a thread-local message (errors.hpp:10-22 mapping).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>
#include <pthread.h>
#include <string>
#include <vector>

#include "../../include/cyc_gen.h"
#include "extend.cuh"
#include "fused.cuh"
#include "gen.cuh"
#include "ingest.cuh"
#include "map_run.cuh"
#include "plan.cuh"
#include "shard.cuh"
#include "owcty.cuh"
#include "scc.cuh"

std::atomic<uint64_t> cyc::g_launches{0};

namespace {
thread_local std::string g_err;
thread_local int g_parse[3] = {0, 0, 0};  // code, line, col of the last CYC_E_PARSE
}

[[noreturn]] void cyc::throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  cyc_status code = e == cudaErrorMemoryAllocation ? CYC_E_RESOURCE : CYC_E_CUDA;
  throw Error(code, std::string(cudaGetErrorName(e)) + " (" + cudaGetErrorString(e) + ") at " +
                        what + " [" + file + ":" + std::to_string(line) + "]");
}

namespace {
struct BigBlock {
  void* p;
  size_t cap;
  int device;
  cudaEvent_t ready;  // recorded on the releasing stream
};
std::mutex g_big_mu;
std::vector<BigBlock> g_big_free;

void big_drop_all(int device, cudaStream_t st) {  // caller holds g_big_mu
  for (size_t i = 0; i < g_big_free.size();) {
    BigBlock& b = g_big_free[i];
    if (b.device != device) {
      ++i;
      continue;
    }
    cudaStreamWaitEvent(st, b.ready, 0);
    cudaEventDestroy(b.ready);
    cudaFreeAsync(b.p, st);
    g_big_free[i] = g_big_free.back();
    g_big_free.pop_back();
  }
}
}  // namespace

namespace {
void big_trim(int device, cudaStream_t st) {  // a context goes away: hand the cached blocks back
  std::lock_guard<std::mutex> lk(g_big_mu);
  big_drop_all(device, st);
}
}  // namespace

namespace {
std::mutex g_coop_mu;
cudaEvent_t g_coop_last[64] = {};  // per device: completion of the latest cooperative grid
}  // namespace

void cyc::coop_launch(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t st) {
  int dev = 0;
  CYC_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_coop_mu);
  cudaEvent_t& last = g_coop_last[dev & 63];
  if (last) CYC_CUDA(cudaStreamWaitEvent(st, last, 0));
  else CYC_CUDA(cudaEventCreateWithFlags(&last, cudaEventDisableTiming));
  CYC_CUDA(cudaLaunchCooperativeKernel(fn, grid, block, args, smem, st));
  CYC_CUDA(cudaEventRecord(last, st));
}

void* cyc::big_alloc(size_t n, cudaStream_t st, size_t* cap) {
  int dev = 0;
  CYC_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_big_mu);
  size_t best = SIZE_MAX;
  for (size_t i = 0; i < g_big_free.size(); ++i) {
    const BigBlock& b = g_big_free[i];
    if (b.device == dev && b.cap >= n && b.cap <= n + n / 4 + (64ull << 20) &&
        (best == SIZE_MAX || b.cap < g_big_free[best].cap))
      best = i;
  }
  if (best != SIZE_MAX) {
    BigBlock b = g_big_free[best];
    g_big_free[best] = g_big_free.back();
    g_big_free.pop_back();
    CYC_CUDA(cudaStreamWaitEvent(st, b.ready, 0));
    cudaEventDestroy(b.ready);
    *cap = b.cap;
    return b.p;
  }
  const size_t c = (n + (2ull << 20) - 1) & ~((2ull << 20) - 1);
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, c, st);
  if (e == cudaErrorMemoryAllocation) {  // give the cached blocks back and retry
    cudaGetLastError();
    big_drop_all(dev, st);
    e = cudaMallocAsync(&p, c, st);
  }
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw Error(CYC_E_RESOURCE, "device memory exhausted allocating " + std::to_string(n) + " bytes");
  }
  CYC_CUDA(e);
  *cap = c;
  return p;
}

void cyc::big_free(void* p, size_t cap, cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaEvent_t ev = nullptr;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventRecord(ev, st) != cudaSuccess) {
    cudaGetLastError();
    if (ev) cudaEventDestroy(ev);
    cudaFreeAsync(p, st);
    return;
  }
  std::lock_guard<std::mutex> lk(g_big_mu);
  g_big_free.push_back(BigBlock{p, cap, dev, ev});
}

// A context lives until cyc_ctx_destroy was called AND its last graph is gone
// (graphs keep a reference), so teardown order between them does not matter.
struct cyc_ctx {
  int device = 0;
  cudaStream_t s = nullptr;
  cudaStream_t own = nullptr;  // the context's own stream (s may be an external one)
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr, e3 = nullptr;
  cyc::DevBuf flush;
  cyc::BuildArena arena;  // grow-only build temporaries, reused by every build
  // the second CSR of a large build runs on its own stream / arena / host
  // thread, overlapping the first (created on first use)
  cudaStream_t s2 = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cyc::BuildArena arena2;
  std::thread reserver;  // cyc_ctx_reserve(background): maps pool memory off the caller's thread
  std::atomic<int> refs{1};
};

namespace {
void big_trim(int device, cudaStream_t st);
// builds wait for a background cyc_ctx_reserve (it owns the arenas meanwhile)
void join_reserve(cyc_ctx* ctx) {
  if (ctx->reserver.joinable()) ctx->reserver.join();
}
void ctx_release(cyc_ctx* ctx) {
  if (ctx->refs.fetch_sub(1) != 1) return;
  join_reserve(ctx);
  cudaSetDevice(ctx->device);
  ctx->flush.release();
  ctx->arena = cyc::BuildArena();
  ctx->arena2 = cyc::BuildArena();
  big_trim(ctx->device, ctx->s);
  cudaStreamSynchronize(ctx->s);
  cudaEventDestroy(ctx->e0);
  cudaEventDestroy(ctx->e1);
  cudaEventDestroy(ctx->e2);
  cudaEventDestroy(ctx->e3);
  cudaStreamDestroy(ctx->own);
  if (ctx->s2) {
    cudaStreamSynchronize(ctx->s2);
    cudaStreamDestroy(ctx->s2);
    cudaEventDestroy(ctx->ev_in);
    cudaEventDestroy(ctx->ev_out);
  }
  delete ctx;
}
}  // namespace

struct cyc_fused {
  cyc_ctx* ctx = nullptr;
  const cyc_graph* g = nullptr;
  cyc::FusedShard sh;
};

struct cyc_shard {
  cyc_ctx* ctx = nullptr;
  cyc::ShardGraph g;
};

struct cyc_explicit {
  cyc_ctx* ctx = nullptr;
  cyc::ExplicitDev g;
};

struct cyc_graph {
  cyc_ctx* ctx = nullptr;
  int orientation = CYC_TRANSPOSED;
  int restricted = 0;
  uint64_t m_log = 0;  // logged-edge prefix the snapshot was built from (extend needs it)
  cyc::DevCsr snap;  // the snapshot relation (rows as CsrSnapshot), push side
  cyc::DevCsr gath;  // its reverse: the MaxPropagation gather index, pull side
  cyc::DevBuf acc;   // u64 words
  cyc::DevBuf kept;  // u32[n] original ids (restricted graphs)
  cyc::RunWs ws;
  cyc::MapPlan plan;  // storage layout of the MAP loop (plan.cuh), built on first use
  uint64_t runs = 0;  // MAP loops run on this graph (auto layout builds the plan from the second)
  uint32_t n() const { return gath.n; }
};

namespace {

using cyc::DevBuf;
using cyc::Error;

// CYC_TRACE_CALLS=1: enter/exit lines per ABI call and thread (diagnostics)
struct CallTrace {
  const char* name;
  bool on;
  explicit CallTrace(const char* n) : name(n), on(std::getenv("CYC_TRACE_CALLS") != nullptr) {
    if (on) std::fprintf(stderr, "[cyc %zx] enter %s\n", (size_t)pthread_self() & 0xFFFFFF, name);
  }
  ~CallTrace() {
    if (on) std::fprintf(stderr, "[cyc %zx] exit %s\n", (size_t)pthread_self() & 0xFFFFFF, name);
  }
};

// Calls from different contexts run concurrently (one call in flight per
// context is the contract). Round 1 serialised every call behind one
// process-wide lock to stop an intermittent hang of threads with their own
// contexts; its cause was a race in the frontier engine's solo mode (a block
// could read a level length that CTA 0 had already rewritten, frontier.cuh),
// fixed in round 2. CYC_SERIALIZE=1 restores the lock (diagnostics).
std::recursive_mutex g_api_mu;
const bool g_serialize = [] {
  const char* e = std::getenv("CYC_SERIALIZE");
  return e && e[0] == '1';
}();

template <class F>
cyc_status guard(F&& f) {
  std::unique_lock<std::recursive_mutex> api_lock(g_api_mu, std::defer_lock);
  if (g_serialize) api_lock.lock();
  try {
    f();
    return CYC_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const cyc::ParseFailure& e) {  // ParseError::what(), errors.cpp:18-22
    static const char* names[] = {"syntax", "unknown-identifier", "type-mismatch", "duplicate-name",
                                  "property-restriction", "range"};
    g_err = std::to_string(e.line) + ":" + std::to_string(e.col) + ": error[" + names[e.code] + "]: " + e.what();
    g_parse[0] = e.code;
    g_parse[1] = e.line;
    g_parse[2] = e.col;
    return CYC_E_PARSE;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return CYC_E_RESOURCE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CYC_E_CUDA;
  }
}

void require(bool ok, cyc_status code, const char* msg) {
  if (!ok) throw Error(code, msg);
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Returns a device view of `p` (copying host data into tmp on stream s).
template <class T>
const T* stage_in(const T* p, size_t count, DevBuf& tmp, cudaStream_t s) {
  if (!p || count == 0) return p;
  if (is_device_ptr(p)) return p;
  tmp.alloc(count * sizeof(T), s);
  CYC_CUDA(cudaMemcpyAsync(tmp.p, p, count * sizeof(T), cudaMemcpyHostToDevice, s));
  return tmp.as<T>();
}

// Copies `count` items from device src to dst (host or device).
template <class T>
void copy_out(T* dst, const T* src, size_t count, cudaStream_t s) {
  if (!dst || count == 0) return;
  CYC_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDefault, s));
}

size_t acc_words64(uint32_t n) { return ((size_t)n + 63) / 64; }

__global__ void k_trim_tail(uint64_t* w, uint32_t n) {
  if (n & 63u) w[n >> 6] &= (1ull << (n & 63u)) - 1ull;
}

// Device copy of an accepting set (trimmed), from host/device words or zero.
void load_acc(const uint64_t* words, uint32_t n, DevBuf& dst, cudaStream_t s) {
  size_t nw = acc_words64(n);
  dst.alloc((nw + 1) * 8, s);
  CYC_CUDA(cudaMemsetAsync(dst.p, 0, (nw + 1) * 8, s));
  if (words && nw) {
    CYC_CUDA(cudaMemcpyAsync(dst.p, words, nw * 8, cudaMemcpyDefault, s));
    k_trim_tail<<<1, 1, 0, s>>>(dst.as<uint64_t>(), n);
    CYC_LAUNCHED();
  }
}

__global__ void k_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

void export_offsets(const cyc::DevCsr& g, uint64_t* dst, cudaStream_t s) {
  if (!dst) return;
  DevBuf wide(((size_t)g.n + 1) * 8, s);
  k_u32_to_u64<<<cyc::grid_for(g.n + 1ull, 256, 4), 256, 0, s>>>(g.o(), wide.as<uint64_t>(), g.n + 1ull);
  CYC_LAUNCHED();
  copy_out(dst, wide.as<uint64_t>(), (size_t)g.n + 1, s);
  CYC_CUDA(cudaStreamSynchronize(s));
}

__global__ void k_gen(cyc_gen_params p, uint32_t* edges, uint64_t* acc, uint64_t nwords) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < p.m; i += stride) {
    uint32_t a, b;
    cyc_gen_edge(&p, i, &a, &b);
    reinterpret_cast<uint2*>(edges)[i] = make_uint2(a, b);
  }
  if (acc) {
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords; w += stride) {
      uint64_t bits = 0;
      for (uint32_t k = 0; k < 64; ++k) {
        uint64_t v = w * 64 + k;
        if (v < p.n && cyc_gen_accepting(&p, (uint32_t)v)) bits |= 1ull << k;
      }
      acc[w] = bits;
    }
  }
}

constexpr uint64_t kOverlapEdges = 1ull << 24;  // smaller logs build both CSRs in sequence

void build_graph(cyc_ctx* ctx, const uint32_t* edges, uint64_t m_log, uint32_t n,
                 const uint64_t* acc_words, int orientation, cyc_graph* g) {
  require(orientation == CYC_FORWARD || orientation == CYC_TRANSPOSED, CYC_E_CONTRACT,
          "build_snapshot: bad orientation");
  require(n < 0x80000000u, CYC_E_RESOURCE, "vertex count must be < 2^31");
  require(m_log < 0xFFFFFFFFull, CYC_E_RESOURCE, "edge log prefix must be < 2^32");
  require(m_log == 0 || edges, CYC_E_CONTRACT, "build_snapshot: null edge array");
  join_reserve(ctx);
  cudaStream_t s = ctx->s;
  DevBuf tmp_edges, err(16, s);
  CYC_CUDA(cudaMemsetAsync(err.p, 0, 16, s));
  const uint32_t* de = stage_in(edges, (size_t)m_log * 2, tmp_edges, s);
  g->ctx = ctx;
  g->orientation = orientation;
  g->m_log = m_log;
  const int snap_key_dst = orientation == CYC_TRANSPOSED;
  if (m_log >= kOverlapEdges && !std::getenv("CYC_BUILD_SEQUENTIAL")) {
    // the two CSRs are independent given the log: the gather index is built
    // on a second stream by a helper thread (every phase has host syncs, so
    // one thread cannot keep both streams busy), overlapping the snapshot
    if (!ctx->s2) {
      CYC_CUDA(cudaStreamCreateWithFlags(&ctx->s2, cudaStreamNonBlocking));
      CYC_CUDA(cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming));
      CYC_CUDA(cudaEventCreateWithFlags(&ctx->ev_out, cudaEventDisableTiming));
    }
    CYC_CUDA(cudaEventRecord(ctx->ev_in, s));
    std::exception_ptr helper_err;
    std::thread helper([&] {
      try {
        CYC_CUDA(cudaSetDevice(ctx->device));
        CYC_CUDA(cudaStreamWaitEvent(ctx->s2, ctx->ev_in, 0));
        cyc::build_csr(de, m_log, n, !snap_key_dst, ctx->s2, g->gath, err.as<uint32_t>(), ctx->arena2);
        CYC_CUDA(cudaEventRecord(ctx->ev_out, ctx->s2));
      } catch (...) {
        helper_err = std::current_exception();
      }
    });
    std::exception_ptr main_err;
    try {
      cyc::build_csr(de, m_log, n, snap_key_dst, s, g->snap, err.as<uint32_t>(), ctx->arena);
    } catch (...) {
      main_err = std::current_exception();
    }
    helper.join();
    if (main_err || helper_err) {
      // nothing queued on s2 may outlive the staged log and err (allocated on s)
      cudaStreamSynchronize(ctx->s2);
      std::rethrow_exception(main_err ? main_err : helper_err);
    }
    CYC_CUDA(cudaStreamWaitEvent(s, ctx->ev_out, 0));
    // the gather CSR was allocated on s2; release it on s, after everything
    // that reads it (DevBuf frees on its stream, and the block cache reuses
    // blocks in that stream's order)
    g->gath.off.s = s;
    g->gath.col.s = s;
  } else {
    cyc::build_csr(de, m_log, n, snap_key_dst, s, g->snap, err.as<uint32_t>(), ctx->arena);
    cyc::build_csr(de, m_log, n, !snap_key_dst, s, g->gath, err.as<uint32_t>(), ctx->arena);
  }
  const bool dbg = std::getenv("CYC_DEBUG_TIMING") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  uint32_t herr = 0;
  CYC_CUDA(cudaMemcpyAsync(&herr, err.p, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  require(herr == 0, CYC_E_CONTRACT, "build_snapshot: edge endpoint >= n (not interned)");
  require(g->snap.m == g->gath.m, CYC_E_CUDA, "internal: snapshot/gather edge counts differ");
  cyc::build_heavy(g->gath, cyc::kHeavyDeg, cyc::kHeavyChunk, s, cyc::pull_col_blocks(g->gath.n));
  cyc::build_heavy(g->snap, cyc::kHeavyDeg, cyc::kHeavyChunk, s);
  cyc::build_ell(g->gath, s);
  load_acc(acc_words, n, g->acc, s);
  if (dbg) {
    CYC_CUDA(cudaStreamSynchronize(s));
    std::fprintf(stderr, "[cyc build] heavy+ell+acc  %9.3f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
}

void fill_stats(const cyc::RunOut& o, cyc_map_stats* st) {
  if (!st) return;
  std::memset(st, 0, sizeof *st);
  st->cycle_found = (int32_t)o.res[cyc::kResCycle];
  st->witness = (uint32_t)o.res[cyc::kResWitness];
  st->iterations = o.res[cyc::kResIterations];
  st->kernel_calls = o.res[cyc::kResKernelCalls];
  st->demoted_total = o.res[cyc::kResDemoted];
  st->steps_last = o.res[cyc::kResStepsLast];
  st->pull_steps = o.res[cyc::kResPullSteps];
  st->push_steps = o.res[cyc::kResPushSteps];
  st->edges_touched = o.res[cyc::kResEdges];
  st->rows_touched = o.res[cyc::kResRows];
  st->algorithmic_bytes = o.res[cyc::kResBytes];
  st->loop_ms = o.ms;
  st->grid_blocks = o.grid;
  st->block_threads = o.block;
  st->plan_ms = o.plan_ms;
  st->layout = o.layout;
  st->world = 1;
  st->exchanged_rows = 0;
}

cyc_map_options default_opts() {
  cyc_map_options o;
  std::memset(&o, 0, sizeof o);
  o.early_exit = 1;
  return o;
}

// Common body of fixpoint/run_map: loads F, launches the device loop.
cyc::RunOut run_loop(cyc_ctx* ctx, cyc_graph* g, const uint64_t* acc_words,
                     const cyc_map_options& o, uint64_t cap) {
  cudaStream_t s = ctx->s;
  const uint32_t n = g->n();
  require(o.mode >= CYC_MODE_AUTO && o.mode <= CYC_MODE_PUSH, CYC_E_CONTRACT, "bad mode");
  require(o.layout >= CYC_LAYOUT_AUTO && o.layout <= CYC_LAYOUT_DEGREE, CYC_E_CONTRACT, "bad layout");
  const auto tp = std::chrono::steady_clock::now();
  // Auto layout: a graph's first loop runs in id order and the storage plan
  // is built from its second loop on. The plan costs ~36 ms on config 3,
  // more than it saves in one loop (8 steps: 19 ms; an early-exit verdict
  // after 2 steps: 4 ms), so one-shot checks (cyc_check, a verdict per
  // snapshot) never pay it and repeated runs amortise it.
  int layout = o.layout;
  if (layout == CYC_LAYOUT_AUTO && g->runs == 0 && !(g->plan.decided && g->plan.layout == CYC_LAYOUT_AUTO))
    layout = CYC_LAYOUT_IDENTITY;
  ++g->runs;
  const bool planned = cyc::build_plan(g->snap, g->gath, layout, g->plan, s);
  const double plan_ms =
      planned ? std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp).count() : 0.0;
  const bool rl = g->plan.relabel;
  const cyc::DevCsr& snap = rl ? g->plan.snap : g->snap;
  const cyc::DevCsr& gath = rl ? g->plan.gath : g->gath;
  const uint32_t* orig = rl ? g->plan.orig.as<uint32_t>() : nullptr;
  const uint32_t* perm = rl ? g->plan.perm.as<uint32_t>() : nullptr;
  g->ws.ensure(n, gath.m, snap.o(), s);
  const size_t nw = acc_words64(n);
  DevBuf fin;  // accepting words in vertex-id order, permuted into storage order below
  if (rl) fin.alloc((nw + 1) * 8, s);
  uint64_t* F = rl ? fin.as<uint64_t>() : g->ws.F.as<uint64_t>();
  if (acc_words) {
    CYC_CUDA(cudaMemcpyAsync(F, acc_words, nw * 8, cudaMemcpyDefault, s));
  } else {
    CYC_CUDA(cudaMemcpyAsync(F, g->acc.p, nw * 8, cudaMemcpyDeviceToDevice, s));
  }
  if (nw) {
    k_trim_tail<<<1, 1, 0, s>>>(F, n);
    CYC_LAUNCHED();
  }
  if (rl) cyc::permute_bits(reinterpret_cast<const uint32_t*>(F), orig, n, g->ws.F.as<uint32_t>(), s);
  cyc::RunOut out;
  out.plan_ms = plan_ms;
  out.layout = rl ? CYC_LAYOUT_DEGREE : CYC_LAYOUT_IDENTITY;
  cyc::launch_map_run(snap, gath, orig, perm, rl ? g->plan.sdesc.as<uint4>() : nullptr,
                      rl ? g->plan.sell.as<uint32_t>() : nullptr, rl ? g->plan.hcol.as<uint32_t>() : nullptr,
                      rl ? g->plan.hrow.as<uint32_t>() : nullptr, rl ? g->plan.n_hchunks : 0u, g->ws, o.early_exit != 0, o.mode, o.max_iterations,
                      o.max_steps, o.push_alpha, cap, o.trace_cap, s, ctx->e0, ctx->e1, out);
  return out;
}

}  // namespace

extern "C" {

const char* cyc_last_error(void) { return g_err.c_str(); }
uint64_t cyc_launch_count(void) { return cyc::g_launches.load(); }

cyc_status cyc_ctx_create(int device, cyc_ctx** out) {
  return guard([&] {
    require(out != nullptr, CYC_E_CONTRACT, "null out");
    int count = 0;
    CYC_CUDA(cudaGetDeviceCount(&count));
    require(device >= 0 && device < count, CYC_E_CONTRACT, "no such CUDA device");
    CYC_CUDA(cudaSetDevice(device));
    int major = 0, minor = 0;
    CYC_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    CYC_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    require(major == 10 && minor == 0, CYC_E_INVALID,
            "this library is built for sm_100a (B200) only");
    auto* c = new cyc_ctx;
    c->device = device;
    CYC_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
    c->s = c->own;
    CYC_CUDA(cudaEventCreate(&c->e0));
    CYC_CUDA(cudaEventCreate(&c->e1));
    CYC_CUDA(cudaEventCreate(&c->e2));
    CYC_CUDA(cudaEventCreate(&c->e3));
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    *out = c;
  });
}

void cyc_ctx_destroy(cyc_ctx* ctx) {
  if (ctx) ctx_release(ctx);
}

// First touch of device memory costs ~150 GB/s on a B200
// (scripts/micro/map_rate.cu): config 3's first call maps ~60 GB of build
// temporaries and outputs (~0.4 s of a ~0.7 s first call). cyc_ctx_reserve
// allocates them ahead, sized for a log of m_log edges over n vertices: the
// two build arenas at the sizes build_csr asks for, and blocks of the staged
// log / CSR columns / offsets parked in the big-block cache, where the
// build's own requests pick them up.
cyc_status cyc_ctx_reserve(cyc_ctx* ctx, uint64_t m_log, uint32_t n, int background) {
  return guard([&] {
    require(ctx, CYC_E_CONTRACT, "null ctx");
    join_reserve(ctx);
    if (!m_log) return;
    auto work = [ctx, m_log, n] {
      try {
        CYC_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->own;
        const size_t nn = (size_t)n + 1;
        for (cyc::BuildArena* a : {&ctx->arena, &ctx->arena2}) {
          a->get<uint8_t>(a->tmp, m_log * 8, s);
          a->get<uint8_t>(a->tmp2, m_log * 8, s);
          a->get<uint8_t>(a->raw, m_log * 4, s);
          a->get<uint8_t>(a->roff, nn * 4, s);
          a->get<uint8_t>(a->ucnt, nn * 4, s);
          a->get<uint8_t>(a->lists, nn * 12, s);
        }
        // staged log, snapshot / gather columns, the plan's two relabelled
        // column arrays and heavy slab (built on a graph's second loop), offsets
        const size_t sizes[] = {m_log * 8, m_log * 4, m_log * 4, m_log * 4, m_log * 4, m_log * 4,
                                nn * 4,    nn * 4,    nn * 4,    nn * 4,    nn * 4,    nn * 4};
        std::vector<std::pair<void*, size_t>> got;
        for (size_t b : sizes) {
          if (b < cyc::kBigBlock) continue;
          size_t cap = 0;
          void* p = cyc::big_alloc(b, s, &cap);
          got.emplace_back(p, cap);
        }
        for (auto& pc : got) cyc::big_free(pc.first, pc.second, s);
        CYC_CUDA(cudaStreamSynchronize(s));
      } catch (...) {
        cudaGetLastError();  // out of memory: the builds allocate as they go
      }
    };
    if (background) ctx->reserver = std::thread(work);
    else work();
  });
}

cyc_status cyc_ctx_synchronize(cyc_ctx* ctx) {
  return guard([&] { CYC_CUDA(cudaStreamSynchronize(ctx->s)); });
}

void* cyc_ctx_stream(cyc_ctx* ctx) { return ctx ? (void*)ctx->s : nullptr; }

cyc_status cyc_ctx_set_stream(cyc_ctx* ctx, void* stream, int external) {
  return guard([&] {
    require(ctx, CYC_E_CONTRACT, "null ctx");
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CYC_CUDA(cudaStreamIsCapturing(ctx->s, &cs));
    if (cs == cudaStreamCaptureStatusNone) CYC_CUDA(cudaStreamSynchronize(ctx->s));
    ctx->s = external ? static_cast<cudaStream_t>(stream) : ctx->own;
  });
}

cyc_status cyc_graph_build(cyc_ctx* ctx, const uint32_t* edges, uint64_t m_log, uint32_t n,
                           const uint64_t* acc_words, int orientation, cyc_graph** out) {
  CallTrace trace_("cyc_graph_build");
  return guard([&] {
    require(ctx && out, CYC_E_CONTRACT, "null argument");
    CYC_CUDA(cudaSetDevice(ctx->device));
    auto* g = new cyc_graph;
    try {
      build_graph(ctx, edges, m_log, n, acc_words, orientation, g);
    } catch (...) {
      delete g;
      throw;
    }
    ctx->refs.fetch_add(1);
    *out = g;
  });
}

// CSR (row, col) entries back to the logged (src, dst) pairs of the prefix.
__global__ void k_csr_to_log(uint32_t n, const uint64_t* __restrict__ off, const uint32_t* __restrict__ col,
                             int transposed, uint2* __restrict__ edges) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride)
    for (uint64_t i = off[v]; i < off[v + 1]; ++i)
      edges[i] = transposed ? make_uint2(col[i], v) : make_uint2(v, col[i]);
}

cyc_status cyc_graph_from_csr(cyc_ctx* ctx, const uint64_t* row_offsets, const uint32_t* col_indices,
                              uint32_t n, uint64_t m, const uint64_t* acc_words, int orientation,
                              cyc_graph** out) {
  return guard([&] {
    require(ctx && out && row_offsets, CYC_E_CONTRACT, "null argument");
    require(m < 0xFFFFFFFFull, CYC_E_RESOURCE, "snapshot edges must be < 2^32");
    CYC_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->s;
    DevBuf toff, tcol, edges((m ? m : 1) * 8, s);
    const uint64_t* doff = stage_in(row_offsets, (size_t)n + 1, toff, s);
    const uint32_t* dcol = stage_in(col_indices, (size_t)m, tcol, s);
    if (n && m) {
      k_csr_to_log<<<cyc::grid_for(n, 256, 8), 256, 0, s>>>(n, doff, dcol, orientation == CYC_TRANSPOSED,
                                                           edges.as<uint2>());
      CYC_LAUNCHED();
    }
    auto* g = new cyc_graph;
    try {
      build_graph(ctx, edges.as<uint32_t>(), m, n, acc_words, orientation, g);
    } catch (...) {
      delete g;
      throw;
    }
    ctx->refs.fetch_add(1);
    *out = g;
  });
}

cyc_status cyc_graph_extend(cyc_ctx* ctx, const cyc_graph* prev, const uint32_t* new_edges, uint64_t m_new,
                            uint32_t n, const uint64_t* acc_words, cyc_graph** out) {
  return guard([&] {
    require(ctx && prev && out, CYC_E_CONTRACT, "extend_snapshot: null argument");
    require(!prev->restricted, CYC_E_CONTRACT, "extend_snapshot: restricted snapshots cannot grow");
    require(n >= prev->n(), CYC_E_CONTRACT, "extend_snapshot: vertex prefix shrinks");
    CYC_CUDA(cudaSetDevice(ctx->device));
    auto* g = new cyc_graph;
    try {
      cyc_graph delta;
      build_graph(ctx, new_edges, m_new, n, acc_words, prev->orientation, &delta);
      cudaStream_t s = ctx->s;
      g->ctx = ctx;
      g->orientation = prev->orientation;
      g->m_log = prev->m_log + m_new;
      require(g->m_log < 0xFFFFFFFFull, CYC_E_RESOURCE, "edge log prefix must be < 2^32");
      cyc::merge_csr(prev->snap, delta.snap, n, s, g->snap);
      cyc::merge_csr(prev->gath, delta.gath, n, s, g->gath);
      require(g->snap.m == g->gath.m, CYC_E_CUDA, "internal: snapshot/gather edge counts differ");
      cyc::build_heavy(g->gath, cyc::kHeavyDeg, cyc::kHeavyChunk, s, cyc::pull_col_blocks(g->gath.n));
      cyc::build_heavy(g->snap, cyc::kHeavyDeg, cyc::kHeavyChunk, s);
      cyc::build_ell(g->gath, s);
      if (acc_words) {
        load_acc(acc_words, n, g->acc, s);
      } else {  // previous accepting bits, new vertices not accepting
        const size_t nw = acc_words64(n), pw = acc_words64(prev->n());
        g->acc.alloc((nw + 1) * 8, s);
        CYC_CUDA(cudaMemsetAsync(g->acc.p, 0, (nw + 1) * 8, s));
        if (pw) CYC_CUDA(cudaMemcpyAsync(g->acc.p, prev->acc.p, pw * 8, cudaMemcpyDeviceToDevice, s));
      }
      CYC_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      delete g;
      throw;
    }
    ctx->refs.fetch_add(1);
    *out = g;
  });
}

cyc_status cyc_graph_log_prefix(const cyc_graph* g, uint64_t* m_log) {
  return guard([&] {
    require(g && m_log, CYC_E_CONTRACT, "null argument");
    *m_log = g->m_log;
  });
}

cyc_status cyc_graph_restrict(cyc_ctx* ctx, const cyc_graph* in, cyc_graph** out) {
  CallTrace trace_("cyc_graph_restrict");
  return guard([&] {
    require(ctx && in && out, CYC_E_CONTRACT, "null argument");
    CYC_CUDA(cudaSetDevice(ctx->device));
    auto* g = new cyc_graph;
    try {
      g->ctx = ctx;
      g->orientation = in->orientation;
      g->restricted = 1;
      cyc::restrict_graph(in->snap, in->gath, in->acc.as<uint64_t>(), ctx->s, g->snap, g->gath,
                          g->acc, g->kept);
      cyc::build_heavy(g->gath, cyc::kHeavyDeg, cyc::kHeavyChunk, ctx->s, cyc::pull_col_blocks(g->gath.n));
      cyc::build_heavy(g->snap, cyc::kHeavyDeg, cyc::kHeavyChunk, ctx->s);
      cyc::build_ell(g->gath, ctx->s);
    } catch (...) {
      delete g;
      throw;
    }
    ctx->refs.fetch_add(1);
    *out = g;
  });
}

void cyc_graph_destroy(cyc_graph* g) {
  if (!g) return;
  cyc_ctx* ctx = g->ctx;
  cudaSetDevice(ctx->device);
  delete g;
  ctx_release(ctx);
}

cyc_status cyc_graph_info(const cyc_graph* g, uint32_t* n, uint64_t* m, int* orientation,
                          int* restricted) {
  return guard([&] {
    require(g, CYC_E_CONTRACT, "null graph");
    if (n) *n = g->n();
    if (m) *m = g->snap.m;
    if (orientation) *orientation = g->orientation;
    if (restricted) *restricted = g->restricted;
  });
}

cyc_status cyc_graph_export(const cyc_graph* g, uint64_t* row_offsets, uint32_t* col_indices,
                            uint64_t* acc_words, uint32_t* kept) {
  return guard([&] {
    require(g, CYC_E_CONTRACT, "null graph");
    cudaStream_t s = g->ctx->s;
    export_offsets(g->snap, row_offsets, s);
    copy_out(col_indices, g->snap.c(), g->snap.m, s);
    copy_out(acc_words, g->acc.as<uint64_t>(), acc_words64(g->n()), s);
    if (g->restricted) copy_out(kept, g->kept.as<uint32_t>(), g->n(), s);
    CYC_CUDA(cudaStreamSynchronize(s));
  });
}

cyc_status cyc_graph_export_gather(const cyc_graph* g, uint64_t* row_offsets,
                                   uint32_t* col_indices) {
  return guard([&] {
    require(g, CYC_E_CONTRACT, "null graph");
    cudaStream_t s = g->ctx->s;
    export_offsets(g->gath, row_offsets, s);
    copy_out(col_indices, g->gath.c(), g->gath.m, s);
    CYC_CUDA(cudaStreamSynchronize(s));
  });
}

cyc_status cyc_map_step(cyc_ctx* ctx, const cyc_graph* g, const uint64_t* acc_words,
                        const uint32_t* x, uint32_t* out, int32_t* changed, uint32_t* witness) {
  return guard([&] {
    require(ctx && g && x && out, CYC_E_CONTRACT, "propagate_step: null argument");
    cudaStream_t s = ctx->s;
    const uint32_t n = g->n();
    DevBuf tx, tacc, accb, dout, flags(16, s);
    const uint32_t* dx = stage_in(x, n, tx, s);
    const uint64_t* dacc = g->acc.as<uint64_t>();
    if (acc_words) {
      load_acc(acc_words, n, accb, s);
      dacc = accb.as<uint64_t>();
    }
    uint32_t* dst = out;
    const bool dev_out = is_device_ptr(out);
    if (!dev_out) {
      dout.alloc(((size_t)n + 1) * 4, s);
      dst = dout.as<uint32_t>();
    }
    cyc::launch_step_pull(g->gath, dx, reinterpret_cast<const uint32_t*>(dacc), dst,
                          flags.as<uint32_t>(), s);
    if (!dev_out) copy_out(out, dst, n, s);
    uint32_t hf[2];
    CYC_CUDA(cudaMemcpyAsync(hf, flags.p, 8, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
    if (changed) *changed = (int32_t)hf[0];
    if (witness) *witness = hf[1];
  });
}

cyc_status cyc_fixpoint(cyc_ctx* ctx, const cyc_graph* g, const uint64_t* acc_words,
                        const cyc_map_options* opt, uint32_t* values, uint64_t* steps,
                        uint32_t* witness) {
  return guard([&] {
    require(ctx && g, CYC_E_CONTRACT, "fixpoint: null argument");
    cyc_map_options o = opt ? *opt : default_opts();
    o.max_iterations = 1;
    auto* gg = const_cast<cyc_graph*>(g);
    cyc::RunOut r = run_loop(ctx, gg, acc_words, o, 0);
    const uint32_t n = g->n();
    // fixpoint from an empty accepting set still performs one step
    // (map_engine.cpp:98-112); the device loop skips it (run_map semantics),
    // so account for it here: x stays all-NIL and nothing changes.
    uint64_t st = r.res[cyc::kResIterations] ? r.res[cyc::kResStepsLast] : 1;
    if (steps) *steps = st;
    if (witness) *witness = r.res[cyc::kResCycle] ? (uint32_t)r.res[cyc::kResWitness] : cyc::kNone;
    if (values && n) {
      if (r.res[cyc::kResIterations] == 0) {
        CYC_CUDA(cudaMemsetAsync(gg->ws.P[0].p, 0, (size_t)n * 4, ctx->s));
        r.res[cyc::kResCur] = 0;
      }
      if (is_device_ptr(values)) {
        cyc::strip_codes(gg->ws, (int)r.res[cyc::kResCur], n, values, ctx->s);
      } else {
        DevBuf tmp((size_t)n * 4, ctx->s);
        cyc::strip_codes(gg->ws, (int)r.res[cyc::kResCur], n, tmp.as<uint32_t>(), ctx->s);
        copy_out(values, tmp.as<uint32_t>(), n, ctx->s);
      }
      CYC_CUDA(cudaStreamSynchronize(ctx->s));
    }
  });
}

cyc_status cyc_demote(cyc_ctx* ctx, const uint32_t* values, uint32_t n,
                      const uint64_t* acc_words, uint64_t* remaining, uint32_t* demoted,
                      uint64_t* n_demoted) {
  return guard([&] {
    require(ctx && (values || n == 0) && acc_words, CYC_E_CONTRACT, "demote: null argument");
    cudaStream_t s = ctx->s;
    DevBuf tx, accb, rem((acc_words64(n) + 1) * 8, s), dem(((size_t)n + 1) * 4, s);
    const uint32_t* dx = stage_in(values, n, tx, s);
    load_acc(acc_words, n, accb, s);
    uint64_t nd = cyc::run_demote(dx, n, reinterpret_cast<const uint32_t*>(accb.p),
                                  rem.as<uint32_t>(), demoted ? dem.as<uint32_t>() : nullptr, s);
    copy_out(remaining, rem.as<uint64_t>(), acc_words64(n), s);
    if (demoted) copy_out(demoted, dem.as<uint32_t>(), nd, s);
    CYC_CUDA(cudaStreamSynchronize(s));
    if (n_demoted) *n_demoted = nd;
  });
}

cyc_status cyc_map_run(cyc_ctx* ctx, const cyc_graph* g, const uint64_t* acc_words,
                       const cyc_map_options* opt, cyc_map_stats* stats, uint32_t* final_values,
                       uint64_t* iter_hash, uint64_t* iter_steps, uint64_t cap) {
  CallTrace trace_("cyc_map_run");
  return guard([&] {
    require(ctx && g, CYC_E_CONTRACT, "run_map: null argument");
    cyc_map_options o = opt ? *opt : default_opts();
    auto* gg = const_cast<cyc_graph*>(g);
    const uint64_t hcap = (iter_hash || iter_steps) ? cap : 0;
    cyc::RunOut r = run_loop(ctx, gg, acc_words, o, hcap);
    fill_stats(r, stats);  // witness in this snapshot's ids, as run_map returns it
    const uint32_t n = g->n();
    if (final_values && n) {
      if (r.res[cyc::kResIterations] == 0) {
        CYC_CUDA(cudaMemsetAsync(gg->ws.P[0].p, 0, (size_t)n * 4, ctx->s));
        r.res[cyc::kResCur] = 0;
      }
      if (is_device_ptr(final_values)) {
        cyc::strip_codes(gg->ws, (int)r.res[cyc::kResCur], n, final_values, ctx->s);
      } else {
        DevBuf tmp((size_t)n * 4, ctx->s);
        cyc::strip_codes(gg->ws, (int)r.res[cyc::kResCur], n, tmp.as<uint32_t>(), ctx->s);
        copy_out(final_values, tmp.as<uint32_t>(), n, ctx->s);
      }
    }
    const uint64_t rec = hcap < r.res[cyc::kResIterations] ? hcap : r.res[cyc::kResIterations];
    if (iter_hash && rec) copy_out(iter_hash, (uint64_t*)gg->ws.hist.p, rec, ctx->s);
    if (iter_steps && rec) copy_out(iter_steps, (uint64_t*)gg->ws.hist.p + hcap, rec, ctx->s);
    CYC_CUDA(cudaStreamSynchronize(ctx->s));
  });
}

cyc_status cyc_scc_verdict(cyc_ctx* ctx, const cyc_graph* g, int32_t* cycle, uint32_t* witness,
                           uint32_t* cyclic_accepting, uint64_t* count) {
  return guard([&] {
    require(ctx && g, CYC_E_CONTRACT, "scc_verdict: null argument");
    DevBuf list;
    const uint32_t k = cyc::scc_cyclic_accepting(g->snap, g->gath, g->acc.as<uint64_t>(), ctx->s, list);
    uint32_t first = cyc::kNone;
    if (k) CYC_CUDA(cudaMemcpyAsync(&first, list.p, 4, cudaMemcpyDeviceToHost, ctx->s));
    if (cyclic_accepting && k) copy_out(cyclic_accepting, list.as<uint32_t>(), k, ctx->s);
    CYC_CUDA(cudaStreamSynchronize(ctx->s));
    if (cycle) *cycle = k > 0;
    if (witness) *witness = first;
    if (count) *count = k;
  });
}

cyc_status cyc_owcty(cyc_ctx* ctx, const cyc_graph* g, const uint64_t* acc_words, int32_t* cycle,
                     uint32_t* witness, cyc_owcty_stats* stats) {
  CallTrace trace_("cyc_owcty");
  return guard([&] {
    require(ctx && g, CYC_E_CONTRACT, "run_owcty: null argument");
    CYC_CUDA(cudaSetDevice(ctx->device));
    DevBuf accb;
    const uint64_t* dacc = g->acc.as<uint64_t>();
    if (acc_words) {
      load_acc(acc_words, g->n(), accb, ctx->s);
      dacc = accb.as<uint64_t>();
    }
    const cyc::OwctyResult r = cyc::run_owcty_device(g->snap, g->gath, dacc, ctx->s);
    if (cycle) *cycle = r.cycle;
    if (witness) *witness = r.witness;
    if (stats) {
      stats->outer_iterations = r.outer_iterations;
      stats->final_size = r.final_size;
      stats->reach_ms = r.reach_ms;
      stats->elim_ms = r.elim_ms;
    }
  });
}

cyc_status cyc_last_parse_error(int* code, int* line, int* col) {
  if (code) *code = g_parse[0];
  if (line) *line = g_parse[1];
  if (col) *col = g_parse[2];
  return CYC_OK;
}

cyc_status cyc_explicit_parse(cyc_ctx* ctx, const char* text, uint64_t len, cyc_explicit** out) {
  return guard([&] {
    require(ctx && out && (text || !len), CYC_E_CONTRACT, "parse_explicit_graph: null argument");
    CYC_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->s;
    DevBuf staged;
    const uint8_t* d = reinterpret_cast<const uint8_t*>(text);
    if (len && (!is_device_ptr(text) || (reinterpret_cast<uintptr_t>(text) & 15u))) {
      staged.alloc(len + 16, s);
      CYC_CUDA(cudaMemcpyAsync(staged.p, text, len, cudaMemcpyDefault, s));
      d = staged.as<uint8_t>();
    }
    auto* e = new cyc_explicit;
    try {
      e->ctx = ctx;
      cyc::parse_explicit_device(d, len, s, e->g);
      CYC_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      delete e;
      throw;
    }
    ctx->refs.fetch_add(1);
    *out = e;
  });
}

// Binary layout: "CYCGRAPH", u32 version (1), u32 n, u64 m, u64 accepting
// words[ceil(n/64)], u32 edges[2m] (src, dst in log order).
cyc_status cyc_explicit_load_binary(cyc_ctx* ctx, const void* data, uint64_t len, cyc_explicit** out) {
  return guard([&] {
    require(ctx && out && data, CYC_E_CONTRACT, "load_binary_graph: null argument");
    CYC_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->s;
    struct Hdr {
      char magic[8];
      uint32_t version, n;
      uint64_t m;
    } h;
    require(len >= sizeof h, CYC_E_CONTRACT, "load_binary_graph: truncated header");
    CYC_CUDA(cudaMemcpy(&h, data, sizeof h, cudaMemcpyDefault));
    require(std::memcmp(h.magic, "CYCGRAPH", 8) == 0 && h.version == 1, CYC_E_CONTRACT,
            "load_binary_graph: not a CYCGRAPH v1 file");
    const uint64_t nw = ((uint64_t)h.n + 63) / 64;
    require(len == sizeof h + nw * 8 + h.m * 8, CYC_E_CONTRACT, "load_binary_graph: size does not match header");
    auto* e = new cyc_explicit;
    try {
      e->ctx = ctx;
      e->g.n = h.n;
      e->g.m = h.m;
      e->g.has_words = true;
      e->g.acc_words.alloc(nw * 8 + 8, s);
      e->g.edges.alloc(h.m * 8 + 8, s);
      const char* base = static_cast<const char*>(data) + sizeof h;
      if (nw) CYC_CUDA(cudaMemcpyAsync(e->g.acc_words.p, base, nw * 8, cudaMemcpyDefault, s));
      if (h.m) CYC_CUDA(cudaMemcpyAsync(e->g.edges.p, base + nw * 8, h.m * 8, cudaMemcpyDefault, s));
      cyc::explicit_acc_ids_from_words(e->g, s);
      CYC_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
      delete e;
      throw;
    }
    ctx->refs.fetch_add(1);
    *out = e;
  });
}

cyc_status cyc_explicit_info(const cyc_explicit* g, uint32_t* n, uint64_t* n_accepting, uint64_t* m) {
  return guard([&] {
    require(g, CYC_E_CONTRACT, "null graph");
    if (n) *n = g->g.n;
    if (n_accepting) *n_accepting = g->g.n_acc;
    if (m) *m = g->g.m;
  });
}

cyc_status cyc_explicit_export(const cyc_explicit* g, uint32_t* accepting, uint32_t* edges) {
  return guard([&] {
    require(g, CYC_E_CONTRACT, "null graph");
    cudaStream_t s = g->ctx->s;
    if (accepting && g->g.n_acc) copy_out(accepting, g->g.acc_ids.as<uint32_t>(), g->g.n_acc, s);
    if (edges && g->g.m) copy_out(edges, g->g.edges.as<uint32_t>(), g->g.m * 2, s);
    CYC_CUDA(cudaStreamSynchronize(s));
  });
}

cyc_status cyc_explicit_snapshot(cyc_ctx* ctx, const cyc_explicit* eg, int orientation, cyc_graph** out) {
  return guard([&] {
    require(ctx && eg && out, CYC_E_CONTRACT, "null argument");
    CYC_CUDA(cudaSetDevice(ctx->device));
    DevBuf words;
    cyc::explicit_acc_words(eg->g, ctx->s, words);
    auto* g = new cyc_graph;
    try {
      build_graph(ctx, eg->g.edges.as<uint32_t>(), eg->g.m, eg->g.n, words.as<uint64_t>(), orientation, g);
      CYC_CUDA(cudaStreamSynchronize(ctx->s));
    } catch (...) {
      delete g;
      throw;
    }
    ctx->refs.fetch_add(1);
    *out = g;
  });
}

void cyc_explicit_destroy(cyc_explicit* g) {
  if (!g) return;
  cyc_ctx* c = g->ctx;
  if (c) cudaSetDevice(c->device);
  delete g;
  if (c) ctx_release(c);
}

cyc_status cyc_check(cyc_ctx* ctx, const uint32_t* edges, uint64_t m_log, uint32_t n,
                     const uint64_t* acc_words, int orientation, int scc_restrict,
                     const cyc_map_options* opt, cyc_map_stats* stats, double* ms_out) {
  return guard([&] {
    require(ctx, CYC_E_CONTRACT, "null ctx");
    CYC_CUDA(cudaSetDevice(ctx->device));
    using clk = std::chrono::steady_clock;
    auto t0 = clk::now();
    cyc_graph base;
    build_graph(ctx, edges, m_log, n, acc_words, orientation, &base);
    auto t1 = clk::now();
    cyc_graph restricted;
    cyc_graph* run_on = &base;
    if (scc_restrict) {
      restricted.ctx = ctx;
      restricted.orientation = orientation;
      restricted.restricted = 1;
      cyc::restrict_graph(base.snap, base.gath, base.acc.as<uint64_t>(), ctx->s, restricted.snap,
                          restricted.gath, restricted.acc, restricted.kept);
      cyc::build_heavy(restricted.gath, cyc::kHeavyDeg, cyc::kHeavyChunk, ctx->s, cyc::pull_col_blocks(restricted.gath.n));
      cyc::build_heavy(restricted.snap, cyc::kHeavyDeg, cyc::kHeavyChunk, ctx->s);
      cyc::build_ell(restricted.gath, ctx->s);
      run_on = &restricted;
    }
    auto t2 = clk::now();
    cyc_map_options o = opt ? *opt : default_opts();
    cyc::RunOut r = run_loop(ctx, run_on, nullptr, o, 0);
    fill_stats(r, stats);
    if (stats && run_on->restricted && stats->cycle_found) {
      uint32_t orig = 0;
      CYC_CUDA(cudaMemcpyAsync(&orig, run_on->kept.as<uint32_t>() + stats->witness, 4,
                               cudaMemcpyDeviceToHost, ctx->s));
      CYC_CUDA(cudaStreamSynchronize(ctx->s));
      stats->witness = orig;
    }
    auto t3 = clk::now();
    if (ms_out) {
      auto ms = [](clk::time_point a, clk::time_point b) {
        return std::chrono::duration<double, std::milli>(b - a).count();
      };
      ms_out[0] = ms(t0, t1);
      ms_out[1] = ms(t1, t2);
      ms_out[2] = ms(t2, t3);
      ms_out[3] = ms(t0, t3);
    }
  });
}

cyc_status cyc_shard_build(cyc_ctx* ctx, const uint32_t* edges, uint64_t m_log, uint32_t n,
                           const uint64_t* acc_words, int orientation, int layout, int world, int rank,
                           cyc_shard** out) {
  CallTrace trace_("cyc_shard_build");
  return guard([&] {
    require(ctx && out, CYC_E_CONTRACT, "null argument");
    require(orientation == CYC_FORWARD || orientation == CYC_TRANSPOSED, CYC_E_CONTRACT,
            "build_snapshot: bad orientation");
    require(layout >= CYC_LAYOUT_AUTO && layout <= CYC_LAYOUT_DEGREE, CYC_E_CONTRACT, "bad layout");
    require(n < 0x80000000u, CYC_E_RESOURCE, "vertex count must be < 2^31");
    require(m_log < 0xFFFFFFFFull, CYC_E_RESOURCE, "edge log prefix must be < 2^32");
    require(m_log == 0 || edges, CYC_E_CONTRACT, "build_snapshot: null edge array");
    CYC_CUDA(cudaSetDevice(ctx->device));
    join_reserve(ctx);
    DevBuf tmp, tacc;
    const uint32_t* de = stage_in(edges, (size_t)m_log * 2, tmp, ctx->s);
    const uint64_t* da = stage_in(acc_words, acc_words64(n), tacc, ctx->s);
    auto* sh = new cyc_shard;
    sh->ctx = ctx;
    try {
      cyc::build_shard(de, m_log, n, da, orientation, world, rank, layout, sh->g, ctx->arena, ctx->s);
    } catch (...) {
      delete sh;
      throw;
    }
    ctx->refs.fetch_add(1);
    *out = sh;
  });
}

cyc_status cyc_shard_info(const cyc_shard* sh, uint32_t* row_lo, uint32_t* row_hi, uint64_t* local_edges,
                          uint64_t* device_bytes) {
  return guard([&] {
    require(sh, CYC_E_CONTRACT, "null shard");
    if (row_lo) *row_lo = sh->g.row_lo;
    if (row_hi) *row_hi = sh->g.row_hi;
    if (local_edges) *local_edges = sh->g.m_local;
    if (device_bytes) *device_bytes = sh->g.device_bytes();
  });
}

cyc_status cyc_shard_handle(const cyc_shard* sh, void* out) {
  static_assert(sizeof(cyc::ShardHandles) <= CYC_SHARD_HANDLE_BYTES, "handle blob too small");
  return guard([&] {
    require(sh && out, CYC_E_CONTRACT, "null argument");
    CYC_CUDA(cudaSetDevice(sh->g.device));
    cyc::ShardHandles h;
    std::memset(&h, 0, sizeof h);
    cyc::shard_export(sh->g, h);
    std::memset(out, 0, CYC_SHARD_HANDLE_BYTES);
    std::memcpy(out, &h, sizeof h);
  });
}

cyc_status cyc_shard_connect(cyc_shard* sh, const void* handles) {
  return guard([&] {
    require(sh && handles, CYC_E_CONTRACT, "null argument");
    CYC_CUDA(cudaSetDevice(sh->g.device));
    std::vector<cyc::ShardHandles> all(sh->g.world);
    for (int p = 0; p < sh->g.world; ++p)
      std::memcpy(&all[p], static_cast<const char*>(handles) + (size_t)p * CYC_SHARD_HANDLE_BYTES, sizeof all[p]);
    cyc::shard_connect_ipc(sh->g, all.data(), sh->g.world);
  });
}

cyc_status cyc_shard_connect_local(cyc_shard* const* shards, int world) {
  return guard([&] {
    require(shards && world >= 1 && world <= cyc::kMaxWorld, CYC_E_CONTRACT, "bad shards");
    std::vector<cyc::ShardGraph*> gs(world);
    for (int i = 0; i < world; ++i) {
      require(shards[i] != nullptr, CYC_E_CONTRACT, "null shard");
      gs[i] = &shards[i]->g;
    }
    cyc::shard_connect_local(gs.data(), world);
  });
}

cyc_status cyc_shard_run_map(cyc_shard* const* shards, int count, const uint64_t* acc_words,
                             const cyc_map_options* opt, cyc_map_stats* stats, uint32_t* final_values,
                             uint64_t* iter_hash, uint64_t* iter_steps, uint64_t cap) {
  CallTrace trace_("cyc_shard_run_map");
  return guard([&] {
    require(shards && count >= 1 && count <= cyc::kMaxWorld, CYC_E_CONTRACT, "run_map: bad shards");
    cyc_map_options o = opt ? *opt : default_opts();
    require(o.mode >= CYC_MODE_AUTO && o.mode <= CYC_MODE_PUSH, CYC_E_CONTRACT, "bad mode");
    std::vector<cyc::ShardGraph*> gs(count);
    std::vector<cudaStream_t> ss(count);
    for (int i = 0; i < count; ++i) {
      require(shards[i] != nullptr, CYC_E_CONTRACT, "null shard");
      gs[i] = &shards[i]->g;
      ss[i] = shards[i]->ctx->s;
    }
    require(count == 1 || count == gs[0]->world, CYC_E_CONTRACT, "run_map: pass one rank or all of them");
    const uint64_t hcap = (iter_hash || iter_steps) ? cap : 0;
    std::vector<cyc::RunOut> outs(count);
    cyc::shard_run(gs.data(), count, acc_words, o.early_exit != 0, o.mode, o.max_iterations, o.max_steps,
                   o.push_alpha, hcap, ss.data(), nullptr, nullptr, outs.data());
    const cyc::RunOut& r = outs[0];
    fill_stats(r, stats);
    if (stats) {
      stats->layout = gs[0]->relabel ? CYC_LAYOUT_DEGREE : CYC_LAYOUT_IDENTITY;
      stats->world = gs[0]->world;
      stats->exchanged_rows = r.res[cyc::kResRaised];
    }
    cyc_ctx* ctx = shards[0]->ctx;
    CYC_CUDA(cudaSetDevice(ctx->device));
    const uint32_t n = gs[0]->n;
    if (final_values && n) {
      int cur = (int)r.res[cyc::kResCur];
      if (r.res[cyc::kResIterations] == 0) {
        CYC_CUDA(cudaMemsetAsync(gs[0]->xP[0], 0, (size_t)n * 4, ctx->s));
        cur = 0;
      }
      DevBuf tmp((size_t)n * 4, ctx->s);
      cyc::shard_values(*gs[0], cur, tmp.as<uint32_t>(), ctx->s);
      copy_out(final_values, tmp.as<uint32_t>(), n, ctx->s);
    }
    const uint64_t rec = hcap < r.res[cyc::kResIterations] ? hcap : r.res[cyc::kResIterations];
    if (iter_hash && rec) copy_out(iter_hash, (uint64_t*)gs[0]->ws.hist.p, rec, ctx->s);
    if (iter_steps && rec) copy_out(iter_steps, (uint64_t*)gs[0]->ws.hist.p + hcap, rec, ctx->s);
    CYC_CUDA(cudaStreamSynchronize(ctx->s));
  });
}

void cyc_shard_destroy(cyc_shard* sh) {
  if (!sh) return;
  cyc_ctx* ctx = sh->ctx;
  cudaSetDevice(ctx->device);
  delete sh;
  ctx_release(ctx);
}

cyc_status cyc_gen_preset(int index, void* gen_params) {
  return guard([&] {
    require(gen_params, CYC_E_CONTRACT, "null params");
    require(cyc_gen_config(static_cast<cyc_gen_params*>(gen_params), index) == 0, CYC_E_CONTRACT,
            "unknown generator config");
  });
}

cyc_status cyc_gen_prepare(void* gen_params) {
  return guard([&] {
    require(gen_params, CYC_E_CONTRACT, "null params");
    require(cyc_gen_init(static_cast<cyc_gen_params*>(gen_params)) == 0, CYC_E_CONTRACT,
            "bad generator parameters");
  });
}

cyc_status cyc_gen_fill(cyc_ctx* ctx, const void* gen_params, uint32_t* edges,
                        uint64_t* acc_words) {
  return guard([&] {
    require(ctx && gen_params, CYC_E_CONTRACT, "null argument");
    const cyc_gen_params p = *static_cast<const cyc_gen_params*>(gen_params);
    cudaStream_t s = ctx->s;
    const uint64_t nw = acc_words64(p.n);
    DevBuf te, ta;
    uint32_t* de = edges;
    uint64_t* da = acc_words;
    const bool dev_e = is_device_ptr(edges), dev_a = is_device_ptr(acc_words);
    if (edges && !dev_e) {
      te.alloc(p.m * 8 + 8, s);
      de = te.as<uint32_t>();
    }
    if (acc_words && !dev_a) {
      ta.alloc(nw * 8 + 8, s);
      da = ta.as<uint64_t>();
    }
    if (p.kind == CYC_GEN_PRODUCT) {
      cyc::gen_product_device(p, edges ? de : nullptr, acc_words ? da : nullptr, s);
    } else {
      cyc_gen_params q = p;
      if (!edges) q.m = 0;
      k_gen<<<cyc::grid_for(p.m > nw ? p.m : nw, 256, 16), 256, 0, s>>>(q, de, da, nw);
      CYC_LAUNCHED();
    }
    if (edges && !dev_e) copy_out(edges, de, p.m * 2, s);
    if (acc_words && !dev_a) copy_out(acc_words, da, nw, s);
    CYC_CUDA(cudaStreamSynchronize(s));
  });
}

cyc_status cyc_host_alloc(size_t bytes, void** out) {
  return guard([&] {
    require(out, CYC_E_CONTRACT, "null out");
    CYC_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocDefault));
  });
}

void cyc_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

cyc_status cyc_device_alloc(cyc_ctx* ctx, size_t bytes, void** out) {
  return guard([&] {
    require(ctx && out, CYC_E_CONTRACT, "null argument");
    CYC_CUDA(cudaSetDevice(ctx->device));
    cudaError_t e = cudaMalloc(out, bytes ? bytes : 1);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      throw Error(CYC_E_RESOURCE, "device memory exhausted");
    }
    CYC_CUDA(e);
  });
}

void cyc_device_free(cyc_ctx* ctx, void* p) {
  if (!p) return;
  if (ctx) cudaSetDevice(ctx->device);
  cudaFree(p);
}

cyc_status cyc_memcpy(cyc_ctx* ctx, void* dst, const void* src, size_t bytes) {
  return guard([&] {
    require(ctx, CYC_E_CONTRACT, "null ctx");
    CYC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->s));
    CYC_CUDA(cudaStreamSynchronize(ctx->s));
  });
}

cyc_status cyc_memcpy_async(cyc_ctx* ctx, void* dst, const void* src, size_t bytes) {
  return guard([&] {
    require(ctx, CYC_E_CONTRACT, "null ctx");
    CYC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->s));
  });
}

cyc_status cyc_flush_l2(cyc_ctx* ctx, size_t bytes) {
  return guard([&] {
    require(ctx, CYC_E_CONTRACT, "null ctx");
    if (ctx->flush.bytes < bytes) ctx->flush.alloc(bytes, ctx->s);
    CYC_CUDA(cudaMemsetAsync(ctx->flush.p, (int)(cyc::g_launches.load() & 0xFF), bytes, ctx->s));
  });
}

cyc_status cyc_shard_step(cyc_ctx* ctx, const cyc_graph* g, uint32_t lo, uint32_t hi,
                          const uint32_t* x, const uint64_t* acc_words, uint32_t* out, int64_t* rec,
                          const int64_t* state, int first_only) {
  return guard([&] {
    require(ctx && g && x && acc_words && rec && (out || hi <= lo), CYC_E_CONTRACT,
            "shard_step: null argument");
    require(lo <= hi && hi <= g->n(), CYC_E_CONTRACT, "shard_step: bad row range");
    require(is_device_ptr(x) && is_device_ptr(acc_words) && is_device_ptr(rec) &&
                (!state || is_device_ptr(state)),
            CYC_E_CONTRACT, "shard_step: vectors must be device memory");
    require(!first_only || state, CYC_E_CONTRACT, "shard_step: first_only needs the state");
    cyc::launch_step_range(g->gath, lo, hi, x, reinterpret_cast<const uint32_t*>(acc_words), out,
                           reinterpret_cast<long long*>(rec), reinterpret_cast<const long long*>(state),
                           first_only, ctx->s);
  });
}

cyc_status cyc_shard_post(cyc_ctx* ctx, const int64_t* rec, int64_t* state, const uint32_t* x_pad,
                          const uint32_t* bounds, int world, uint32_t maxrows, uint32_t* x) {
  return guard([&] {
    require(ctx && rec && state && bounds && world >= 1 && (x_pad || !maxrows) && (x || !maxrows),
            CYC_E_CONTRACT, "shard_post: bad argument");
    cyc::launch_shard_post(reinterpret_cast<const long long*>(rec), reinterpret_cast<long long*>(state),
                           x_pad, bounds, world, maxrows, x, ctx->s);
  });
}

cyc_status cyc_shard_collect(cyc_ctx* ctx, uint32_t lo, uint32_t hi, const uint32_t* x, const uint32_t* out,
                             uint32_t cap, uint32_t* sp, const int64_t* state, int list_mode,
                             const uint32_t* rlist, const uint32_t* rcnt, uint32_t* rbits,
                             const uint64_t* acc_words, int64_t* rec) {
  return guard([&] {
    require(ctx && x && sp && state && (out || hi <= lo), CYC_E_CONTRACT, "shard_collect: null argument");
    require(!list_mode || (rlist && rcnt && rbits && acc_words && rec), CYC_E_CONTRACT,
            "shard_collect: list mode needs the raised list and the record");
    cyc::launch_shard_collect(lo, hi, x, out, cap, reinterpret_cast<uint2*>(sp),
                              reinterpret_cast<const long long*>(state), list_mode, rlist, rcnt, rbits,
                              reinterpret_cast<const uint32_t*>(acc_words), reinterpret_cast<long long*>(rec),
                              ctx->s);
  });
}

cyc_status cyc_shard_push(cyc_ctx* ctx, const cyc_graph* g, uint32_t lo, uint32_t hi, const uint32_t* sp_all,
                          int world, uint32_t cap, const uint64_t* acc_words, uint32_t* out, uint32_t* rbits,
                          uint32_t* rlist, uint32_t* rcnt, const int64_t* state) {
  return guard([&] {
    require(ctx && g && sp_all && acc_words && out && rbits && rlist && rcnt && state && world >= 1,
            CYC_E_CONTRACT, "shard_push: null argument");
    require(lo <= hi && hi <= g->n(), CYC_E_CONTRACT, "shard_push: bad row range");
    cyc::launch_shard_push(reinterpret_cast<const uint2*>(sp_all), world, cap, g->snap, lo, hi,
                           reinterpret_cast<const uint32_t*>(acc_words), out, rbits, rlist, rcnt,
                           reinterpret_cast<const long long*>(state), ctx->s);
  });
}

cyc_status cyc_shard_post_sparse(cyc_ctx* ctx, const int64_t* rec, int64_t* state, const uint32_t* sp_all,
                                 int world, uint32_t cap, uint32_t* x) {
  return guard([&] {
    require(ctx && rec && state && sp_all && x && world >= 1, CYC_E_CONTRACT, "shard_post_sparse: bad argument");
    cyc::launch_shard_post_sparse(reinterpret_cast<const long long*>(rec), reinterpret_cast<long long*>(state),
                                  reinterpret_cast<const uint2*>(sp_all), world, cap, x, ctx->s);
  });
}

cyc_status cyc_fused_open(cyc_ctx* ctx, const cyc_graph* g, uint32_t lo, uint32_t hi, int rank, int world,
                          cyc_fused** out, void* handle_out) {
  return guard([&] {
    require(ctx && g && out && handle_out, CYC_E_CONTRACT, "fused_open: null argument");
    CYC_CUDA(cudaSetDevice(ctx->device));
    auto* f = new cyc_fused;
    try {
      f->ctx = ctx;
      f->g = g;
      f->sh.open(g->gath, lo, hi, rank, world, handle_out);
    } catch (...) {
      delete f;
      throw;
    }
    ctx->refs.fetch_add(1);
    *out = f;
  });
}

cyc_status cyc_fused_connect(cyc_fused* f, const void* handles) {
  return guard([&] {
    require(f && handles, CYC_E_CONTRACT, "fused_connect: null argument");
    CYC_CUDA(cudaSetDevice(f->ctx->device));
    f->sh.connect(handles);
  });
}

cyc_status cyc_fused_run(cyc_fused* f, const uint64_t* acc_words, int early_exit, cyc_map_stats* st,
                         uint32_t* final_values) {
  return guard([&] {
    require(f && acc_words, CYC_E_CONTRACT, "fused_run: null argument");
    CYC_CUDA(cudaSetDevice(f->ctx->device));
    unsigned long long res[6];
    f->sh.run(acc_words, early_exit, f->ctx->s, res);
    if (st) {
      std::memset(st, 0, sizeof *st);
      st->cycle_found = (int32_t)res[0];
      st->witness = (uint32_t)res[1];
      st->iterations = res[2];
      st->kernel_calls = res[3];
      st->demoted_total = res[4];
    }
    if (final_values) f->sh.final_vector(final_values, f->ctx->s);
  });
}

void cyc_fused_close(cyc_fused* f) {
  if (!f) return;
  cyc_ctx* c = f->ctx;
  cudaSetDevice(c->device);
  delete f;
  ctx_release(c);
}

cyc_status cyc_shard_demote(cyc_ctx* ctx, const uint32_t* x, uint32_t n, const uint64_t* acc_words,
                            uint64_t* remaining, uint64_t* counts) {
  return guard([&] {
    require(ctx && (x || !n) && acc_words && remaining && counts, CYC_E_CONTRACT,
            "shard_demote: null argument");
    const size_t words = ((size_t)n + 31) / 32 + 2;
    if (ctx->flush.bytes < words * 4) ctx->flush.alloc(words * 4, ctx->s);  // reused as scratch
    CYC_CUDA(cudaMemsetAsync(ctx->flush.p, 0, words * 4, ctx->s));
    cyc::launch_demote_async(x, n, reinterpret_cast<const uint32_t*>(acc_words),
                             reinterpret_cast<uint32_t*>(remaining),
                             reinterpret_cast<unsigned long long*>(counts), ctx->flush.as<uint32_t>(),
                             ctx->s);
  });
}

// map_engine.cpp:35-43: bounds[w] = lower_bound(offsets, total*w/parts).
cyc_status cyc_map_trace(const cyc_graph* g, uint64_t* out, uint32_t cap, uint32_t* len) {
  return guard([&] {
    require(g && len, CYC_E_CONTRACT, "null argument");
    const uint32_t k = g->ws.trace_len < cap ? g->ws.trace_len : cap;
    *len = k;
    if (k && out) {
      copy_out(out, g->ws.trace.as<uint64_t>(), (size_t)k * 64, g->ctx->s);
      CYC_CUDA(cudaStreamSynchronize(g->ctx->s));
    }
  });
}

cyc_status cyc_shard_bounds(const uint64_t* row_offsets, uint32_t n, int parts, uint32_t* bounds) {
  return guard([&] {
    require(row_offsets && bounds && parts >= 1, CYC_E_CONTRACT, "shard_bounds: bad argument");
    const uint64_t total = row_offsets[n];
    bounds[0] = 0;
    for (int w = 1; w < parts; ++w) {
      uint64_t target = total * (uint64_t)w / (uint64_t)parts;
      uint32_t lo = 0, hi = n + 1;  // first index with offsets[idx] >= target
      while (lo < hi) {
        uint32_t mid = lo + (hi - lo) / 2;
        if (row_offsets[mid] < target) lo = mid + 1; else hi = mid;
      }
      bounds[w] = lo < n ? lo : n;
    }
    bounds[parts] = n;
  });
}

}  // extern "C"
