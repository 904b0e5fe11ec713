// ingest.cu — explicit-graph ingestion on the device:
// parse_explicit_graph (reference graph.cpp:259-297) for files far beyond
// what a std::getline/istringstream loop reads in reasonable time, plus a
// binary edge-list format for the same graphs.
//
// Text format (graph.hpp:136-146): "graph <n>", "accepting <id>...", then
// "edge <src> <dst>" lines; '#' starts a comment; blank lines are skipped.
// The parse is data-parallel over bytes and lines:
//   1. newline positions: per-tile counts, scan, per-tile write (uint4 loads);
//   2. one thread per line: comment cut, whitespace tokens (isspace set of the
//      "C" locale), line kind, and for edge lines the two ids parsed with
//      parse_vertex_id's semantics made n-independent (digit prefix before
//      the first non-digit, saturated, plus flags) so they can be parsed
//      before n is known;
//   3. scan of the non-empty flags: rank 0 is the graph line, rank 1 the
//      accepting line, ranks >= 2 are edges in file order;
//   4. the graph line is parsed on the host (one line, exact std::stoul
//      semantics); the accepting line token-parallel on the device;
//   5. edge lines validated against n, first failing line by atomicMin.
// The earliest failing line wins, as the reference's sequential loop throws
// at the first offending line; its message is rebuilt on the host from that
// one line so it matches ParseError's text exactly.
#include <cstring>
#include <string>
#include <vector>

#include "ingest.cuh"

namespace cyc {

namespace {

constexpr int kT = 256;
constexpr uint32_t kTileBytes = kT * 16;  // one uint4 per thread per tile

// line status byte: bits 0-2 kind, 3 tok1 has non-digit, 4 tok2 has non-digit,
// 5 exactly three tokens
enum : uint8_t { kEmpty = 0, kGraph = 1, kAccepting = 2, kEdge = 3, kOther = 4 };
constexpr uint8_t kNd1 = 8, kNd2 = 16, kThree = 32;

__device__ __forceinline__ bool is_space(uint8_t c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

__global__ void k_nl_count(const uint8_t* __restrict__ t, uint64_t len, uint32_t* tilecnt, uint32_t ntiles) {
  __shared__ uint32_t s;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    if (threadIdx.x == 0) s = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)tile * kTileBytes + threadIdx.x * 16ull;
    uint32_t c = 0;
    if (base + 16 <= len) {
      const uint4 w = *reinterpret_cast<const uint4*>(t + base);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) c += __popc(__vcmpeq4(ws[k], 0x0A0A0A0Au)) >> 3;  // 0xFF per '\n' byte
    } else {
      for (uint64_t i = base; i < len && i < base + 16; ++i) c += t[i] == '\n';
    }
    c = __reduce_add_sync(kFull, c);
    if ((threadIdx.x & 31u) == 0 && c) atomicAdd(&s, c);
    __syncthreads();
    if (threadIdx.x == 0) tilecnt[tile] = s;
    __syncthreads();
  }
}

__global__ void k_nl_write(const uint8_t* __restrict__ t, uint64_t len, const uint32_t* __restrict__ tilebase,
                           uint32_t ntiles, uint64_t* nl) {
  __shared__ uint32_t warp_sum[kT / 32];
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t base = (uint64_t)tile * kTileBytes + threadIdx.x * 16ull;
    uint8_t b[16];
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      b[k] = base + k < len ? t[base + k] : 0;
      c += b[k] == '\n';
    }
    const uint32_t incl = warp_incl_scan(c);
    if ((threadIdx.x & 31u) == 31u) warp_sum[threadIdx.x >> 5] = incl;
    __syncthreads();
    uint32_t before = 0;
    for (uint32_t w = 0; w < (threadIdx.x >> 5); ++w) before += warp_sum[w];
    uint32_t pos = tilebase[tile] + before + incl - c;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (b[k] == '\n') nl[pos++] = base + k;
    __syncthreads();
  }
}

struct LineSpan {
  const uint64_t* nl;
  uint64_t n_nl, len;
  __device__ void get(uint64_t i, uint64_t& b, uint64_t& e) const {
    b = i ? nl[i - 1] + 1 : 0;
    e = i < n_nl ? nl[i] : len;
  }
};

// digit prefix of a token (saturated to 0xFFFFFFFF) and whether a non-digit
// follows it (parse_vertex_id, graph.cpp:245-256, minus the n-dependent break)
__device__ __forceinline__ void prefix_value(const uint8_t* t, uint64_t b, uint64_t e, uint32_t& val, bool& nd) {
  uint64_t v = 0;
  nd = false;
  for (uint64_t i = b; i < e; ++i) {
    const uint8_t c = t[i];
    if (c < '0' || c > '9') {
      nd = true;
      break;
    }
    v = v * 10 + (c - '0');
    if (v > 0xFFFFFFFFull) v = 0x100000000ull;  // saturate (any n is < 2^32)
  }
  val = v > 0xFFFFFFFEull ? 0xFFFFFFFFu : (uint32_t)v;
}

__device__ __forceinline__ bool tok_is(const uint8_t* t, uint64_t b, uint64_t e, const char* w, int wl) {
  if (e - b != (uint64_t)wl) return false;
  for (int k = 0; k < wl; ++k)
    if (t[b + k] != (uint8_t)w[k]) return false;
  return true;
}

__global__ void k_lines(const uint8_t* __restrict__ t, LineSpan ls, uint64_t nlines, uint8_t* status,
                        uint32_t* nonempty, uint2* raw) {
  for (uint64_t li = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; li < nlines;
       li += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t b, e;
    ls.get(li, b, e);
    uint64_t tb[3] = {0, 0, 0}, te[3] = {0, 0, 0};
    uint32_t nt = 0;
    bool in = false;
    for (uint64_t i = b; i < e; ++i) {
      const uint8_t c = t[i];
      if (c == '#') break;
      if (is_space(c)) {
        if (in && nt <= 3) te[nt - 1] = i;
        in = false;
      } else if (!in) {
        in = true;
        ++nt;
        if (nt <= 3) tb[nt - 1] = i;
        if (nt > 3) break;  // more than three tokens: only the kind matters
      }
    }
    if (in && nt <= 3) {  // token running to the comment / end of line
      uint64_t i = tb[nt - 1];
      while (i < e && t[i] != '#' && !is_space(t[i])) ++i;
      te[nt - 1] = i;
    }
    uint8_t st = kEmpty;
    if (nt) {
      if (tok_is(t, tb[0], te[0], "graph", 5)) st = kGraph;
      else if (tok_is(t, tb[0], te[0], "accepting", 9)) st = kAccepting;
      else if (tok_is(t, tb[0], te[0], "edge", 4)) st = kEdge;
      else st = kOther;
    }
    uint2 r = make_uint2(0, 0);
    if (st == kEdge && nt == 3) {
      bool nd1, nd2;
      prefix_value(t, tb[1], te[1], r.x, nd1);
      prefix_value(t, tb[2], te[2], r.y, nd2);
      st |= kThree | (nd1 ? kNd1 : 0) | (nd2 ? kNd2 : 0);
    }
    status[li] = st;
    nonempty[li] = nt ? 1u : 0u;
    raw[li] = r;
  }
}

// checks one parsed id against n exactly as parse_vertex_id: 0 ok, 1 syntax, 2 range
__device__ __forceinline__ uint32_t id_check(uint32_t val, bool nd, uint32_t n) {
  if (nd && val <= n) return 1;
  return val >= n ? 2u : 0u;
}

__global__ void k_find_heads(uint64_t nlines, const uint32_t* nonempty, const uint32_t* rank, uint64_t* heads) {
  for (uint64_t li = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; li < nlines;
       li += (uint64_t)gridDim.x * blockDim.x)
    if (nonempty[li] && rank[li] < 2) heads[rank[li]] = li;
}

__global__ void k_edges(uint64_t nlines, uint64_t first, const uint8_t* status, const uint32_t* nonempty,
                        const uint32_t* rank, const uint2* raw, uint32_t n, uint2* edges,
                        unsigned long long* err_line) {
  for (uint64_t li = first + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; li < nlines;
       li += (uint64_t)gridDim.x * blockDim.x) {
    if (!nonempty[li]) continue;
    const uint8_t st = status[li];
    bool bad = (st & 7) != kEdge || !(st & kThree);
    const uint2 r = raw[li];
    if (!bad) bad = id_check(r.x, st & kNd1, n) || id_check(r.y, st & kNd2, n);
    if (bad) {
      atomicMin(err_line, (unsigned long long)li);
    } else {
      edges[rank[li] - 2] = r;
    }
  }
}

// accepting line: token starts in [b, e) (comment already excluded)
__global__ void k_tok_starts(const uint8_t* __restrict__ t, uint64_t b, uint64_t e, uint32_t* flag) {
  for (uint64_t i = b + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const bool tok = !is_space(t[i]) && (i == b || is_space(t[i - 1]));
    flag[i - b] = tok ? 1u : 0u;
  }
}

__global__ void k_acc_parse(const uint8_t* __restrict__ t, uint64_t b, uint64_t e, const uint32_t* flag,
                            const uint32_t* pos, uint32_t n, uint32_t* ids, unsigned long long* err_tok) {
  for (uint64_t i = b + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (!flag[i - b]) continue;
    const uint32_t k = pos[i - b];
    if (k == 0) continue;  // the word "accepting"
    uint64_t j = i;
    while (j < e && !is_space(t[j])) ++j;
    uint32_t val;
    bool nd;
    prefix_value(t, i, j, val, nd);
    if (id_check(val, nd, n)) atomicMin(err_tok, (unsigned long long)k);
    else ids[k - 1] = val;
  }
}

__global__ void k_ids_to_words(const uint32_t* ids, uint64_t k, uint32_t* words) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k; i += (uint64_t)gridDim.x * blockDim.x)
    atomicOr(words + (ids[i] >> 5), 1u << (ids[i] & 31u));
}

__global__ void k_words_to_ids(const uint32_t* words, uint32_t n, const uint32_t* pos, uint32_t* ids) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if ((words[v >> 5] >> (v & 31u)) & 1u) ids[pos[v]] = v;
}

__global__ void k_bits32(const uint32_t* words, uint32_t n, uint32_t* f) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    f[v] = (words[v >> 5] >> (v & 31u)) & 1u;
}

// ---- host side: exact re-statement for the one line that decides an error
bool host_space(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

std::vector<std::string> host_tokens(const std::string& line) {
  std::string body = line.substr(0, line.find('#'));
  std::vector<std::string> toks;
  size_t i = 0;
  while (i < body.size()) {
    while (i < body.size() && host_space(body[i])) ++i;
    size_t j = i;
    while (j < body.size() && !host_space(body[j])) ++j;
    if (j > i) toks.push_back(body.substr(i, j - i));
    i = j;
  }
  return toks;
}

[[noreturn]] void parse_fail(int code, uint64_t line, const std::string& msg) {
  throw ParseFailure(code, (int)line, 1, msg);
}

// parse_vertex_id (graph.cpp:245-256)
uint32_t host_vertex_id(const std::string& tok, uint32_t n, uint64_t line) {
  uint64_t value = 0;
  for (char c : tok) {
    if (c < '0' || c > '9') parse_fail(kDiagSyntax, line, "expected vertex id, got '" + tok + "'");
    value = value * 10 + (uint64_t)(c - '0');
    if (value > n) break;
  }
  if (value >= n)
    parse_fail(kDiagRange, line, "vertex id " + tok + " out of range [0, " + std::to_string(n) + ")");
  return (uint32_t)value;
}

// std::stoul(tok) then the VertexId cast (graph.cpp:269-273)
uint32_t host_vertex_count(const std::string& tok, uint64_t line) {
  size_t i = 0;
  bool neg = false;
  if (i < tok.size() && (tok[i] == '+' || tok[i] == '-')) neg = tok[i++] == '-';
  const size_t d0 = i;
  unsigned long long v = 0;
  bool overflow = false;
  for (; i < tok.size() && tok[i] >= '0' && tok[i] <= '9'; ++i) {
    const unsigned d = (unsigned)(tok[i] - '0');
    if (v > (~0ull - d) / 10) overflow = true;
    v = v * 10 + d;
  }
  if (i == d0 || overflow) parse_fail(kDiagSyntax, line, "bad vertex count '" + tok + "'");
  if (neg) v = 0ull - v;
  return (uint32_t)v;
}

std::string line_text(const uint8_t* dtext, const std::vector<uint64_t>& span, cudaStream_t s) {
  std::string str(span[1] - span[0], '\0');
  if (!str.empty()) {
    CYC_CUDA(cudaMemcpyAsync(&str[0], dtext + span[0], str.size(), cudaMemcpyDefault, s));
    CYC_CUDA(cudaStreamSynchronize(s));
  }
  return str;
}

}  // namespace

void parse_explicit_device(const uint8_t* dtext, uint64_t len, cudaStream_t s, ExplicitDev& out) {
  // 1. newlines
  const uint32_t ntiles = (uint32_t)((len + kTileBytes - 1) / kTileBytes);
  DevBuf tilecnt(((size_t)ntiles + 1) * 4, s), tilebase(((size_t)ntiles + 2) * 4, s), scratch;
  uint32_t n_nl = 0;
  if (ntiles) {
    k_nl_count<<<grid_for(ntiles, 1, 8), kT, 0, s>>>(dtext, len, tilecnt.as<uint32_t>(), ntiles);
    CYC_LAUNCHED();
  }
  exclusive_scan(tilecnt.as<uint32_t>(), tilebase.as<uint32_t>(), ntiles, nullptr, s, scratch);
  CYC_CUDA(cudaMemcpyAsync(&n_nl, tilebase.as<uint32_t>() + ntiles, 4, cudaMemcpyDeviceToHost, s));
  uint8_t last = '\n';
  if (len) CYC_CUDA(cudaMemcpyAsync(&last, dtext + len - 1, 1, cudaMemcpyDefault, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  DevBuf nl(((size_t)n_nl + 1) * 8, s);
  if (ntiles) {
    k_nl_write<<<grid_for(ntiles, 1, 8), kT, 0, s>>>(dtext, len, tilebase.as<uint32_t>(), ntiles,
                                                     nl.as<uint64_t>());
    CYC_LAUNCHED();
  }
  const uint64_t nlines = (uint64_t)n_nl + (len && last != '\n' ? 1 : 0);
  require_ingest(nlines < 0xFFFFFFFFull, "explicit graph: too many lines");
  LineSpan ls{nl.as<uint64_t>(), n_nl, len};
  // 2. per-line scan
  DevBuf status(nlines + 1, s), nonempty((nlines + 1) * 4, s), rank((nlines + 2) * 4, s), raw((nlines + 1) * 8, s);
  if (nlines) {
    k_lines<<<grid_for(nlines, kT, 8), kT, 0, s>>>(dtext, ls, nlines, status.as<uint8_t>(),
                                                   nonempty.as<uint32_t>(), raw.as<uint2>());
    CYC_LAUNCHED();
  }
  // 3. ranks of non-empty lines
  exclusive_scan(nonempty.as<uint32_t>(), rank.as<uint32_t>(), (uint32_t)nlines, nullptr, s, scratch);
  uint32_t nne = 0;
  DevBuf heads(16, s);
  CYC_CUDA(cudaMemsetAsync(heads.p, 0xFF, 16, s));
  CYC_CUDA(cudaMemcpyAsync(&nne, rank.as<uint32_t>() + nlines, 4, cudaMemcpyDeviceToHost, s));
  if (nlines) {
    k_find_heads<<<grid_for(nlines, kT, 8), kT, 0, s>>>(nlines, nonempty.as<uint32_t>(), rank.as<uint32_t>(),
                                                        heads.as<uint64_t>());
    CYC_LAUNCHED();
  }
  uint64_t hl[2];
  CYC_CUDA(cudaMemcpyAsync(hl, heads.p, 16, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  auto span_of = [&](uint64_t li) {
    std::vector<uint64_t> sp(2);
    uint64_t h[2] = {0, 0};
    if (li) CYC_CUDA(cudaMemcpyAsync(&h[0], nl.as<uint64_t>() + li - 1, 8, cudaMemcpyDeviceToHost, s));
    if (li < n_nl) CYC_CUDA(cudaMemcpyAsync(&h[1], nl.as<uint64_t>() + li, 8, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
    sp[0] = li ? h[0] + 1 : 0;
    sp[1] = li < n_nl ? h[1] : len;
    return sp;
  };
  // 4a. graph line (section 0)
  if (nne == 0) parse_fail(kDiagSyntax, nlines, "empty graph file");
  {
    const auto toks = host_tokens(line_text(dtext, span_of(hl[0]), s));
    if (toks[0] != "graph" || toks.size() != 2) parse_fail(kDiagSyntax, hl[0] + 1, "expected 'graph <n>'");
    out.n = host_vertex_count(toks[1], hl[0] + 1);
  }
  const uint32_t n = out.n;
  // 4b. accepting line (section 1), token-parallel
  if (nne == 1) parse_fail(kDiagSyntax, nlines, "missing 'accepting' line");
  {
    const auto sp = span_of(hl[1]);
    uint8_t st = 0;
    CYC_CUDA(cudaMemcpyAsync(&st, status.as<uint8_t>() + hl[1], 1, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
    if ((st & 7) != kAccepting) parse_fail(kDiagSyntax, hl[1] + 1, "expected 'accepting ...'");
    // the comment cut: first '#' of the line (found on the device by a scan
    // would be overkill; lines are read once more here in tiles)
    uint64_t b = sp[0], e = sp[1];
    {
      std::string probe;
      const uint64_t chunk = 1 << 20;
      for (uint64_t at = b; at < e; at += chunk) {
        probe.assign((size_t)std::min<uint64_t>(chunk, e - at), '\0');
        CYC_CUDA(cudaMemcpyAsync(&probe[0], dtext + at, probe.size(), cudaMemcpyDefault, s));
        CYC_CUDA(cudaStreamSynchronize(s));
        const size_t h = probe.find('#');
        if (h != std::string::npos) {
          e = at + h;
          break;
        }
      }
    }
    const uint64_t w = e - b;
    require_ingest(w < 0xFFFFFFFFull, "explicit graph: accepting line too long");
    DevBuf flag((w + 1) * 4, s), pos((w + 2) * 4, s), errt(8, s);
    if (w) {
      k_tok_starts<<<grid_for(w, kT, 8), kT, 0, s>>>(dtext, b, e, flag.as<uint32_t>());
      CYC_LAUNCHED();
    }
    exclusive_scan(flag.as<uint32_t>(), pos.as<uint32_t>(), (uint32_t)w, nullptr, s, scratch);
    uint32_t ntok = 0;
    CYC_CUDA(cudaMemcpyAsync(&ntok, pos.as<uint32_t>() + w, 4, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
    out.n_acc = ntok ? ntok - 1 : 0;
    out.acc_ids.alloc((out.n_acc + 1) * 4, s);
    CYC_CUDA(cudaMemsetAsync(errt.p, 0xFF, 8, s));
    if (w) {
      k_acc_parse<<<grid_for(w, kT, 8), kT, 0, s>>>(dtext, b, e, flag.as<uint32_t>(), pos.as<uint32_t>(), n,
                                                     out.acc_ids.as<uint32_t>(),
                                                     reinterpret_cast<unsigned long long*>(errt.p));
      CYC_LAUNCHED();
    }
    unsigned long long bad_tok = ~0ull;
    CYC_CUDA(cudaMemcpyAsync(&bad_tok, errt.p, 8, cudaMemcpyDeviceToHost, s));
    CYC_CUDA(cudaStreamSynchronize(s));
    if (bad_tok != ~0ull) {  // rebuild the message from that token on the host
      const auto toks = host_tokens(line_text(dtext, sp, s));
      for (size_t k = 1; k < toks.size(); ++k) host_vertex_id(toks[k], n, hl[1] + 1);
      throw Error(CYC_E_CUDA, "internal: accepting-line parse disagrees with the host check");
    }
  }
  // 5. edges (section 2)
  out.m = nne - 2;
  out.edges.alloc((out.m + 1) * 8, s);
  DevBuf errl(8, s);
  CYC_CUDA(cudaMemsetAsync(errl.p, 0xFF, 8, s));
  if (out.m) {
    k_edges<<<grid_for(nlines - hl[1], kT, 8), kT, 0, s>>>(nlines, hl[1] + 1, status.as<uint8_t>(),
                                                           nonempty.as<uint32_t>(), rank.as<uint32_t>(),
                                                           raw.as<uint2>(), n, out.edges.as<uint2>(),
                                                           reinterpret_cast<unsigned long long*>(errl.p));
    CYC_LAUNCHED();
  }
  unsigned long long bad_line = ~0ull;
  CYC_CUDA(cudaMemcpyAsync(&bad_line, errl.p, 8, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  if (bad_line != ~0ull) {
    const auto toks = host_tokens(line_text(dtext, span_of(bad_line), s));
    if (toks[0] != "edge" || toks.size() != 3) parse_fail(kDiagSyntax, bad_line + 1, "expected 'edge <src> <dst>'");
    host_vertex_id(toks[1], n, bad_line + 1);
    host_vertex_id(toks[2], n, bad_line + 1);
    throw Error(CYC_E_CUDA, "internal: edge-line parse disagrees with the host check");
  }
}

void explicit_acc_words(const ExplicitDev& g, cudaStream_t s, DevBuf& words) {
  const size_t nw = ((size_t)g.n + 63) / 64 + 1;
  words.alloc(nw * 8, s);
  CYC_CUDA(cudaMemsetAsync(words.p, 0, nw * 8, s));
  if (g.has_words) {
    CYC_CUDA(cudaMemcpyAsync(words.p, g.acc_words.p, ((size_t)g.n + 63) / 64 * 8, cudaMemcpyDeviceToDevice, s));
  } else if (g.n_acc) {
    k_ids_to_words<<<grid_for(g.n_acc, kT, 8), kT, 0, s>>>(g.acc_ids.as<uint32_t>(), g.n_acc, words.as<uint32_t>());
    CYC_LAUNCHED();
  }
}

void explicit_acc_ids_from_words(ExplicitDev& g, cudaStream_t s) {
  const uint32_t n = g.n;
  DevBuf f(((size_t)n + 1) * 4, s), pos(((size_t)n + 2) * 4, s), scratch;
  if (n) {
    k_bits32<<<grid_for(n, kT, 8), kT, 0, s>>>(g.acc_words.as<uint32_t>(), n, f.as<uint32_t>());
    CYC_LAUNCHED();
  }
  exclusive_scan(f.as<uint32_t>(), pos.as<uint32_t>(), n, nullptr, s, scratch);
  uint32_t k = 0;
  CYC_CUDA(cudaMemcpyAsync(&k, pos.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, s));
  CYC_CUDA(cudaStreamSynchronize(s));
  g.n_acc = k;
  g.acc_ids.alloc(((size_t)k + 1) * 4, s);
  if (n && k) {
    k_words_to_ids<<<grid_for(n, kT, 8), kT, 0, s>>>(g.acc_words.as<uint32_t>(), n, pos.as<uint32_t>(),
                                                      g.acc_ids.as<uint32_t>());
    CYC_LAUNCHED();
  }
}

}  // namespace cyc
