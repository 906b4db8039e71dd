// Text ingestion on the device: parse_edge_list / parse_dimacs_gr
// (core/src/graph.cpp:57-133), SURVEY.md 8(f) row 3.
//
// The reference reads the stream line by line (std::getline), tokenises with
// operator>>, parses ids with std::from_chars, and normalises edges through an
// unordered_set (self-loops and repeated unordered pairs dropped, first
// occurrence kept, in input order).  On the device:
//
//   k_newlines + compact_u8   positions of '\n' -> line boundaries
//   k_parse_lines<kDimacs>    one thread per line: classify, tokenise the
//                             first 2 (edge list) or 4 (DIMACS) tokens,
//                             from_chars-exact i64 parsing, per-line error code
//   k_arc_check (DIMACS)      governing problem line of every arc line by
//                             binary search over the compacted 'p' lines:
//                             "arc line before problem line" and the [1, n]
//                             range check against that line's n
//   k_first_error             the reference throws at the first bad line:
//                             atomicMin over erroneous line indices
//   k_edge_candidates         n, self-loop count, candidate flags
//   2 x sort_pairs            stable LSD sort by (min, max) with the candidate
//                             index as payload -> first occurrence of each pair
//   compact_u8                kept edges in input order
//
// Error messages are the reference's strings; the host formats the one for
// the first bad line from its own copy of the text (the token in "malformed
// integer token '...'").  Node ids must be < 2^32 for the on-device
// deduplication keys (the reference accepts any i64; every downstream device
// stage needs n < 2^31 anyway): larger ids give ETTG_ERANGE.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "api_internal.cuh"
#include "common.cuh"
#include "scan.cuh"
#include "sort.cuh"
#include "trace.cuh"

namespace ettg {
namespace {

enum : uint8_t { kLSkip = 0, kLEdge = 1, kLProblem = 2, kLArc = 3 };
enum : uint8_t {
  kEOk = 0,
  kETwoTokens,   // "expected two integer tokens"
  kEMalformedA,  // first id token
  kEMalformedB,  // second id token
  kENegative,    // "negative node id"
  kEProblem,     // "malformed problem line"
  kEMalformedN,  // problem line's n token
  kEArcTokens,   // "expected two node ids"
  kEArcBefore,   // "arc line before problem line"
  kERange,       // "node id outside [1, n]"
};

__device__ __forceinline__ bool is_ws(uint8_t c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// Next whitespace-delimited token in [p, end) (operator>> on a string).
__device__ __forceinline__ bool next_token(const uint8_t* t, u64& p, u64 end, u64& t0, u64& t1) {
  while (p < end && is_ws(t[p])) ++p;
  if (p >= end) return false;
  t0 = p;
  while (p < end && !is_ws(t[p])) ++p;
  t1 = p;
  return true;
}

// std::from_chars(first, last, i64): optional '-', >= 1 decimal digit, no
// overflow, and the whole token consumed.
__device__ __forceinline__ bool parse_i64(const uint8_t* t, u64 t0, u64 t1, long long& out) {
  bool neg = false;
  if (t0 < t1 && t[t0] == '-') {
    neg = true;
    ++t0;
  }
  if (t0 >= t1) return false;
  const u64 lim = neg ? (u64(1) << 63) : (u64(1) << 63) - 1;
  u64 v = 0;
  for (u64 i = t0; i < t1; ++i) {
    const uint8_t c = t[i];
    if (c < '0' || c > '9') return false;
    const u64 d = c - '0';
    if (v > (lim - d) / 10) return false;  // v * 10 + d > lim
    v = v * 10 + d;
  }
  out = neg ? static_cast<long long>(0 - v) : static_cast<long long>(v);
  return true;
}

__global__ void k_newlines(const uint8_t* __restrict__ t, u64 len, uint8_t* __restrict__ nl) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < len; i += u64(gridDim.x) * blockDim.x)
    nl[i] = t[i] == '\n';
}

struct PosOut {
  u32* pos;
  __device__ __forceinline__ void operator()(u64 i, u32 rank) const { pos[rank] = static_cast<u32>(i); }
};

struct Lines {
  const uint8_t* text;
  u64 len;
  const u32* nlpos;
  u32 nnl;
  __device__ __forceinline__ void bounds(u32 j, u64& s, u64& e) const {
    s = j == 0 ? 0 : u64(nlpos[j - 1]) + 1;
    e = j < nnl ? u64(nlpos[j]) : len;
  }
};

template <bool kDimacs>
__global__ void k_parse_lines(Lines L, u32 nlines, uint8_t* __restrict__ kind,
                              uint8_t* __restrict__ err, long long* __restrict__ va,
                              long long* __restrict__ vb) {
  for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < nlines; j += gridDim.x * blockDim.x) {
    u64 s, e;
    L.bounds(j, s, e);
    const uint8_t* t = L.text;
    uint8_t k = kLSkip, er = kEOk;
    long long a = 0, b = 0;
    u64 p = s, t0, t1, u0, u1;
    if (!kDimacs) {
      if (s < e && t[s] != '#' && t[s] != '%' && next_token(t, p, e, t0, t1)) {
        k = kLEdge;
        if (!next_token(t, p, e, u0, u1)) er = kETwoTokens;
        else if (!parse_i64(t, t0, t1, a)) er = kEMalformedA;
        else if (!parse_i64(t, u0, u1, b)) er = kEMalformedB;
        else if (a < 0 || b < 0) er = kENegative;
      }
    } else if (s < e && t[s] != 'c' && next_token(t, p, e, t0, t1) && t1 == t0 + 1) {
      const uint8_t c = t[t0];
      if (c == 'p') {
        k = kLProblem;
        u64 w0, w1;
        if (!next_token(t, p, e, w0, w1) || !next_token(t, p, e, u0, u1) ||
            !next_token(t, p, e, w0, w1))
          er = kEProblem;
        else if (!parse_i64(t, u0, u1, a)) er = kEMalformedN;
      } else if (c == 'a' || c == 'e') {
        k = kLArc;
        if (!next_token(t, p, e, t0, t1) || !next_token(t, p, e, u0, u1)) er = kEArcTokens;
        else if (!parse_i64(t, t0, t1, a)) er = kEMalformedA;
        else if (!parse_i64(t, u0, u1, b)) er = kEMalformedB;
      }
    }
    kind[j] = k;
    err[j] = er;
    va[j] = a;
    vb[j] = b;
  }
}

__global__ void k_kind_flags(const uint8_t* __restrict__ kind, u32 nlines, uint8_t want,
                             uint8_t* __restrict__ flags) {
  for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < nlines; j += gridDim.x * blockDim.x)
    flags[j] = kind[j] == want;
}

// DIMACS: the problem line governing arc line j is the last one before it
// (core/src/graph.cpp:96-118 keeps overwriting declared_n).
__global__ void k_arc_check(const uint8_t* __restrict__ kind, uint8_t* __restrict__ err,
                            const long long* __restrict__ va, const long long* __restrict__ vb,
                            u32 nlines, const u32* __restrict__ plist, u32 np) {
  for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < nlines; j += gridDim.x * blockDim.x) {
    if (kind[j] != kLArc) continue;
    u32 lo = 0, hi = np;  // first p index >= j
    while (lo < hi) {
      const u32 mid = (lo + hi) >> 1;
      if (plist[mid] < j) lo = mid + 1;
      else hi = mid;
    }
    if (lo == 0) {
      err[j] = kEArcBefore;
      continue;
    }
    if (err[j] != kEOk) continue;
    const long long n = va[plist[lo - 1]];
    const long long u = va[j], v = vb[j];
    if (u < 1 || u > n || v < 1 || v > n) err[j] = kERange;
  }
}

__global__ void k_first_error(const uint8_t* __restrict__ err, u32 nlines, u32* first) {
  u32 best = 0xFFFFFFFFu;
  for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < nlines; j += gridDim.x * blockDim.x)
    if (err[j] != kEOk) best = min(best, j);
  for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best != 0xFFFFFFFFu) atomicMin(first, best);
}

// Counters: [0] n (max id + 1, or declared n), [1] self-loops, [2] too-large flag
__global__ void k_edge_candidates(const uint8_t* __restrict__ kind, const long long* __restrict__ va,
                                  const long long* __restrict__ vb, u32 nlines, bool dimacs,
                                  uint8_t* __restrict__ cand, unsigned long long* counters) {
  unsigned long long nmax = 0, loops = 0, big = 0;
  for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < nlines; j += gridDim.x * blockDim.x) {
    uint8_t c = 0;
    const uint8_t k = kind[j];
    if (dimacs && k == kLProblem) {
      const long long d = va[j];
      if (d > 0) nmax = max(nmax, static_cast<unsigned long long>(d));
    } else if (k == (dimacs ? kLArc : kLEdge)) {
      const long long off = dimacs ? 1 : 0;
      const unsigned long long u = static_cast<unsigned long long>(va[j] - off);
      const unsigned long long v = static_cast<unsigned long long>(vb[j] - off);
      nmax = max(nmax, max(u, v) + 1);
      if (u == v) ++loops;
      else c = 1;
      if (max(u, v) > 0xFFFFFFFFull) big = 1;
    }
    cand[j] = c;
  }
  atomicMax(&counters[0], nmax);
  if (loops) atomicAdd(&counters[1], loops);
  if (big) atomicOr(&counters[2], big);
}

struct CandOut {  // candidate c <- line j: normalised (min, max) as u32 keys
  const long long* va;
  const long long* vb;
  long long off;
  u32* kmin;
  u32* kmax;
  u32* iota;
  __device__ __forceinline__ void operator()(u64 j, u32 c) const {
    const u32 u = static_cast<u32>(va[j] - off), v = static_cast<u32>(vb[j] - off);
    kmin[c] = min(u, v);
    kmax[c] = max(u, v);
    iota[c] = c;
  }
};

__global__ void k_gather_keys(const u32* __restrict__ kmin, const u32* __restrict__ perm, u32 C,
                              u32* __restrict__ out) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < C; i += gridDim.x * blockDim.x)
    out[i] = kmin[perm[i]];
}

// perm = candidates sorted by (min, max), stable: the first of each run of
// equal pairs is the earliest occurrence (the unordered_set keeps it).
__global__ void k_first_occurrence(const u32* __restrict__ kmin, const u32* __restrict__ kmax,
                                   const u32* __restrict__ perm, u32 C,
                                   uint8_t* __restrict__ keep) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < C; i += gridDim.x * blockDim.x) {
    const u32 c = perm[i];
    bool first = i == 0;
    if (!first) {
      const u32 p = perm[i - 1];
      first = kmin[c] != kmin[p] || kmax[c] != kmax[p];
    }
    keep[c] = first;
  }
}

struct EdgeOut {  // u32 pairs: half the D2H bytes; widened to i64 on the host
  const u32* kmin;
  const u32* kmax;
  u32 cap;
  uint2* out;
  __device__ __forceinline__ void operator()(u64 c, u32 r) const {
    if (r < cap) out[r] = make_uint2(kmin[c], kmax[c]);
  }
};

struct ParseWs {
  uint8_t* text = nullptr;
  uint8_t* flags = nullptr;  // newline flags (len) / per-line flags (nlines)
  u64* scan = nullptr;
  u32* nlpos = nullptr;
  uint8_t* kind = nullptr;
  uint8_t* err = nullptr;
  long long* va = nullptr;
  long long* vb = nullptr;
  u32* plist = nullptr;
  u32 *kmin = nullptr, *kmax = nullptr, *iota = nullptr, *k1 = nullptr, *v1 = nullptr,
      *k2 = nullptr, *v2 = nullptr;
  uint8_t* keep = nullptr;
  uint2* edges = nullptr;
  unsigned long long* counters = nullptr;
  u32* words = nullptr;
  SortWs sort;
  void carve(Carver& c, u64 len, u32 maxlines) {
    const u64 L = maxlines;  // `text` is allocated apart (it lands before the count)
    flags = c.take<uint8_t>(std::max<u64>(len, L) + 16);
    scan = c.take<u64>(scan_ws_words(std::max<u64>(len, L) + 1));
    nlpos = c.take<u32>(L + 1);
    kind = c.take<uint8_t>(L + 16);
    err = c.take<uint8_t>(L + 16);
    va = c.take<long long>(L);
    vb = c.take<long long>(L);
    plist = c.take<u32>(L + 1);
    kmin = c.take<u32>(L + 1);
    kmax = c.take<u32>(L + 1);
    iota = c.take<u32>(L + 1);
    k1 = c.take<u32>(L + 1);
    v1 = c.take<u32>(L + 1);
    k2 = c.take<u32>(L + 1);
    v2 = c.take<u32>(L + 1);
    keep = c.take<uint8_t>(L + 16);
    edges = c.take<uint2>(L + 1);
    counters = c.take<unsigned long long>(4);
    words = c.take<u32>(8);
    sort.carve(c, L + 1);
  }
};

// Host-side message for the first bad line (the reference's strings).
std::string host_token(const char* text, u64 s, u64 e, int which) {
  auto ws = [](char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
  };
  u64 p = s;
  for (int k = 0;; ++k) {
    while (p < e && ws(text[p])) ++p;
    const u64 t0 = p;
    while (p < e && !ws(text[p])) ++p;
    if (k == which) return std::string(text + t0, text + p);
  }
}

[[noreturn]] void parse_error(const char* text, u64 s, u64 e, u32 line, uint8_t code,
                              bool dimacs) {
  const std::string at = "line " + std::to_string(static_cast<u64>(line) + 1) + ": ";
  switch (code) {
    case kETwoTokens: throw Error(ETTG_EPARSE, at + "expected two integer tokens");
    case kEMalformedA:
    case kEMalformedB:
    case kEMalformedN: {
      // token index: edge list a/b = 0/1; DIMACS "a u v" u/v = 1/2, "p sp n m" n = 2
      const int which = code == kEMalformedN ? 2 : (code == kEMalformedA ? 0 : 1) + (dimacs ? 1 : 0);
      throw Error(ETTG_EPARSE, at + "malformed integer token '" + host_token(text, s, e, which) +
                                   "'");
    }
    case kENegative: throw Error(ETTG_EPARSE, at + "negative node id");
    case kEProblem: throw Error(ETTG_EPARSE, at + "malformed problem line");
    case kEArcTokens: throw Error(ETTG_EPARSE, at + "expected two node ids");
    case kEArcBefore: throw Error(ETTG_EPARSE, at + "arc line before problem line");
    case kERange: throw Error(ETTG_EPARSE, at + "node id outside [1, n]");
    default: throw Error(ETTG_EINTERNAL, at + "unknown parse error");
  }
}

void run_parse(const char* text, i64 len64, bool dimacs, int device, int64_t* edges_out,
               int64_t cap, int64_t* n_out, int64_t* m_out, ettg_parse_stats* stats) {
  if (len64 < 0 || (len64 > 0 && !text)) einval("null or negative text");
  if (!n_out || !m_out) einval("null argument");
  if (cap < 0 || (cap > 0 && !edges_out)) einval("null edge buffer");
  if (len64 >= (i64(1) << 32)) throw Error(ETTG_ERANGE, "text larger than 4 GiB");
  const u64 len = static_cast<u64>(len64);
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct SG {
    cudaStream_t s;
    ~SG() { cudaStreamDestroy(s); }
  } sg{st};
  // The text goes up first, into its own stream-ordered allocation; the host
  // threads count the newlines while they fill the pinned stage (the staging
  // copy reads every byte anyway), which sizes the per-line workspace.
  // lines = newlines + (1 if the text does not end in '\n'); the device
  // re-derives the newline positions.
  struct TextBuf {
    uint8_t* p = nullptr;
    cudaStream_t s = nullptr;
    ~TextBuf() {
      if (p) cudaFreeAsync(p, s);
    }
  } tb;
  tb.s = st;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&tb.p), len + 16, st));
  const u64 nnl_host = len ? staged_h2d_count(tb.p, text, len, '\n', device, st) : 0;
  const u64 nlines64 = nnl_host + ((len > 0 && text[len - 1] != '\n') ? 1 : 0);
  if (nlines64 >= 0xFFFFFFFFull) throw Error(ETTG_ERANGE, "too many lines");
  const u32 nlines = static_cast<u32>(nlines64);
  const int sms = sm_count(device);
  const unsigned g = sms * 8;
  ParseWs ws;
  Carver c;
  ws.carve(c, len, nlines);
  Lease lease(device, st, c.off);
  c = Carver{lease.base()};
  ws.carve(c, len, nlines);
  ws.text = tb.p;

  Trace tr(dimacs ? "parse_dimacs_gr" : "parse_edge_list", st);
  CK(cudaMemsetAsync(ws.counters, 0, 4 * sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(ws.words, 0xFF, 8 * sizeof(u32), st));
  tr.mark("h2d");
  if (len) {
    k_newlines<<<std::min(g, blocks_for(len, 256)), 256, 0, st>>>(ws.text, len, ws.flags);
    CK_LAUNCH();
    compact_u8(ws.flags, len, PosOut{ws.nlpos}, ws.scan, ws.words + 1, st);
  }
  tr.mark("lines");
  const Lines L{ws.text, len, ws.nlpos, static_cast<u32>(nnl_host)};
  if (nlines) {
    if (dimacs)
      k_parse_lines<true><<<std::min(g, blocks_for(nlines, 256)), 256, 0, st>>>(
          L, nlines, ws.kind, ws.err, ws.va, ws.vb);
    else
      k_parse_lines<false><<<std::min(g, blocks_for(nlines, 256)), 256, 0, st>>>(
          L, nlines, ws.kind, ws.err, ws.va, ws.vb);
    CK_LAUNCH();
  }
  tr.mark("tokens");
  u32 np = 0;
  if (dimacs && nlines) {
    k_kind_flags<<<std::min(g, blocks_for(nlines, 256)), 256, 0, st>>>(ws.kind, nlines,
                                                                       kLProblem, ws.flags);
    CK_LAUNCH();
    compact_u8(ws.flags, nlines, PosOut{ws.plist}, ws.scan, ws.words + 2, st);
    CK(cudaMemcpyAsync(&np, ws.words + 2, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    k_arc_check<<<std::min(g, blocks_for(nlines, 256)), 256, 0, st>>>(ws.kind, ws.err, ws.va,
                                                                      ws.vb, nlines, ws.plist, np);
    CK_LAUNCH();
  }
  if (nlines) {
    k_first_error<<<std::min(g, blocks_for(nlines, 256)), 256, 0, st>>>(ws.err, nlines,
                                                                        ws.words + 0);
    CK_LAUNCH();
  }
  u32 first[2];
  CK(cudaMemcpyAsync(first, ws.words, sizeof first, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (first[0] != 0xFFFFFFFFu) {
    uint8_t code = 0;
    CK(cudaMemcpy(&code, ws.err + first[0], 1, cudaMemcpyDeviceToHost));
    u32 sb[2] = {0, static_cast<u32>(len)};
    if (first[0] > 0) CK(cudaMemcpy(&sb[0], ws.nlpos + first[0] - 1, 4, cudaMemcpyDeviceToHost));
    if (first[0] < nnl_host) CK(cudaMemcpy(&sb[1], ws.nlpos + first[0], 4, cudaMemcpyDeviceToHost));
    const u64 s = first[0] > 0 ? u64(sb[0]) + 1 : 0;
    parse_error(text, s, sb[1], first[0], code, dimacs);
  }
  if (dimacs && np == 0) throw Error(ETTG_EPARSE, "missing DIMACS problem line");
  tr.mark("errors");

  // ---- normalise: n, self-loops, first occurrence of each unordered pair ----
  unsigned long long cnt[4] = {0, 0, 0, 0};
  u32 C = 0;
  if (nlines) {
    k_edge_candidates<<<std::min(g, blocks_for(nlines, 256)), 256, 0, st>>>(
        ws.kind, ws.va, ws.vb, nlines, dimacs, ws.flags, ws.counters);
    CK_LAUNCH();
    CK(cudaMemcpyAsync(cnt, ws.counters, sizeof cnt, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (cnt[2]) throw Error(ETTG_ERANGE, "node id >= 2^32: outside the device parser's id range");
    compact_u8(ws.flags, nlines,
               CandOut{ws.va, ws.vb, dimacs ? 1 : 0, ws.kmin, ws.kmax, ws.iota}, ws.scan,
               ws.words + 3, st);
    CK(cudaMemcpyAsync(&C, ws.words + 3, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  tr.mark("candidates");
  u32 m = 0;
  if (C) {
    const u64 nmax = cnt[0];
    const int bits = bits_for(static_cast<u32>(std::min<u64>(nmax ? nmax - 1 : 0, 0xFFFFFFFFull)));
    sort_pairs(ws.kmax, ws.iota, ws.k1, ws.v1, C, bits, ws.sort, st);
    k_gather_keys<<<std::min(g, blocks_for(C, 256)), 256, 0, st>>>(ws.kmin, ws.v1, C, ws.k1);
    CK_LAUNCH();
    sort_pairs(ws.k1, ws.v1, ws.k2, ws.v2, C, bits, ws.sort, st);
    k_first_occurrence<<<std::min(g, blocks_for(C, 256)), 256, 0, st>>>(ws.kmin, ws.kmax, ws.v2,
                                                                        C, ws.keep);
    CK_LAUNCH();
    compact_u8(ws.keep, C, EdgeOut{ws.kmin, ws.kmax, C, ws.edges}, ws.scan, ws.words + 4, st);
    CK(cudaMemcpyAsync(&m, ws.words + 4, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  tr.mark("dedup");
  *n_out = static_cast<int64_t>(cnt[0]);
  *m_out = m;
  if (stats) {
    stats->self_loops_removed = static_cast<int64_t>(cnt[1]);
    stats->duplicates_removed = static_cast<int64_t>(C) - m;
  }
  if (static_cast<u64>(cap) < m) throw Error(ETTG_ERANGE, "edge buffer too small (m returned)");
  if (m) staged_d2h_widen_pairs(edges_out, ws.edges, m, device, st);
  tr.mark("d2h");
}

}  // namespace
}  // namespace ettg

using namespace ettg;

extern "C" {

int ettg_parse_edge_list(const char* text, int64_t len, int device, int64_t* edges, int64_t cap,
                         int64_t* n, int64_t* m, ettg_parse_stats* stats) {
  return guard([&] {
    DeviceScope ds(device);
    run_parse(text, len, false, device, edges, cap, n, m, stats);
  });
}

int ettg_parse_dimacs_gr(const char* text, int64_t len, int device, int64_t* edges, int64_t cap,
                         int64_t* n, int64_t* m, ettg_parse_stats* stats) {
  return guard([&] {
    DeviceScope ds(device);
    run_parse(text, len, true, device, edges, cap, n, m, stats);
  });
}

}  // extern "C"
