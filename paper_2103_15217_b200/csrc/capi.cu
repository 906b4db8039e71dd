// C-ABI plumbing: error state, device scope, scratch arena, primitives.
#include <omp.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "api_internal.cuh"
#include "common.cuh"
#include "listrank.cuh"
#include "scan.cuh"
#include "sort.cuh"

namespace ettg {

namespace {
thread_local std::string g_last_error;

struct Arena {
  std::mutex mu;
  char* base = nullptr;
  size_t cap = 0;
  cudaEvent_t last = nullptr;  // recorded after the last user's work
};

std::mutex g_arenas_mu;
std::map<int, std::unique_ptr<Arena>> g_arenas;

Arena& arena_for(int device) {
  std::lock_guard<std::mutex> lk(g_arenas_mu);
  auto& a = g_arenas[device];
  if (!a) a = std::make_unique<Arena>();
  return *a;
}
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }

DeviceScope::DeviceScope(int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw Error(ETTG_ECUDA, "no CUDA device available (the pipeline has no CPU fallback)");
  }
  if (device < 0 || device >= count) throw Error(ETTG_EINVAL, "device ordinal out of range");
  CK(cudaGetDevice(&prev_));
  if (prev_ != device) {
    CK(cudaSetDevice(device));
    changed_ = true;
  }
}

DeviceScope::~DeviceScope() {
  if (changed_) cudaSetDevice(prev_);
}

int sm_count(int device) {
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(device);
  if (it != cache.end()) return it->second;
  int v = kSMs;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) v = kSMs;
  cache[device] = v;
  return v;
}

Lease::Lease(int device, cudaStream_t stream, size_t bytes) : device_(device), stream_(stream) {
  Arena& a = arena_for(device);
  a.mu.lock();
  try {
    if (!a.last) CK(cudaEventCreateWithFlags(&a.last, cudaEventDisableTiming));
    if (a.cap < bytes) {
      if (a.base) {
        CK(cudaEventSynchronize(a.last));
        CK(cudaFree(a.base));
        a.base = nullptr;
        a.cap = 0;
      }
      size_t want = bytes + bytes / 8 + (size_t(1) << 20);
      CK(cudaMalloc(&a.base, want));
      a.cap = want;
    } else {
      CK(cudaStreamWaitEvent(stream, a.last, 0));  // previous user on another stream
    }
    base_ = a.base;
  } catch (...) {
    a.mu.unlock();
    throw;
  }
}

Lease::~Lease() {
  Arena& a = arena_for(device_);
  cudaEventRecord(a.last, stream_);
  a.mu.unlock();
}

// ---- pinned staging --------------------------------------------------------
namespace {
constexpr size_t kStageChunk = size_t(16) << 20;
// Three 16-MB buffers: host threads fill one while the copy engine drains
// another (tools/stage_micro.cu on the B200 host, 4 GB of int64 ids narrowed
// and sent: 2 x 16 MB 45.2 ms, 3 x 16 MB 39.9 ms = the 54 GB/s link, 4 x 16 MB
// 46.1 ms).
struct Stage {
  std::mutex mu;
  char* buf[kStageBufs] = {nullptr, nullptr, nullptr};  // pinned, kStageChunk each
  cudaEvent_t done[kStageBufs] = {nullptr, nullptr, nullptr};
};
std::mutex g_stage_mu;
std::map<int, std::unique_ptr<Stage>> g_stages;
Stage& stage_for(int device) {
  std::lock_guard<std::mutex> lk(g_stage_mu);
  auto& s = g_stages[device];
  if (!s) s = std::make_unique<Stage>();
  return *s;
}
// Host threads for staging copies: ETTG_HOST_THREADS, else up to 16 of the
// visible cores (independent of OMP_NUM_THREADS, which launchers such as
// torchrun set to 1 per rank).
int host_threads() {
  static const int t = [] {
    if (const char* e = std::getenv("ETTG_HOST_THREADS")) return std::max(1, std::atoi(e));
    return std::max(1, std::min(16, omp_get_num_procs()));
  }();
  return t;
}
// Per calling thread: a multi-GPU call splits the host threads between the
// replicas it drives (ScopedHostThreads).
thread_local int t_host_threads = 0;
}  // namespace
int host_thread_count();
namespace {
void stage_init(Stage& s) {
  if (s.buf[0]) return;
  for (int i = 0; i < kStageBufs; ++i) {
    CK(cudaHostAlloc(reinterpret_cast<void**>(&s.buf[i]), kStageChunk, cudaHostAllocPortable));
    CK(cudaEventCreateWithFlags(&s.done[i], cudaEventDisableTiming));
  }
}
void par_copy_impl(char* dst, const char* src, size_t n) {
  const size_t kPiece = size_t(1) << 20;
  const long pieces = static_cast<long>((n + kPiece - 1) / kPiece);
#pragma omp parallel for schedule(static) num_threads(host_thread_count()) if (pieces > 1)
  for (long i = 0; i < pieces; ++i) {
    const size_t o = static_cast<size_t>(i) * kPiece;
    std::memcpy(dst + o, src + o, std::min(kPiece, n - o));
  }
}
}  // namespace

void par_copy(char* dst, const char* src, size_t n) { par_copy_impl(dst, src, n); }
int host_thread_count() { return t_host_threads > 0 ? t_host_threads : host_threads(); }
int host_thread_budget() { return host_threads(); }
ScopedHostThreads::ScopedHostThreads(int t) : prev_(t_host_threads) { t_host_threads = t; }
ScopedHostThreads::~ScopedHostThreads() { t_host_threads = prev_; }
bool narrow_enabled() {
  const char* e = std::getenv("ETTG_NARROW");  // per call: A/B runs flip it
  return !e || std::atoi(e) != 0;
}

StageLease::StageLease(int device) : s_(&stage_for(device)) {
  Stage& s = *static_cast<Stage*>(s_);
  s.mu.lock();
  try {
    stage_init(s);
  } catch (...) {
    s.mu.unlock();
    throw;
  }
}
StageLease::~StageLease() { static_cast<Stage*>(s_)->mu.unlock(); }
char* StageLease::buf(int k) const { return static_cast<Stage*>(s_)->buf[k]; }
cudaEvent_t StageLease::done(int k) const { return static_cast<Stage*>(s_)->done[k]; }
size_t StageLease::bytes() { return kStageChunk; }

void check_host_ptr(const void* p);

void staged_h2d(void* d_dst, const void* h_src, size_t bytes, int device, cudaStream_t st) {
  check_host_ptr(h_src);  // a device pointer here would be written by host threads
  Stage& s = stage_for(device);
  std::lock_guard<std::mutex> lk(s.mu);
  stage_init(s);
  const char* src = static_cast<const char*>(h_src);
  char* dst = static_cast<char*>(d_dst);
  int k = 0;
  for (size_t o = 0; o < bytes; o += kStageChunk, k = (k + 1) % kStageBufs) {
    const size_t n = std::min(kStageChunk, bytes - o);
    CK(cudaEventSynchronize(s.done[k]));  // the copy that last read this buffer
    par_copy(s.buf[k], src + o, n);
    CK(cudaMemcpyAsync(dst + o, s.buf[k], n, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(s.done[k], st));
  }
  CK(cudaStreamSynchronize(st));
}

size_t staged_h2d_count(void* d_dst, const void* h_src, size_t bytes, char c, int device,
                        cudaStream_t st) {
  check_host_ptr(h_src);
  Stage& s = stage_for(device);
  std::lock_guard<std::mutex> lk(s.mu);
  stage_init(s);
  const char* src = static_cast<const char*>(h_src);
  char* dst = static_cast<char*>(d_dst);
  size_t total = 0;
  int k = 0;
  for (size_t o = 0; o < bytes; o += kStageChunk, k = (k + 1) % kStageBufs) {
    const size_t n = std::min(kStageChunk, bytes - o);
    CK(cudaEventSynchronize(s.done[k]));
    const size_t kPiece = size_t(1) << 18;
    const long pieces = static_cast<long>((n + kPiece - 1) / kPiece);
    char* out = s.buf[k];
    const char* in = src + o;
    size_t cnt = 0;
#pragma omp parallel for schedule(static) num_threads(host_thread_count()) reduction(+ : cnt) \
    if (pieces > 1)
    for (long i = 0; i < pieces; ++i) {
      const size_t a = static_cast<size_t>(i) * kPiece, len = std::min(kPiece, n - a);
      std::memcpy(out + a, in + a, len);
      size_t m = 0;
      for (size_t j = 0; j < len; ++j) m += out[a + j] == c;  // from the just-written (cached) copy
      cnt += m;
    }
    total += cnt;
    CK(cudaMemcpyAsync(dst + o, s.buf[k], n, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(s.done[k], st));
  }
  CK(cudaStreamSynchronize(st));
  return total;
}

void staged_d2h_widen_pairs(int64_t* h_dst, const uint2* d_src, size_t count, int device,
                            cudaStream_t st) {
  check_host_ptr(h_dst);  // a device pointer here would be written by host threads
  Stage& s = stage_for(device);
  std::lock_guard<std::mutex> lk(s.mu);
  stage_init(s);
  const size_t per = kStageChunk / sizeof(uint2);
  const size_t chunks = (count + per - 1) / per;
  auto issue = [&](size_t c) {
    const size_t lo = c * per, n = std::min(per, count - lo);
    CK(cudaMemcpyAsync(s.buf[c & 1], d_src + lo, n * sizeof(uint2), cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(s.done[c & 1], st));
  };
  if (chunks) issue(0);
  for (size_t c = 0; c < chunks; ++c) {
    if (c + 1 < chunks) issue(c + 1);  // lands while chunk c is widened
    CK(cudaEventSynchronize(s.done[c & 1]));
    const size_t lo = c * per, n = std::min(per, count - lo);
    // pairs are 2n consecutive u32 ids: zero-extended with streaming stores
    host_widen_u32(h_dst + 2 * lo, reinterpret_cast<const uint32_t*>(s.buf[c & 1]), 2 * n, false,
                   host_thread_count());
  }
}

void staged_d2h(void* h_dst, const void* d_src, size_t bytes, int device, cudaStream_t st) {
  check_host_ptr(h_dst);  // a device pointer here would be written by host threads
  Stage& s = stage_for(device);
  std::lock_guard<std::mutex> lk(s.mu);
  stage_init(s);
  const size_t chunks = (bytes + kStageChunk - 1) / kStageChunk;
  const char* src = static_cast<const char*>(d_src);
  char* dst = static_cast<char*>(h_dst);
  auto issue = [&](size_t c) {
    const size_t o = c * kStageChunk, n = std::min(kStageChunk, bytes - o);
    CK(cudaMemcpyAsync(s.buf[c & 1], src + o, n, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(s.done[c & 1], st));
  };
  if (chunks) issue(0);
  for (size_t c = 0; c < chunks; ++c) {
    if (c + 1 < chunks) issue(c + 1);
    CK(cudaEventSynchronize(s.done[c & 1]));
    const size_t o = c * kStageChunk, n = std::min(kStageChunk, bytes - o);
    par_copy(dst + o, s.buf[c & 1], n);
  }
}

void staged_d2h_widen_u32(int64_t* h_dst, const uint32_t* d_src, size_t count, int device,
                          cudaStream_t st) {
  check_host_ptr(h_dst);  // a device pointer here would be written by host threads
  Stage& s = stage_for(device);
  std::lock_guard<std::mutex> lk(s.mu);
  stage_init(s);
  const size_t per = kStageChunk / sizeof(uint32_t);
  const size_t chunks = (count + per - 1) / per;
  auto issue = [&](size_t c) {
    const size_t lo = c * per, n = std::min(per, count - lo);
    CK(cudaMemcpyAsync(s.buf[c & 1], d_src + lo, n * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(s.done[c & 1], st));
  };
  if (chunks) issue(0);
  for (size_t c = 0; c < chunks; ++c) {
    if (c + 1 < chunks) issue(c + 1);
    CK(cudaEventSynchronize(s.done[c & 1]));
    const size_t lo = c * per, n = std::min(per, count - lo);
    const uint32_t* in = reinterpret_cast<const uint32_t*>(s.buf[c & 1]);
    host_widen_u32(h_dst + lo, in, n, true, host_thread_count());  // streaming stores
  }
}

// Device narrowing of an int64 chunk that crossed the link as is.
__global__ void k_narrow_u32(const int64_t* __restrict__ in, u64 n, uint64_t bound,
                             bool allow_none, uint32_t* __restrict__ out, u32* bad) {
  u32 b = 0;
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n;
       i += u64(gridDim.x) * blockDim.x) {
    const int64_t x = in[i];
    const bool ok = static_cast<uint64_t>(x) < bound || (allow_none && x == -1);
    b |= !ok;
    out[i] = ok ? static_cast<uint32_t>(x) : 0xFFFFFFFFu;
  }
  if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

double raw_fraction(double dflt) {
  if (const char* e = std::getenv("ETTG_RAW_FRAC")) {
    if (std::strcmp(e, "auto") == 0) return kRawAdaptive;
    return std::min(1.0, std::max(0.0, std::atof(e)));
  }
  return dflt;
}

bool chunk_is_raw(u64 c, double frac) {
  return frac > 0 && static_cast<u64>((c + 1) * frac) > static_cast<u64>(c * frac);
}

bool RawPolicy::raw_next(u64 c) const {
  if (frac == kRawAdaptive) {
    // the link has drained everything enqueued: the host is the bottleneck
    // right now, so this chunk goes as is
    return !last || cudaEventQuery(last) == cudaSuccess;
  }
  return chunk_is_raw(c, frac);
}

u64 staged_h2d_narrow_u32(uint32_t* d_dst, const int64_t* h_src, size_t count, uint64_t bound,
                          bool allow_none, int device, cudaStream_t st,
                          const std::function<void(size_t, size_t)>& on_chunk,
                          double raw_frac) {
  check_host_ptr(h_src);  // a device pointer here would be written by host threads
  if (raw_frac != 0 && !is_pinned(h_src)) raw_frac = 0;  // raw chunks need DMA-able memory
  Stage& s = stage_for(device);
  std::lock_guard<std::mutex> lk(s.mu);
  stage_init(s);
  const size_t per = kStageChunk / sizeof(uint32_t);
  // raw chunks land in one of two int64 scratch buffers (stream-ordered
  // allocations; reuse is ordered on `st`), plus a device bad-value flag
  struct Scratch {
    char* p = nullptr;
    cudaStream_t s = nullptr;
    ~Scratch() {
      if (p) cudaFreeAsync(p, s);
    }
  } sc;
  int64_t* raw[2] = {nullptr, nullptr};
  u32* dflag = nullptr;
  cudaEvent_t raw_ev[2] = {nullptr, nullptr};
  struct EvFree {
    cudaEvent_t* e;
    ~EvFree() {
      for (int i = 0; i < 2; ++i)
        if (e[i]) cudaEventDestroy(e[i]);
    }
  } ev_free{raw_ev};
  if (raw_frac != 0) {
    for (auto& e : raw_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    sc.s = st;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&sc.p), 2 * per * 8 + 256, st));
    raw[0] = reinterpret_cast<int64_t*>(sc.p);
    raw[1] = raw[0] + per;
    dflag = reinterpret_cast<u32*>(sc.p + 2 * per * 8);
    CK(cudaMemsetAsync(dflag, 0, 4, st));
  }
  const int sms = sm_count(device);
  const char* tr = std::getenv("ETTG_TRACE");
  const bool trace = tr && *tr && *tr != '0';
  double t_wait = 0, t_narrow = 0;
  const double t_start = trace ? omp_get_wtime() : 0;
  u64 bad = 0, nraw = 0;
  int k = 0, r = 0;
  u64 c = 0;
  RawPolicy pol{raw_frac, nullptr};
  for (size_t lo = 0; lo < count; lo += per, ++c) {
    const size_t n = std::min(per, count - lo);
    if (raw_frac != 0 && pol.raw_next(c)) {
      // the link carries this chunk as int64 (no host work); the device
      // narrows it -- host memory bandwidth, not the link, bounds an
      // all-narrowed upload on the B200 host (e2e)
      CK(cudaMemcpyAsync(raw[r], h_src + lo, n * 8, cudaMemcpyHostToDevice, st));
      k_narrow_u32<<<std::min<u64>((n + 255) / 256, u64(sms) * 8), 256, 0, st>>>(
          raw[r], n, bound, allow_none, d_dst + lo, dflag);
      CK(cudaGetLastError());
      CK(cudaEventRecord(raw_ev[r], st));
      pol.last = raw_ev[r];
      r ^= 1;
      ++nraw;
      if (on_chunk) on_chunk(lo, n);
      continue;
    }
    double t0 = trace ? omp_get_wtime() : 0;
    CK(cudaEventSynchronize(s.done[k]));  // the copy that last read this buffer
    if (trace) {
      const double t1 = omp_get_wtime();
      t_wait += t1 - t0;
      t0 = t1;
    }
    uint32_t* out = reinterpret_cast<uint32_t*>(s.buf[k]);
    const int64_t* in = h_src + lo;
    u64 b = 0;
#pragma omp parallel for schedule(static) num_threads(host_thread_count()) reduction(+ : b) \
    if (n > 65536)
    for (long i = 0; i < static_cast<long>(n); ++i) {
      const uint64_t v = static_cast<uint64_t>(in[i]);
      const bool ok = v < bound || (allow_none && in[i] == -1);
      b += !ok;
      out[i] = ok ? static_cast<uint32_t>(v) : 0xFFFFFFFFu;
    }
    if (trace) t_narrow += omp_get_wtime() - t0;
    bad += b;
    if (b) break;  // the caller fails the call: skip the rest
    CK(cudaMemcpyAsync(d_dst + lo, out, n * 4, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(s.done[k], st));
    pol.last = s.done[k];
    k = (k + 1) % kStageBufs;
    if (on_chunk) on_chunk(lo, n);
  }
  if (dflag) {
    u32 f = 0;
    CK(cudaMemcpyAsync(&f, dflag, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    bad += f;
  }
  CK(cudaStreamSynchronize(st));
  if (trace)
    std::fprintf(stderr,
                 "[ettg trace] h2d_narrow: %llu ids, %llu chunks, %llu raw (policy %.2f) "
                 "narrow=%.3f wait=%.3f wall=%.3f ms\n",
                 static_cast<unsigned long long>(count), static_cast<unsigned long long>(c),
                 static_cast<unsigned long long>(nraw), raw_frac, t_narrow * 1e3, t_wait * 1e3,
                 (omp_get_wtime() - t_start) * 1e3);
  return bad;
}

void staged_d2h_expand_bits(uint8_t* h_dst, const uint32_t* d_bits, size_t count, int device,
                            cudaStream_t st) {
  check_host_ptr(h_dst);  // a device pointer here would be written by host threads
  Stage& s = stage_for(device);
  std::lock_guard<std::mutex> lk(s.mu);
  stage_init(s);
  const size_t words = (count + 31) / 32;
  const size_t per = kStageChunk / 4;  // words per chunk
  const size_t chunks = (words + per - 1) / per;
  auto issue = [&](size_t c) {
    const size_t lo = c * per, n = std::min(per, words - lo);
    CK(cudaMemcpyAsync(s.buf[c & 1], d_bits + lo, n * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(s.done[c & 1], st));
  };
  if (chunks) issue(0);
  for (size_t c = 0; c < chunks; ++c) {
    if (c + 1 < chunks) issue(c + 1);
    CK(cudaEventSynchronize(s.done[c & 1]));
    const size_t lo = c * per, n = std::min(per, words - lo);
    const uint32_t* in = reinterpret_cast<const uint32_t*>(s.buf[c & 1]);
    host_expand_bits(h_dst, in, lo, lo + n, count, host_thread_count());  // streaming stores
  }
}

void check_host_ptr(const void* p) {
  if (p) (void)is_pinned(p);
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  // host-buffer entry points: a device pointer here is a caller error (the
  // _dev variants take device memory); managed memory is host-accessible
  if (a.type == cudaMemoryTypeDevice)
    throw Error(ETTG_EINVAL, "device pointer passed where a host buffer is expected");
  return a.type == cudaMemoryTypeHost;
}

void copy_h2d(void* d_dst, const void* h_src, size_t bytes, int device, cudaStream_t st) {
  if (!bytes) return;
  if (is_pinned(h_src) || bytes < (size_t(1) << 20))
    CK(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, st));
  else
    staged_h2d(d_dst, h_src, bytes, device, st);
}

void copy_d2h(void* h_dst, const void* d_src, size_t bytes, int device, cudaStream_t st) {
  if (!bytes) return;
  if (is_pinned(h_dst) || bytes < (size_t(1) << 20))
    CK(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, st));
  else
    staged_d2h(h_dst, d_src, bytes, device, st);
}


}  // namespace ettg

using namespace ettg;

extern "C" {

const char* ettg_last_error(void) { return g_last_error.c_str(); }

int ettg_version(void) { return 100; }

int ettg_device_count(int* count) {
  return guard([&] {
    if (!count) einval("null argument");
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *count = c;
  });
}

int ettg_set_l2_fetch_granularity(int device, int bytes) {
  return guard([&] {
    DeviceScope ds(device);
    CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, static_cast<size_t>(bytes)));
  });
}

int ettg_get_l2_fetch_granularity(int device, int* bytes) {
  return guard([&] {
    if (!bytes) einval("null argument");
    DeviceScope ds(device);
    size_t v = 0;
    CK(cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity));
    *bytes = static_cast<int>(v);
  });
}

int ettg_list_rank_dev(const uint32_t* d_succ, int64_t k, int64_t head, uint32_t* d_rank,
                       int device, void* stream) {
  return guard([&] {
    if (k < 0 || k >= (int64_t(1) << 32) - 1) einval("list too long");
    if (k == 0) return;
    if (!d_succ || !d_rank) einval("null argument");
    if (head < 0 || head >= k) einval("list head out of range");
    DeviceScope ds(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const u32 kk = static_cast<u32>(k);
    ListRankWs ws;
    Carver c;
    ws.carve(c, kk, true);
    u32* pred = c.take<u32>(kk);
    Lease lease(device, st, c.off);
    c = Carver{lease.base()};
    ws.carve(c, kk, true);
    pred = c.take<u32>(kk);
    CK(cudaMemcpyAsync(ws.succ0, d_succ, static_cast<u64>(kk) * 4, cudaMemcpyDeviceToDevice, st));
    const int sms = sm_count(device);
    list_rank_core(kk, static_cast<u32>(head), NoDown{}, ws, st, sms, pred);
    k_lr_rank_out<<<blocks_for(kk, 256), 256, 0, st>>>(lr0_view(ws), kk, d_rank);
    CK_LAUNCH();
    u32 err = 0;
    read_back(&err, ws.counters + LrCounters::kErr, sizeof err, st);
    if (err & kErrStructure) einval("linked list contains a cycle or does not cover all elements");
    if (err & kErrCapacity) throw Error(ETTG_EINTERNAL, "list ranking: splitter capacity exceeded");
  });
}

int ettg_exclusive_scan_dev(const uint32_t* d_in, int64_t n, uint32_t* d_out, int device,
                            void* stream) {
  return guard([&] {
    if (n < 0) einval("negative length");
    if (n == 0) return;
    if (!d_in || !d_out) einval("null argument");
    DeviceScope ds(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Carver c;
    u64* status = c.take<u64>(scan_ws_words(n));
    Lease lease(device, st, c.off);
    c = Carver{lease.base()};
    status = c.take<u64>(scan_ws_words(n));
    scan_exclusive(ArrayIn{d_in}, ArrayOut{d_out}, static_cast<u64>(n), status, nullptr, st);
  });
}

int ettg_sort_pairs_dev(const uint32_t* d_keys, const uint32_t* d_vals, int64_t n,
                        uint32_t* d_keys_out, uint32_t* d_vals_out, int device, void* stream) {
  return guard([&] {
    if (n < 0 || n >= (int64_t(1) << 32)) einval("bad length");
    if (n == 0) return;
    if (!d_keys || !d_vals || !d_keys_out || !d_vals_out) einval("null argument");
    DeviceScope ds(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    SortWs ws;
    Carver c;
    ws.carve(c, n);
    Lease lease(device, st, c.off);
    c = Carver{lease.base()};
    ws.carve(c, n);
    sort_pairs(d_keys, d_vals, d_keys_out, d_vals_out, static_cast<u32>(n), 32, ws, st);
  });
}

}  // extern "C"
