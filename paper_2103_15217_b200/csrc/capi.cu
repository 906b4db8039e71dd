// C-ABI plumbing: error state, device scope, scratch arena, primitives.
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
    ws.carve(c, kk);
    u32* pred = c.take<u32>(kk);
    Lease lease(device, st, c.off);
    c = Carver{lease.base()};
    ws.carve(c, kk);
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
