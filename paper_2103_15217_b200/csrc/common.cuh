// Shared device helpers for the sm_100a Euler-tour pipeline.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>

namespace ettg {

using u32 = uint32_t;
using u64 = uint64_t;
using i64 = int64_t;

constexpr u32 kNone = 0xFFFFFFFFu;
constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs (queried at run time too)

// ---- error plumbing (host) -----------------------------------------------
// Exceptions are caught at the C-ABI boundary (capi.cu) and turned into
// ETTG_* codes; they never cross extern "C".
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file,
                       int line) {
  if (e != cudaSuccess) {
    char buf[512];
    snprintf(buf, sizeof buf, "%s failed at %s:%d: %s", what, file, line,
             cudaGetErrorString(e));
    throw Error(e == cudaErrorMemoryAllocation ? 4 : 3, buf);
  }
}
#define CK(x) ::ettg::cuda_check((x), #x, __FILE__, __LINE__)
#define CK_LAUNCH() ::ettg::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

inline unsigned blocks_for(u64 n, unsigned threads, unsigned cap = 148u * 64u) {
  u64 b = (n + threads - 1) / threads;
  if (b == 0) b = 1;
  return b > cap ? cap : static_cast<unsigned>(b);
}

// ---- bit helpers (device) -------------------------------------------------
__device__ __forceinline__ int hb32(u32 x) { return 31 - __clz(x); }  // x != 0
__device__ __forceinline__ int tz32(u32 x) { return __ffs(x) - 1; }   // x != 0

__device__ __forceinline__ u32 lanemask_lt() {
  u32 m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Read-only gathers of index records (one 32-B sector each).  L1-allocating
// on purpose: on B200 random 16-B gathers run 1.6x faster than with
// L1::no_allocate / .cg (profiles/r1_gather_micro.md).
__device__ __forceinline__ uint4 ldg_rec(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ u32 ldg_u32(const u32* p) {
  u32 r;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldg_rec(const uint2* p) {
  uint2 r;
  asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
// 6-B records {inlabel:24, ascendant:24}, five per 32-B sector (bytes 6k of
// sector v / 5, k = v % 5; 2 bytes of padding): one 256-bit load
// (LDG.E.256 on sm_100a) reads a whole sector, so a record never costs a
// second load or sector.
constexpr u32 kRec6PerSector = 5;
__host__ __device__ __forceinline__ u64 rec6_bytes(u64 n) {
  return (n + kRec6PerSector - 1) / kRec6PerSector * 32;
}
struct Sector32 {
  u32 w[8];
};
// Not volatile: the two endpoint gathers of a query must be free to issue
// back to back (a volatile asm pinned them in order with one register set).
__device__ __forceinline__ Sector32 ldg_sector(const uint32_t* p) {
  Sector32 r;
  asm("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
        "=r"(r.w[6]), "=r"(r.w[7])
      : "l"(p));
  return r;
}
// L2 eviction-priority variants of the index gathers: the policy word comes
// from createpolicy once per thread; evict_last keeps the gathered table's
// lines ahead of the streamed pairs and answers (which load/store with .cs).
__device__ __forceinline__ u64 l2_policy_evict_last() {
  u64 p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ Sector32 ldg_sector_l2(const uint32_t* p, u64 pol) {
  Sector32 r;
  asm("ld.global.nc.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
      : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
        "=r"(r.w[6]), "=r"(r.w[7])
      : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ Sector32 ldg_sector_l2_na(const uint32_t* p, u64 pol) {
  Sector32 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
      : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
        "=r"(r.w[6]), "=r"(r.w[7])
      : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ u32 ldg_u32_l2(const u32* p, u64 pol) {
  u32 r;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ u32 ldg_u32_l2_na(const u32* p, u64 pol) {  // L1::no_allocate too
  u32 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(r)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint2 ldg_rec_l2(const uint2* p, u64 pol) {
  uint2 r;
  asm volatile("ld.global.nc.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ u32 rec6_sector(u32 v) { return __umulhi(v, 0xCCCCCCCDu) >> 2; }
// record k = v - 5 * sector starts at u16 3k: words (w[3k/2], w[3k/2 + 1]),
// shifted right by 16 bits when k is odd
__device__ __forceinline__ uint2 rec6_extract(const Sector32& x, u32 k) {
  const u32 p = k == 0 ? x.w[0] : k == 1 ? x.w[1] : k == 2 ? x.w[3] : k == 3 ? x.w[4] : x.w[6];
  const u32 r = k == 0 ? x.w[1] : k == 1 ? x.w[2] : k == 2 ? x.w[4] : k == 3 ? x.w[5] : x.w[7];
  const u64 rec = ((static_cast<u64>(r) << 32) | p) >> (16 * (k & 1));
  return make_uint2(static_cast<u32>(rec) & 0xFFFFFFu, static_cast<u32>(rec >> 24) & 0xFFFFFFu);
}
// Both endpoint records of a query: the two sector loads issue before either
// is unpacked.
__device__ __forceinline__ void ldg_rec6_pair(const uint32_t* base, u32 x, u32 y, uint2& A,
                                              uint2& B) {
  const u32 sx = rec6_sector(x), sy = rec6_sector(y);
  const Sector32 a = ldg_sector(base + 8 * static_cast<u64>(sx));
  const Sector32 b = ldg_sector(base + 8 * static_cast<u64>(sy));
  A = rec6_extract(a, x - 5 * sx);
  B = rec6_extract(b, y - 5 * sy);
}
template <bool kNoAlloc = false>
__device__ __forceinline__ void ldg_rec6_pair_l2(const uint32_t* base, u32 x, u32 y, uint2& A,
                                                 uint2& B, u64 pol) {
  const u32 sx = rec6_sector(x), sy = rec6_sector(y);
  const Sector32 a = kNoAlloc ? ldg_sector_l2_na(base + 8 * static_cast<u64>(sx), pol)
                              : ldg_sector_l2(base + 8 * static_cast<u64>(sx), pol);
  const Sector32 b = kNoAlloc ? ldg_sector_l2_na(base + 8 * static_cast<u64>(sy), pol)
                              : ldg_sector_l2(base + 8 * static_cast<u64>(sy), pol);
  A = rec6_extract(a, x - 5 * sx);
  B = rec6_extract(b, y - 5 * sy);
}
// 9-B records {inlabel:24, ascendant:24, level:24}, three per 32-B sector
// (bits 72k of sector v / 3; 5 bytes of padding), one 256-bit load each.
constexpr u32 kRec9PerSector = 3;
__host__ __device__ __forceinline__ u64 rec9_bytes(u64 n) {
  return (n + kRec9PerSector - 1) / kRec9PerSector * 32;
}
__device__ __forceinline__ u32 rec9_sector(u32 v) { return __umulhi(v, 0xAAAAAAABu) >> 1; }
__device__ __forceinline__ uint4 rec9_extract(const Sector32& x, u32 k) {
  // record k starts at bit 72k = word 2k, bit 8k
  const u32 v0 = k == 0 ? x.w[0] : k == 1 ? x.w[2] : x.w[4];
  const u32 v1 = k == 0 ? x.w[1] : k == 1 ? x.w[3] : x.w[5];
  const u32 v2 = k == 0 ? x.w[2] : k == 1 ? x.w[4] : x.w[6];
  const u32 sh = 8 * k;
  const u64 a = (static_cast<u64>(v1) << 32) | v0, b = (static_cast<u64>(v2) << 32) | v1;
  return make_uint4(static_cast<u32>(a >> sh) & 0xFFFFFFu,
                    static_cast<u32>(a >> (sh + 24)) & 0xFFFFFFu,
                    static_cast<u32>(b >> (sh + 16)) & 0xFFFFFFu, 0u);
}
// Streaming loads/stores (read once / write once).
__device__ __forceinline__ uint2 ld_stream(const uint2* p) {
  uint2 r;
  asm volatile("ld.global.cs.v2.u32 {%0,%1}, [%2];"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(u32* p, u32 v) {
  asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v));
}

// Device-scope acquire/release for look-back status words.
__device__ __forceinline__ u64 ld_acquire(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(u64* p, u64 v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u32 ld_volatile_u32(const u32* p) {
  u32 v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// One lane, one bit (a RED.OR: nothing waits on it).
__device__ __forceinline__ void set_bit(u32* words, u64 i) {
  atomicOr(words + (i >> 5), 1u << (i & 31));
}
__device__ __forceinline__ bool test_bit(const u32* words, u64 i) {
  return (__ldg(words + (i >> 5)) >> (i & 31)) & 1u;
}

// 32-bit avalanche (murmur3 finaliser) used for splitter sampling.
__device__ __forceinline__ u32 mix32(u32 x) {
  x ^= x >> 16;
  x *= 0x85ebca6bu;
  x ^= x >> 13;
  x *= 0xc2b2ae35u;
  x ^= x >> 16;
  return x;
}

// ---- workspace carving -----------------------------------------------------
// Pipelines lay out their scratch with a Carver twice: once with base ==
// nullptr to measure, once on the leased arena to hand out pointers.
struct Carver {
  char* base = nullptr;
  size_t off = 0;
  template <class T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
};

// Grow-only per-device scratch arena (capi.cu).  A Lease serialises users of
// the arena across host threads and orders reuse across streams.
class Lease {
 public:
  Lease(int device, cudaStream_t stream, size_t bytes);
  ~Lease();
  char* base() const { return base_; }
  Lease(const Lease&) = delete;
  Lease& operator=(const Lease&) = delete;

 private:
  int device_;
  cudaStream_t stream_;
  char* base_;
};

int sm_count(int device);

// Pageable host buffers <-> device through per-device pinned staging (capi.cu):
// host threads (OpenMP) fill / drain one pinned chunk while the copy engine
// moves the other.  A plain cudaMemcpy from pageable memory runs ~10 GB/s
// H2D and, into freshly allocated memory, ~4 GB/s D2H (single-threaded page
// faults); the staged paths run near the link rate.  Both synchronise `st`.
void staged_h2d(void* d_dst, const void* h_src, size_t bytes, int device, cudaStream_t st);
// staged_h2d that also counts the bytes equal to `c` (the host threads read
// every byte while filling the stage anyway).
size_t staged_h2d_count(void* d_dst, const void* h_src, size_t bytes, char c, int device,
                        cudaStream_t st);
// D2H of `count` u32 pairs, widened to int64 pairs into h_dst (the reference's
// i64 ids) by the host threads as the chunks land.
void staged_d2h_widen_pairs(int64_t* h_dst, const uint2* d_src, size_t count, int device,
                            cudaStream_t st);
// The device's kStageBufs pinned staging buffers, held for a custom pipeline.
constexpr int kStageBufs = 3;
class StageLease {
 public:
  explicit StageLease(int device);
  ~StageLease();
  char* buf(int k) const;
  cudaEvent_t done(int k) const;
  static size_t bytes();  // per buffer
  StageLease(const StageLease&) = delete;
  StageLease& operator=(const StageLease&) = delete;

 private:
  void* s_;
};
void par_copy(char* dst, const char* src, size_t n);  // host threads
int host_thread_count();   // threads of the host-side staging passes (this thread)
int host_thread_budget();  // all of them (ETTG_HOST_THREADS, else <= 16 cores)
class ScopedHostThreads {  // caps host_thread_count() on this thread
 public:
  explicit ScopedHostThreads(int t);
  ~ScopedHostThreads();

 private:
  int prev_;
};
// Host int64 ids cross the link narrowed to u32 (default; ETTG_NARROW=0
// sends pinned int64 buffers as they are, for A/B runs).
bool narrow_enabled();
// D2H of `count` u32 values widened to int64 (0xFFFFFFFF -> -1, the
// reference's kNone) by the host threads as the pinned chunks land.
void staged_d2h_widen_u32(int64_t* h_dst, const uint32_t* d_src, size_t count, int device,
                          cudaStream_t st);
// Raw staged D2H into a pageable host buffer (host threads drain the chunks).
void staged_d2h(void* h_dst, const void* d_src, size_t bytes, int device, cudaStream_t st);
// H2D of `count` int64 values narrowed to u32 by the host threads while they
// fill the pinned stage (the link then carries 4 B per id instead of 8).
// Values must lie in [0, bound), or be -1 when allow_none (-> 0xFFFFFFFF);
// the others are stored as 0xFFFFFFFF and counted in the return value (the
// caller raises its own error).  on_chunk(lo, n), if given, runs after chunk
// [lo, lo + n) is enqueued on `st` (to enqueue its consumers).  Synchronises st.
// raw_frac > 0 (pinned h_src only): that fraction of the chunks crosses the
// link as int64 and is narrowed on the device instead, trading link bytes
// for host memory bandwidth (both bind on the B200 host).
u64 staged_h2d_narrow_u32(uint32_t* d_dst, const int64_t* h_src, size_t count, uint64_t bound,
                          bool allow_none, int device, cudaStream_t st,
                          const std::function<void(size_t, size_t)>& on_chunk = {},
                          double raw_frac = 0);
// ETTG_RAW_FRAC if set (0..1, or "auto"), else dflt; and whether chunk c of
// a hybrid upload goes raw (an even spread: floor((c+1) f) > floor(c f)).
// kRawAdaptive: a chunk goes raw whenever the link has drained everything
// enqueued before it (the host narrowing is then the bottleneck), so the
// split follows the host's memory bandwidth, which varies from box to box
// (4 GB narrowed in 33 ms on one B200 host, 72 ms on another).
constexpr double kRawAdaptive = -1.0;
double raw_fraction(double dflt);
bool chunk_is_raw(u64 c, double frac);
struct RawPolicy {
  double frac;       // kRawAdaptive, or a static share
  cudaEvent_t last;  // the last enqueued upload
  bool raw_next(u64 c) const;
};
// D2H of a bit-packed 0/1 mask (`count` bits, LSB first per u32 word) into
// `count` mask bytes, expanded by the host threads as the chunks land: 1/8
// of the bytes over the link.
void staged_d2h_expand_bits(uint8_t* h_dst, const uint32_t* d_bits, size_t count, int device,
                            cudaStream_t st);
// Page-locked (cudaHostAlloc / cudaHostRegister / torch pin_memory) host memory?
// Throws ETTG_EINVAL for a device pointer (host-buffer entry points).
bool is_pinned(const void* p);
// is_pinned for its check only: host-buffer entry points call it on every
// caller buffer, whatever its size or the path it takes.
void check_host_ptr(const void* p);
// hostcopy.cpp: stage -> caller memory with streaming stores
void host_widen_u32(int64_t* dst, const uint32_t* src, size_t n, bool none_to_minus1, int threads);
void host_expand_bits(uint8_t* dst, const uint32_t* in, size_t w0, size_t w1, size_t count,
                      int threads);
// Host <-> device copies of caller buffers: async when the host side is
// pinned, staged (and synchronous) when it is pageable.
void copy_h2d(void* d_dst, const void* h_src, size_t bytes, int device, cudaStream_t st);
void copy_d2h(void* h_dst, const void* d_src, size_t bytes, int device, cudaStream_t st);

// Copy `count` words device->host on `stream` and wait (used for counters
// and error flags; a handful of bytes).
inline void read_back(void* host, const void* dev, size_t bytes,
                      cudaStream_t stream) {
  CK(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, stream));
  CK(cudaStreamSynchronize(stream));
}

}  // namespace ettg
