// Host-side widening / expansion out of the pinned stage into caller memory
// with non-temporal (streaming) stores.
//
// A plain store to a caller buffer that is not in cache first reads the line
// (read-for-ownership), so writing 128 MB of int64 answers cost 256 MB of
// host DRAM traffic; the e2e paths are bound by host DRAM bandwidth
// (profiles/r2_e2e.md), so the streaming stores (AVX2 `vmovntdq`, one
// `sfence` per thread) take that read away.  Unaligned heads and tails, and
// hosts without AVX2, use plain stores.
#include <immintrin.h>
#include <omp.h>

#include <cstddef>
#include <cstdint>
#include <algorithm>
#include <cstring>

namespace ettg {

namespace {

bool have_avx2() {
  static const bool v = __builtin_cpu_supports("avx2");
  return v;
}

__attribute__((target("avx2"))) void widen_nt(int64_t* dst, const uint32_t* src, size_t n,
                                              bool none_to_minus1) {
  size_t i = 0;
  // scalar head up to 32-B alignment of dst
  while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31)) {
    dst[i] = (none_to_minus1 && src[i] == 0xFFFFFFFFu) ? int64_t(-1) : int64_t(src[i]);
    ++i;
  }
  const __m256i none = _mm256_set1_epi64x(0xFFFFFFFFll);
  for (; i + 4 <= n; i += 4) {
    const __m128i v = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    __m256i w = _mm256_cvtepu32_epi64(v);
    if (none_to_minus1) w = _mm256_or_si256(w, _mm256_slli_epi64(_mm256_cmpeq_epi64(w, none), 32));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), w);
  }
  for (; i < n; ++i)
    dst[i] = (none_to_minus1 && src[i] == 0xFFFFFFFFu) ? int64_t(-1) : int64_t(src[i]);
  _mm_sfence();
}

// words [lo, hi) of the mask; in[w - w0] holds word w
__attribute__((target("avx2"))) void expand_nt(uint8_t* dst, const uint32_t* in, size_t w0,
                                               size_t lo, size_t hi, size_t count,
                                               const uint64_t* table) {
  for (size_t w = lo; w < hi; ++w) {
    const size_t base = w * 32;
    const uint32_t x = in[w - w0];
    if (base + 32 <= count) {
      const __m256i q = _mm256_set_epi64x(static_cast<long long>(table[x >> 24]),
                                          static_cast<long long>(table[(x >> 16) & 0xFF]),
                                          static_cast<long long>(table[(x >> 8) & 0xFF]),
                                          static_cast<long long>(table[x & 0xFF]));
      if ((reinterpret_cast<uintptr_t>(dst + base) & 31) == 0)
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + base), q);
      else
        _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + base), q);
    } else {
      for (size_t i = base; i < count; ++i) dst[i] = (x >> (i - base)) & 1;
    }
  }
  _mm_sfence();
}

}  // namespace

// dst[i] = src[i] widened to int64 (0xFFFFFFFF -> -1 when none_to_minus1),
// split over `threads` host threads.
void host_widen_u32(int64_t* dst, const uint32_t* src, size_t n, bool none_to_minus1,
                    int threads) {
  if (n == 0) return;
  const bool nt = have_avx2();
  const int t = n > 65536 ? threads : 1;
#pragma omp parallel num_threads(t)
  {
    const int nt_ = omp_get_num_threads(), me = omp_get_thread_num();
    // thread slices aligned to 4 elements (32 B of output)
    const size_t per = ((n + nt_ - 1) / nt_ + 3) & ~size_t(3);
    const size_t lo = std::min(n, per * me), hi = std::min(n, lo + per);
    if (nt) {
      widen_nt(dst + lo, src + lo, hi - lo, none_to_minus1);
    } else {
      for (size_t i = lo; i < hi; ++i)
        dst[i] = (none_to_minus1 && src[i] == 0xFFFFFFFFu) ? int64_t(-1) : int64_t(src[i]);
    }
  }
}

// Mask bytes (0/1) for bit words [w0, w1), in[w - w0] holding word w (bit i
// of word w is mask byte 32 w + i); count = total mask bytes.
void host_expand_bits(uint8_t* dst, const uint32_t* in, size_t w0, size_t w1, size_t count,
                      int threads) {
  static const auto* table = [] {
    static uint64_t t[256];
    for (int b = 0; b < 256; ++b) {
      t[b] = 0;
      for (int i = 0; i < 8; ++i) t[b] |= static_cast<uint64_t>((b >> i) & 1) << (8 * i);
    }
    return t;
  }();
  if (w1 <= w0) return;
  const bool nt = have_avx2();
  const size_t n = w1 - w0;
  const int t = n > 16384 ? threads : 1;
#pragma omp parallel num_threads(t)
  {
    const int nt_ = omp_get_num_threads(), me = omp_get_thread_num();
    const size_t per = (n + nt_ - 1) / nt_;
    const size_t lo = w0 + std::min(n, per * me), hi = w0 + std::min(n, per * me + per);
    if (nt) {
      expand_nt(dst, in, w0, lo, hi, count, table);
    } else {
      for (size_t w = lo; w < hi; ++w) {
        const size_t base = w * 32;
        const uint32_t x = in[w - w0];
        if (base + 32 <= count) {
          const uint64_t q[4] = {table[x & 0xFF], table[(x >> 8) & 0xFF],
                                 table[(x >> 16) & 0xFF], table[x >> 24]};
          std::memcpy(dst + base, q, 32);
        } else {
          for (size_t i = base; i < count; ++i) dst[i] = (x >> (i - base)) & 1;
        }
      }
    }
  }
}

}  // namespace ettg
