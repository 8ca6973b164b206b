// sf_host_narrow.cpp -- lossless f32 -> u16 narrowing of host spot chunks for the PCIe leg.
//
// The host pipeline (sf_capi.cu:run_shard) is bound by the H2D copy of the pixels (PCIe Gen5 x16,
// ~53 GB/s: 5.9e7 15x15 f32 fits/s).  Camera counts -- and every image the reference simulator
// emits ("non-negative integers representable exactly in 32-bit reals") -- are integers
// in [0, 65535], which 16 bits hold exactly.  For such a chunk the CPU writes the u16 values into a
// pinned buffer, half the bytes cross PCIe, and the fit kernel widens them back exactly
// (fit_kernel<..., uint16_t>, bitwise the same fit: tests/test_gpu_parity.py u16 tests).  A chunk with
// any other value (fraction, negative, -0.0, > 65535, inf, NaN) is sent as f32 unchanged, so results
// never depend on the narrowing.  AVX2 when the CPU has it (runtime check), scalar otherwise, split
// over threads.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <vector>

#include <immintrin.h>

#include "spotfit.h"

namespace {

// exactly representable as u16 with the same float value and a clear sign bit
inline bool narrow_one(float v, uint16_t& out) {
  uint32_t b;
  memcpy(&b, &v, 4);
  if (b > 0x477FFF00u) return false;  // sign set (incl. -0.0), > 65535.0f, inf, NaN
  const uint32_t u = (uint32_t)v;     // v in [0, 65535]: truncation is exact for integers
  out = (uint16_t)u;
  return (float)u == v;
}

// Every narrowing pass gives up as soon as it (or, through `stop`, another thread of the same chunk)
// meets a value that does not narrow: the chunk then goes as f32 and the rest of the pass is wasted.
constexpr size_t kCheck = 4096;  // elements between checks

bool narrow_scalar(uint16_t* dst, const float* src, size_t n, std::atomic<bool>* stop) {
  bool ok = true;
  for (size_t i = 0; i < n; ++i) {
    ok &= narrow_one(src[i], dst[i]);
    if ((i & (kCheck - 1)) == kCheck - 1 && (!ok || (stop && stop->load(std::memory_order_relaxed)))) break;
  }
  if (!ok && stop) stop->store(true, std::memory_order_relaxed);
  return ok && !(stop && stop->load(std::memory_order_relaxed));
}

#ifndef SF_HOST_NT
#define SF_HOST_NT 1  // streaming (non-temporal) stores into the pinned staging buffers
#endif
#ifndef SF_HOST_PF
#define SF_HOST_PF 256  // software prefetch distance in floats (1 KB; profiles/r02_ab_narrow_pinned.txt)
#endif

__attribute__((target("avx2"))) bool narrow_avx2(uint16_t* dst, const float* src, size_t n, std::atomic<bool>* stop) {
  const __m256i lim = _mm256_set1_epi32(0x477FFF00);
  __m256i bad = _mm256_setzero_si256();
  // A 32-byte aligned destination (the pinned staging buffer) takes streaming stores: the lines go
  // to memory for the DMA without being read first
  const bool nt = SF_HOST_NT && ((uintptr_t)dst & 31) == 0;
  size_t i = 0;
  for (; i + 16 <= n; i += 16) {
    if (SF_HOST_PF > 0) _mm_prefetch(reinterpret_cast<const char*>(src + i + SF_HOST_PF), _MM_HINT_T0);
    const __m256 v0 = _mm256_loadu_ps(src + i), v1 = _mm256_loadu_ps(src + i + 8);
    const __m256i b0 = _mm256_castps_si256(v0), b1 = _mm256_castps_si256(v1);
    // signed compare: sign-set patterns are negative (> lim fails, < 0 caught by the gt below)
    const __m256i r0 = _mm256_or_si256(_mm256_cmpgt_epi32(b0, lim), _mm256_cmpgt_epi32(_mm256_setzero_si256(), b0));
    const __m256i r1 = _mm256_or_si256(_mm256_cmpgt_epi32(b1, lim), _mm256_cmpgt_epi32(_mm256_setzero_si256(), b1));
    const __m256i i0 = _mm256_cvttps_epi32(v0), i1 = _mm256_cvttps_epi32(v1);
    const __m256 e0 = _mm256_cmp_ps(_mm256_cvtepi32_ps(i0), v0, _CMP_NEQ_UQ);  // fraction (or NaN)
    const __m256 e1 = _mm256_cmp_ps(_mm256_cvtepi32_ps(i1), v1, _CMP_NEQ_UQ);
    bad = _mm256_or_si256(bad, _mm256_or_si256(_mm256_or_si256(r0, r1),
                                               _mm256_or_si256(_mm256_castps_si256(e0), _mm256_castps_si256(e1))));
    // pack to u16 (per 128-bit lane), then restore element order
    const __m256i p = _mm256_permute4x64_epi64(_mm256_packus_epi32(i0, i1), 0xD8);
    if (nt)
      _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), p);
    else
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + i), p);
    if (((i + 16) & (kCheck - 1)) == 0 &&
        (!_mm256_testz_si256(bad, bad) || (stop && stop->load(std::memory_order_relaxed)))) {
      if (nt) _mm_sfence();
      if (stop) stop->store(true, std::memory_order_relaxed);
      return false;
    }
  }
  if (nt) _mm_sfence();
  bool ok = _mm256_testz_si256(bad, bad) != 0;
  for (; i < n; ++i) ok &= narrow_one(src[i], dst[i]);
  if (!ok && stop) stop->store(true, std::memory_order_relaxed);
  return ok;
}

bool narrow_block(uint16_t* dst, const float* src, size_t n, std::atomic<bool>* stop) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  return avx2 ? narrow_avx2(dst, src, n, stop) : narrow_scalar(dst, src, n, stop);
}

// memcpy into a 32-byte aligned destination with streaming stores (the source unaligned)
__attribute__((target("avx2"))) void copy_nt_avx2(void* dst, const void* src, size_t bytes) {
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  size_t i = 0;
  for (; i + 128 <= bytes; i += 128) {
    if (SF_HOST_PF > 0) _mm_prefetch(s + i + 4 * SF_HOST_PF, _MM_HINT_T0);
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 64));
    const __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 96), e);
  }
  _mm_sfence();
  if (i < bytes) memcpy(d + i, s + i, bytes - i);
}

void copy_block(void* dst, const void* src, size_t bytes) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (SF_HOST_NT && avx2 && ((uintptr_t)dst & 31) == 0 && bytes >= 4096)
    copy_nt_avx2(dst, src, bytes);
  else
    memcpy(dst, src, bytes);
}

}  // namespace

namespace sf {

// memcpy over `threads` threads (pinned staging of pageable input), streaming stores when possible
void par_copy(void* dst, const void* src, size_t bytes, int threads) {
  constexpr size_t kPiece = 4u << 20;
  const int T = (int)std::min<size_t>((size_t)std::max(1, threads), (bytes + kPiece - 1) / kPiece);
  if (T <= 1) {
    copy_block(dst, src, bytes);
    return;
  }
  const size_t per = ((bytes + T - 1) / T + 63) & ~(size_t)63;
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) {
    const size_t a = std::min(bytes, per * t), b = std::min(bytes, per * (t + 1));
    if (b > a) th.emplace_back([=] { copy_block((char*)dst + a, (const char*)src + a, b - a); });
  }
  copy_block(dst, src, std::min(bytes, per));
  for (auto& x : th) x.join();
}

// dst[i] = (uint16_t)src[i] for i < n over `threads` threads; true iff every value narrowed exactly
bool par_narrow_u16(uint16_t* dst, const float* src, size_t n, int threads) {
  constexpr size_t kPiece = 1u << 20;  // elements
  const int T = (int)std::min<size_t>((size_t)std::max(1, threads), (n + kPiece - 1) / kPiece);
  std::atomic<bool> stop{false};
  if (T <= 1) return narrow_block(dst, src, n, &stop);
  const size_t per = ((n + T - 1) / T + 15) & ~(size_t)15;
  std::vector<char> ok(T, 1);
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) {
    const size_t a = std::min(n, per * t), b = std::min(n, per * (t + 1));
    th.emplace_back([&, t, a, b] { ok[t] = narrow_block(dst + a, src + a, b - a, &stop); });
  }
  ok[0] = narrow_block(dst, src, std::min(n, per), &stop);
  for (auto& x : th) x.join();
  return !stop.load() && std::all_of(ok.begin(), ok.end(), [](char c) { return c != 0; });
}

}  // namespace sf

extern "C" int sf_debug_narrow_u16(const float* src, int64_t n, uint16_t* dst, int32_t threads) {
  if (n < 0 || (n > 0 && (!src || !dst))) return -1;
  return sf::par_narrow_u16(dst, src, (size_t)n, threads) ? 1 : 0;
}

extern "C" int sf_debug_par_copy(void* dst, const void* src, int64_t bytes, int32_t threads) {
  if (bytes < 0 || (bytes > 0 && (!src || !dst))) return -1;
  sf::par_copy(dst, src, (size_t)bytes, threads);
  return 0;
}
