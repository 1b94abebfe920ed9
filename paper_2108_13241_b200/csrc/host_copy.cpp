// Host-side bulk copy for the staged transfers (pinned staging <-> caller
// arrays): 32-B non-temporal stores, so a multi-GB readback into fresh
// arrays does not first read every destination line into the cache
// (read-for-ownership) only to overwrite it.  Plain memcpy for small copies,
// for CPUs without AVX2, and with LBM_NT=0.
#include <immintrin.h>

#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>

namespace {

__attribute__((target("avx2"))) void nt_copy_avx2(char* d, const char* s, size_t n) {
  size_t head = (32 - ((uintptr_t)d & 31)) & 31;
  if (head > n) head = n;
  memcpy(d, s, head);
  d += head;
  s += head;
  n -= head;
  const size_t k = n / 128;
  for (size_t i = 0; i < k; ++i, d += 128, s += 128) {
    const __m256i a = _mm256_loadu_si256((const __m256i*)s);
    const __m256i b = _mm256_loadu_si256((const __m256i*)(s + 32));
    const __m256i c = _mm256_loadu_si256((const __m256i*)(s + 64));
    const __m256i e = _mm256_loadu_si256((const __m256i*)(s + 96));
    _mm256_stream_si256((__m256i*)d, a);
    _mm256_stream_si256((__m256i*)(d + 32), b);
    _mm256_stream_si256((__m256i*)(d + 64), c);
    _mm256_stream_si256((__m256i*)(d + 96), e);
  }
  memcpy(d, s, n - k * 128);
  _mm_sfence();  // the streamed lines are visible before a DMA or another thread reads them
}

}  // namespace

__attribute__((visibility("hidden"))) void lbm_bulk_copy(char* d, const char* s, size_t n) {
  static const bool nt = [] {
    const char* v = getenv("LBM_NT");
    return !(v && v[0] == '0') && __builtin_cpu_supports("avx2");
  }();
  if (nt && n >= (64u << 10)) {
    nt_copy_avx2(d, s, n);
    return;
  }
  memcpy(d, s, n);
}
