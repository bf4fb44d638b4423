// lmx_hostload.cpp -- the host side of a load from host memory: narrowing the
// int64 endpoint arrays to u32 with the range / self-loop checks of
// graph.py:70-90 (check_uv in lmx_setup.cu), written into the pinned staging
// ring with streaming stores (no read-for-ownership of the ring lines).
// Compiled by the host compiler (g++ -O3); the AVX2 body is chosen at run time.
#include <immintrin.h>
#include <stddef.h>
#include <stdint.h>

namespace {

bool narrow_scalar(const int64_t *u, const int64_t *v, size_t k, uint64_t n, uint32_t *ou, uint32_t *ov) {
    uint64_t badacc = 0;
    for (size_t i = 0; i < k; ++i) {
        const uint64_t a = (uint64_t)u[i], b = (uint64_t)v[i];
        ou[i] = (uint32_t)a;
        ov[i] = (uint32_t)b;
        badacc |= (uint64_t)((a >= n) | (b >= n) | (a == b));
    }
    return badacc != 0;
}

// 4 edges per step: valid iff 0 <= x < n (signed 64-bit compares suffice as
// n < 2^32) and u != v.  ou / ov must be 16-byte aligned.
template <bool NT>
__attribute__((target("avx2"))) bool narrow_avx2(const int64_t *u, const int64_t *v, size_t k, uint64_t n,
                                                 uint32_t *ou, uint32_t *ov) {
    const __m256i zero = _mm256_setzero_si256();
    const __m256i nv = _mm256_set1_epi64x((long long)n);
    const __m256i lows = _mm256_setr_epi32(0, 2, 4, 6, 0, 2, 4, 6);
    __m256i ok = _mm256_set1_epi64x(-1), eq = zero;
    size_t i = 0;
    for (; i + 4 <= k; i += 4) {
        const __m256i xu = _mm256_loadu_si256((const __m256i *)(u + i));
        const __m256i xv = _mm256_loadu_si256((const __m256i *)(v + i));
        ok = _mm256_and_si256(ok, _mm256_andnot_si256(_mm256_cmpgt_epi64(zero, xu), _mm256_cmpgt_epi64(nv, xu)));
        ok = _mm256_and_si256(ok, _mm256_andnot_si256(_mm256_cmpgt_epi64(zero, xv), _mm256_cmpgt_epi64(nv, xv)));
        eq = _mm256_or_si256(eq, _mm256_cmpeq_epi64(xu, xv));
        const __m128i lu = _mm256_castsi256_si128(_mm256_permutevar8x32_epi32(xu, lows));
        const __m128i lv = _mm256_castsi256_si128(_mm256_permutevar8x32_epi32(xv, lows));
        if (NT) {
            _mm_stream_si128((__m128i *)(ou + i), lu);
            _mm_stream_si128((__m128i *)(ov + i), lv);
        } else {
            _mm_store_si128((__m128i *)(ou + i), lu);
            _mm_store_si128((__m128i *)(ov + i), lv);
        }
    }
    if (NT) _mm_sfence();
    bool bad = _mm256_movemask_epi8(ok) != -1 || _mm256_movemask_epi8(eq) != 0;
    if (i < k) bad |= narrow_scalar(u + i, v + i, k - i, n, ou + i, ov + i);
    return bad;
}

}  // namespace

// true when some edge of the block fails the checks (the caller rescans for
// the first one)
// streaming: non-temporal stores (a ring larger than the last-level cache);
// otherwise cached stores, so the copy engine reads the lines from the cache.
bool lmx_narrow_block(const int64_t *u, const int64_t *v, size_t k, uint64_t n, uint32_t *ou, uint32_t *ov,
                      bool streaming) {
    static const bool avx2 = __builtin_cpu_supports("avx2");
    if (avx2 && ((uintptr_t)ou & 15) == 0 && ((uintptr_t)ov & 15) == 0)
        return streaming ? narrow_avx2<true>(u, v, k, n, ou, ov) : narrow_avx2<false>(u, v, k, n, ou, ov);
    return narrow_scalar(u, v, k, n, ou, ov);
}
