// host_gemv_avx2.cpp -- CPU-lane GEMV for hosts without AVX512-BF16,
// plus the portable scalar path and the run-time ISA selection.
//
// bf16 -> fp32 is a 16-bit left shift; products accumulate in fp32 with FMA.
#include <immintrin.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "hg_internal.h"

namespace hg {
namespace {

inline __m256 bf16x8_to_f32(const uint16_t *p) {
    __m128i h = _mm_loadu_si128((const __m128i *)p);
    return _mm256_castsi256_ps(_mm256_slli_epi32(_mm256_cvtepu16_epi32(h), 16));
}

inline float hsum256(__m256 v) {
    __m128 lo = _mm256_castps256_ps128(v), hi = _mm256_extractf128_ps(v, 1);
    lo = _mm_add_ps(lo, hi);
    lo = _mm_add_ps(lo, _mm_movehl_ps(lo, lo));
    lo = _mm_add_ss(lo, _mm_shuffle_ps(lo, lo, 1));
    return _mm_cvtss_f32(lo);
}

template <int B, int R>
inline void rows_block(const uint16_t *x, int64_t K, const uint16_t *W, int64_t r,
                       const float *bias, float *y, int64_t ldy) {
    __m256 acc[R][B];
    for (int i = 0; i < R; ++i)
        for (int b = 0; b < B; ++b) acc[i][b] = _mm256_setzero_ps();
    for (int64_t k = 0; k < K; k += 8) {  // K % 8 == 0 (ABI contract)
        __m256 wv[R];
        for (int i = 0; i < R; ++i) wv[i] = bf16x8_to_f32(W + (r + i) * K + k);
        for (int b = 0; b < B; ++b) {
            __m256 xv = bf16x8_to_f32(x + b * K + k);
            for (int i = 0; i < R; ++i) acc[i][b] = _mm256_fmadd_ps(wv[i], xv, acc[i][b]);
        }
    }
    for (int i = 0; i < R; ++i)
        for (int b = 0; b < B; ++b) {
            float s = hsum256(acc[i][b]);
            if (bias) s += bias[r + i];
            y[b * ldy + r + i] = s;
        }
}

template <int B>
void rows_tpl(const uint16_t *x, int64_t K, const uint16_t *W, int64_t r0, int64_t r1,
              const float *bias, float *y, int64_t ldy) {
    constexpr int R = B <= 2 ? 4 : (B <= 4 ? 2 : 1);
    int64_t r = r0;
    for (; r + R <= r1; r += R) rows_block<B, R>(x, K, W, r, bias, y, ldy);
    for (; r < r1; ++r) rows_block<B, 1>(x, K, W, r, bias, y, ldy);
}

inline float bf16_f(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

}  // namespace

void host_rows_avx2(const uint16_t *x, int batch, int64_t K, const uint16_t *W, int64_t r0,
                    int64_t r1, const float *bias, float *y, int64_t ldy) {
    switch (batch) {
        case 1: rows_tpl<1>(x, K, W, r0, r1, bias, y, ldy); break;
        case 2: rows_tpl<2>(x, K, W, r0, r1, bias, y, ldy); break;
        case 3: rows_tpl<3>(x, K, W, r0, r1, bias, y, ldy); break;
        case 4: rows_tpl<4>(x, K, W, r0, r1, bias, y, ldy); break;
        case 5: rows_tpl<5>(x, K, W, r0, r1, bias, y, ldy); break;
        case 6: rows_tpl<6>(x, K, W, r0, r1, bias, y, ldy); break;
        case 7: rows_tpl<7>(x, K, W, r0, r1, bias, y, ldy); break;
        default: rows_tpl<8>(x, K, W, r0, r1, bias, y, ldy); break;
    }
}

void host_rows_scalar(const uint16_t *x, int batch, int64_t K, const uint16_t *W, int64_t r0,
                      int64_t r1, const float *bias, float *y, int64_t ldy) {
    for (int64_t r = r0; r < r1; ++r)
        for (int b = 0; b < batch; ++b) {
            float s = 0.f;
            for (int64_t k = 0; k < K; ++k) s += bf16_f(x[b * K + k]) * bf16_f(W[r * K + k]);
            if (bias) s += bias[r];
            y[b * ldy + r] = s;
        }
}

host_rows_fn host_rows_select(const char **name) {
    __builtin_cpu_init();
    const char *force = getenv("HG_HOST_ISA");
    bool bf16 = __builtin_cpu_supports("avx512bf16") && __builtin_cpu_supports("avx512bw");
    bool avx2 = __builtin_cpu_supports("avx2") && __builtin_cpu_supports("fma");
    if (force && !strcmp(force, "scalar")) bf16 = avx2 = false;
    if (force && !strcmp(force, "avx2")) bf16 = false;
    if (bf16) {
        if (name) *name = "avx512bf16";
        return host_rows_avx512bf16;
    }
    if (avx2) {
        if (name) *name = "avx2";
        return host_rows_avx2;
    }
    if (name) *name = "scalar";
    return host_rows_scalar;
}

}  // namespace hg
