// host_gemv.cpp -- the CPU lane's GEMV: y_cpu = x . W_cpu^T.
//
// HeteGen computes its (1-alpha) share of every heterogeneous linear on the host
// CPU while the GPU share is in flight ("The CPU is exclusively dedicated to
// computational tasks"; Table 2's 97.8% CPU busy).  On the B200 box the
// host is a Sapphire/Emerald-Rapids class Xeon with AVX512-BF16, so the K loop is
// one VDPBF16PS per 32 weights: bf16 x bf16 products summed pairwise into fp32
// lanes, i.e. bf16 weights / activations with fp32 accumulation like the GPU lanes.
//
// This file is compiled with -mavx512bf16; hg_host_isa() selects it at run time
// only when the CPU reports avx512_bf16 (otherwise host_gemv_avx2.cpp / scalar).
#include <immintrin.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "hg_internal.h"

namespace hg {
namespace {

// R rows of W share every x load; B batch rows share every W load.  R*B zmm
// accumulators (<= 16) + R weight registers + 1 x register stay within 32 zmm.
template <int B, int R>
inline void rows_block(const uint16_t *x, int64_t K, const uint16_t *W, int64_t r,
                       const float *bias, float *y, int64_t ldy) {
    __m512 acc[R][B];
#pragma GCC unroll 8
    for (int i = 0; i < R; ++i)
#pragma GCC unroll 8
        for (int b = 0; b < B; ++b) acc[i][b] = _mm512_setzero_ps();
    const uint16_t *w[R];
#pragma GCC unroll 8
    for (int i = 0; i < R; ++i) w[i] = W + (r + i) * K;

    const int64_t K32 = K & ~int64_t(31);
    int64_t k = 0;
    for (; k < K32; k += 32) {
        __m512i wv[R];
#pragma GCC unroll 8
        for (int i = 0; i < R; ++i) {
            wv[i] = _mm512_loadu_si512((const void *)(w[i] + k));
            _mm_prefetch((const char *)(w[i] + k + 1024), _MM_HINT_T0);
        }
#pragma GCC unroll 8
        for (int b = 0; b < B; ++b) {
            __m512i xv = _mm512_loadu_si512((const void *)(x + b * K + k));
#pragma GCC unroll 8
            for (int i = 0; i < R; ++i)
                acc[i][b] = _mm512_dpbf16_ps(acc[i][b], (__m512bh)wv[i], (__m512bh)xv);
        }
    }
    if (k < K) {  // K % 8 == 0 tail: masked loads read zeros past the row
        const __mmask32 m = (__mmask32)((1ull << (K - k)) - 1ull);
        __m512i wv[R];
#pragma GCC unroll 8
        for (int i = 0; i < R; ++i) wv[i] = _mm512_maskz_loadu_epi16(m, (const void *)(w[i] + k));
#pragma GCC unroll 8
        for (int b = 0; b < B; ++b) {
            __m512i xv = _mm512_maskz_loadu_epi16(m, (const void *)(x + b * K + k));
#pragma GCC unroll 8
            for (int i = 0; i < R; ++i)
                acc[i][b] = _mm512_dpbf16_ps(acc[i][b], (__m512bh)wv[i], (__m512bh)xv);
        }
    }
#pragma GCC unroll 8
    for (int i = 0; i < R; ++i)
#pragma GCC unroll 8
        for (int b = 0; b < B; ++b) {
            float s = _mm512_reduce_add_ps(acc[i][b]);
            if (bias) s += bias[r + i];
            y[b * ldy + r + i] = s;
        }
}

template <int B>
void rows_tpl(const uint16_t *x, int64_t K, const uint16_t *W, int64_t r0, int64_t r1,
              const float *bias, float *y, int64_t ldy) {
    // More rows in flight = more concurrent DRAM streams per core; at B <= 2 the lane
    // is bound by per-core memory parallelism, not by VDPBF16PS (8 rows: +7% over 4
    // on Sapphire Rapids, measured).
    constexpr int R = B <= 2 ? 8 : (B <= 4 ? 4 : 2);
    static const bool four = getenv("HG_HOST_ROWS") && atoi(getenv("HG_HOST_ROWS")) == 4;  // A/B switch
    int64_t r = r0;
    if constexpr (R == 8) {
        if (four) {
            for (; r + 4 <= r1; r += 4) rows_block<B, 4>(x, K, W, r, bias, y, ldy);
            for (; r < r1; ++r) rows_block<B, 1>(x, K, W, r, bias, y, ldy);
            return;
        }
    }
    for (; r + R <= r1; r += R) rows_block<B, R>(x, K, W, r, bias, y, ldy);
    for (; r < r1; ++r) rows_block<B, 1>(x, K, W, r, bias, y, ldy);
}

}  // namespace

void host_rows_avx512bf16(const uint16_t *x, int batch, int64_t K, const uint16_t *W, int64_t r0,
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

uint64_t host_read_avx512(const void *p, int64_t bytes) {
    const char *c = (const char *)p;
    __m512i a0 = _mm512_setzero_si512(), a1 = a0, a2 = a0, a3 = a0;
    int64_t i = 0;
    for (; i + 256 <= bytes; i += 256) {
        a0 = _mm512_xor_si512(a0, _mm512_loadu_si512(c + i));
        a1 = _mm512_xor_si512(a1, _mm512_loadu_si512(c + i + 64));
        a2 = _mm512_xor_si512(a2, _mm512_loadu_si512(c + i + 128));
        a3 = _mm512_xor_si512(a3, _mm512_loadu_si512(c + i + 192));
    }
    a0 = _mm512_xor_si512(_mm512_xor_si512(a0, a1), _mm512_xor_si512(a2, a3));
    uint64_t out[8];
    _mm512_storeu_si512(out, a0);
    uint64_t s = 0;
    for (int j = 0; j < 8; ++j) s ^= out[j];
    for (; i < bytes; ++i) s += (uint8_t)c[i];
    return s;
}

}  // namespace hg
