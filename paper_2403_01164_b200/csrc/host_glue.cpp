// host_glue.cpp -- the CPU lane's mirror of the GPU glue between linears.
//
// HeteGen keeps the non-linear modules on the GPU and sends the CPU's outputs back "for
// final processing".  On the B200 box the host link is saturated by the streamed weight
// slice, and every small transfer at a linear boundary queues behind it (measured: a 14 KB D2H
// takes 44 us instead of 10, a zero-copy read of the CPU rows 78 us).  Waiting for the GPU's
// glue output before starting the next linear's CPU rows would put both on the CPU lane's
// critical path 192 times per token.  So the CPU lane recomputes the glue itself from the full
// linear output (its own rows + the GPU rows, copied D2H while it was computing) -- the GPU still
// computes the same glue for its own lanes and for the layer output.
//
// Each function reproduces the GPU kernel in glue_sm100.cu operation for operation (IEEE fp32,
// no contraction: this file is built with -ffp-contract=off; LayerNorm's block_sum tree of 256
// threads and 8 warps is emulated exactly), so both lanes see bit-identical activations.
// hg_config.verify_mirror checks that at run time.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "hg_internal.h"

namespace hg {
namespace {

constexpr int kThreads = 256;  // glue_sm100.cu block size
constexpr float kLnEps = 1e-5f;

inline float bf2f(uint16_t v) {
    uint32_t u = (uint32_t)v << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// __float2bfloat16_rn: round to nearest even; NaN -> canonical 0x7FFF (branch-free: vectorises)
inline uint16_t f2bf(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    const uint32_t r = (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;
    return (u & 0x7fffffffu) > 0x7f800000u ? (uint16_t)0x7fff : (uint16_t)r;
}

// glue_sm100.cu block_sum: per-thread partials -> xor butterfly in each warp (all lanes equal) ->
// warp 0 sums the 8 warp totals (lanes >= 8 contribute 0) with the same butterfly.
float block_sum(const float (&part)[kThreads]) {
    float red[kThreads / 32];
    for (int w = 0; w < kThreads / 32; ++w) {
        float v[32];
        for (int l = 0; l < 32; ++l) v[l] = part[w * 32 + l];
        for (int o = 16; o > 0; o >>= 1) {
            float n[32];
            for (int l = 0; l < 32; ++l) n[l] = v[l] + v[l ^ o];
            std::memcpy(v, n, sizeof v);
        }
        red[w] = v[0];
    }
    float t[32];
    for (int l = 0; l < 32; ++l) t[l] = l < kThreads / 32 ? red[l] : 0.f;
    for (int o = 16; o > 0; o >>= 1) {
        float n[32];
        for (int l = 0; l < 32; ++l) n[l] = t[l] + t[l ^ o];
        std::memcpy(t, n, sizeof t);
    }
    return t[0];
}

// LayerNorm of one fp32 row.  Thread t of the GPU kernel accumulates elements t, t+256, ... in
// ascending order; here the same 256 accumulators advance together (k outer, t inner), which
// keeps each accumulator's order and lets the compiler vectorise across t.
void layernorm_row(const float *v, int64_t H, const float *g, const float *b, uint16_t *out) {
    alignas(64) float part[kThreads];
    const int64_t full = H / kThreads * kThreads;
    for (int t = 0; t < kThreads; ++t) part[t] = 0.f;
    for (int64_t k = 0; k < full; k += kThreads)
        for (int t = 0; t < kThreads; ++t) part[t] = part[t] + v[k + t];
    for (int64_t t = 0; t < H - full; ++t) part[t] = part[t] + v[full + t];
    const float mean = block_sum(part) / (float)H;
    for (int t = 0; t < kThreads; ++t) part[t] = 0.f;
    for (int64_t k = 0; k < full; k += kThreads)
        for (int t = 0; t < kThreads; ++t) {
            const float d = v[k + t] - mean;
            part[t] = std::fma(d, d, part[t]);
        }
    for (int64_t t = 0; t < H - full; ++t) {
        const float d = v[full + t] - mean;
        part[t] = std::fma(d, d, part[t]);
    }
    const float var = block_sum(part) / (float)H;
    const float rstd = 1.0f / std::sqrt(var + kLnEps);
    // one straight loop per parameter combination (a per-element `if (g)` kept the loop scalar:
    // ~15 us per 7168-element row against ~1 us vectorised); the same operations in each
    if (g && b) {
        for (int64_t i = 0; i < H; ++i) out[i] = f2bf(((v[i] - mean) * rstd) * g[i] + b[i]);
    } else if (g) {
        for (int64_t i = 0; i < H; ++i) out[i] = f2bf(((v[i] - mean) * rstd) * g[i]);
    } else if (b) {
        for (int64_t i = 0; i < H; ++i) out[i] = f2bf(((v[i] - mean) * rstd) + b[i]);
    } else {
        for (int64_t i = 0; i < H; ++i) out[i] = f2bf((v[i] - mean) * rstd);
    }
}

thread_local std::vector<float> t_row;

}  // namespace

bool hglue_supported() { return __builtin_cpu_supports("avx2") && __builtin_cpu_supports("fma"); }

void hglue_layernorm(const uint16_t *h, int64_t H, int batch, const float *g, const float *b, uint16_t *out) {
    t_row.resize((size_t)H);
    float *row = t_row.data();  // (hoisted: a thread_local vector indexed in the loop blocks vectorisation)
    for (int r = 0; r < batch; ++r) {
        for (int64_t i = 0; i < H; ++i) row[i] = bf2f(h[r * H + i]);
        layernorm_row(row, H, g, b, out + r * H);
    }
}

void hglue_residual_ln(const uint16_t *h, const float *y, int64_t ldy, int64_t H, int batch, uint16_t *h1,
                       const float *g, const float *b, uint16_t *a2) {
    t_row.resize((size_t)H);
    float *row = t_row.data();
    for (int r = 0; r < batch; ++r) {
        for (int64_t i = 0; i < H; ++i) h1[r * H + i] = f2bf(bf2f(h[r * H + i]) + y[r * ldy + i]);
        for (int64_t i = 0; i < H; ++i) row[i] = bf2f(h1[r * H + i]);
        layernorm_row(row, H, g, b, a2 + r * H);
    }
}

void hglue_residual(const uint16_t *h1, const float *y, int64_t ldy, int64_t H, int batch, uint16_t *out) {
    for (int r = 0; r < batch; ++r)
        for (int64_t i = 0; i < H; ++i) out[r * H + i] = f2bf(bf2f(h1[r * H + i]) + y[r * ldy + i]);
}

void hglue_slice_bf16(const float *y, int64_t ldy, int64_t col0, int64_t ncols, int batch, uint16_t *out) {
    for (int r = 0; r < batch; ++r)
        for (int64_t j = 0; j < ncols; ++j) out[r * ncols + j] = f2bf(y[r * ldy + col0 + j]);
}

void hglue_relu_bf16(const float *y, int64_t ldy, int64_t n, int batch, uint16_t *out) {
    for (int r = 0; r < batch; ++r)
        for (int64_t j = 0; j < n; ++j) {
            const float v = y[r * ldy + j];
            out[r * n + j] = f2bf(v > 0.f ? v : 0.f);
        }
}

}  // namespace hg
