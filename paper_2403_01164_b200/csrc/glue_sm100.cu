// glue_sm100.cu -- the small GPU kernels around the heterogeneous linears.
//
// HeteGen keeps every non-linear module on the GPU ("retaining all other
// modules on the GPU").  For the OPT decoder layer at decode position 0
// (reading R22) that is LayerNorm, the attention output (= V for one
// key), residual adds and ReLU, plus the join that lands the CPU lane's output
// (and bias) in its columns of y (the paper's concat).  All arithmetic is
// fp32; activations are stored as bf16 (round-to-nearest-even).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include <utility>

#include <cstdint>

#include "hg_internal.h"

namespace hg {
namespace {

constexpr int kThreads = 256;
constexpr float kLnEps = 1e-5f;

// Programmatic dependent launch: every glue kernel is launched with PDL, lets the next kernel (the
// GEMV, whose W stream does not depend on it) launch at once, and waits for the previous kernel's
// results before touching memory.
__device__ __forceinline__ void pdl_enter() {
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ float bf(const __nv_bfloat16 v) { return __bfloat162float(v); }

// Deterministic block sum (fixed tree) for 256 threads.
__device__ float block_sum(float v, float *red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float t = 0.f;
    if (threadIdx.x < 32) {
        t = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t = __fadd_rn(t, __shfl_xor_sync(0xffffffffu, t, o));
        if (threadIdx.x == 0) red[0] = t;
    }
    __syncthreads();
    return red[0];
}

// LayerNorm of one row held in `row` (fp32 values read through `get`).  Every operation is an
// explicit IEEE intrinsic (no contraction), and block_sum's tree is fixed, so host_glue.cpp can
// reproduce the result bit for bit (the CPU lane's mirrored glue).
template <typename Get>
__device__ void layernorm_row(Get get, int64_t H, const float *g, const float *b,
                              __nv_bfloat16 *out, float *red) {
    float s = 0.f;
    for (int64_t i = threadIdx.x; i < H; i += kThreads) s = __fadd_rn(s, get(i));
    const float mean = __fdiv_rn(block_sum(s, red), (float)H);
    float q = 0.f;
    for (int64_t i = threadIdx.x; i < H; i += kThreads) {
        const float d = __fsub_rn(get(i), mean);
        q = __fmaf_rn(d, d, q);
    }
    const float var = __fdiv_rn(block_sum(q, red), (float)H);
    const float rstd = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, kLnEps)));
    for (int64_t i = threadIdx.x; i < H; i += kThreads) {
        float v = __fmul_rn(__fsub_rn(get(i), mean), rstd);
        if (g) v = __fmul_rn(v, g[i]);
        if (b) v = __fadd_rn(v, b[i]);
        out[i] = __float2bfloat16_rn(v);
    }
}

__global__ void layernorm_kernel(const __nv_bfloat16 *__restrict__ h, int64_t H,
                                 const float *__restrict__ g, const float *__restrict__ b,
                                 __nv_bfloat16 *__restrict__ out) {
    pdl_enter();
    __shared__ float red[32];
    const __nv_bfloat16 *row = h + blockIdx.x * H;
    layernorm_row([&](int64_t i) { return bf(row[i]); }, H, g, b, out + blockIdx.x * H, red);
}

// h1 = bf16(h + y); a2 = LN(h1)
__global__ void residual_ln_kernel(const __nv_bfloat16 *__restrict__ h, const float *__restrict__ y,
                                   int64_t H, __nv_bfloat16 *__restrict__ h1,
                                   const float *__restrict__ g, const float *__restrict__ b,
                                   __nv_bfloat16 *__restrict__ a2) {
    pdl_enter();
    __shared__ float red[32];
    const int64_t off = blockIdx.x * H;
    for (int64_t i = threadIdx.x; i < H; i += kThreads)
        h1[off + i] = __float2bfloat16_rn(__fadd_rn(bf(h[off + i]), y[off + i]));
    __syncthreads();
    const __nv_bfloat16 *row = h1 + off;
    layernorm_row([&](int64_t i) { return bf(row[i]); }, H, g, b, a2 + off, red);
}

// ycpu is normally the CPU lane's mapped pinned buffer: the reads cross PCIe (zero-copy).
__global__ void join_kernel(float *__restrict__ y, int64_t ldy, int64_t col0, int64_t ncols,
                            int batch, const float *__restrict__ ycpu, int64_t ldsrc,
                            const float *__restrict__ bias) {
    pdl_enter();
    const int64_t total = (int64_t)batch * ncols;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / ncols, j = i - b * ncols;
        const float v = ycpu[b * ldsrc + j];
        y[b * ldy + col0 + j] = bias ? __fadd_rn(v, bias[col0 + j]) : v;
    }
}

__global__ void slice_bf16_kernel(const float *__restrict__ y, int64_t ldy, int64_t col0,
                                  int64_t ncols, int batch, __nv_bfloat16 *__restrict__ out) {
    pdl_enter();
    const int64_t total = (int64_t)batch * ncols;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / ncols, j = i - b * ncols;
        out[i] = __float2bfloat16_rn(y[b * ldy + col0 + j]);
    }
}

__global__ void relu_bf16_kernel(const float *__restrict__ y, int64_t total,
                                 __nv_bfloat16 *__restrict__ out) {
    pdl_enter();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __float2bfloat16_rn(y[i] > 0.f ? y[i] : 0.f);  // +0 for -0 and NaN (host mirror)
}

__global__ void residual_kernel(const __nv_bfloat16 *__restrict__ h1, const float *__restrict__ y,
                                int64_t total, __nv_bfloat16 *__restrict__ out) {
    pdl_enter();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __float2bfloat16_rn(__fadd_rn(bf(h1[i]), y[i]));
}

// y[b, p*n_local + j] = gbuf[p][b][j]
__global__ void gather_permute_kernel(const float *__restrict__ gbuf, int P, int batch,
                                      int64_t n_local, float *__restrict__ y) {
    pdl_enter();
    const int64_t total = (int64_t)P * batch * n_local;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = i % n_local;
        const int64_t pb = i / n_local;
        const int64_t b = pb % batch, p = pb / batch;
        y[b * (P * n_local) + p * n_local + j] = gbuf[i];
    }
}

inline unsigned grid_for(int64_t total) {
    int64_t g = (total + kThreads - 1) / kThreads;
    if (g > 148 * 8) g = 148 * 8;
    return (unsigned)(g < 1 ? 1 : g);
}

template <typename... Exp, typename... Act>
int pdl_launch(void (*kernel)(Exp...), unsigned grid, void *stream, Act &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    static const bool pdl = !getenv("HG_GLUE_PDL") || atoi(getenv("HG_GLUE_PDL")) != 0;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Act>(args)...);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}

}  // namespace

int launch_join(float *y, int64_t ldy, int64_t col0, int64_t ncols, int batch, const float *ycpu,
                int64_t ldsrc, const float *bias, void *stream) {
    if (ncols <= 0) return 0;
    return pdl_launch(join_kernel, grid_for(batch * ncols), stream, y, ldy, col0, ncols, batch, ycpu, ldsrc, bias);
}

int launch_layernorm(const void *h, int64_t H, int batch, const float *g, const float *b, void *out,
                     void *stream) {
    return pdl_launch(layernorm_kernel, (unsigned)batch, stream, (const __nv_bfloat16 *)h, H, g, b,
                      (__nv_bfloat16 *)out);
}

int launch_slice_to_bf16(const float *y, int64_t ldy, int64_t col0, int64_t ncols, int batch,
                         void *out, void *stream) {
    return pdl_launch(slice_bf16_kernel, grid_for(batch * ncols), stream, y, ldy, col0, ncols, batch,
                      (__nv_bfloat16 *)out);
}

int launch_residual_ln(const void *h, const float *y, int64_t H, int batch, void *h1,
                       const float *g, const float *b, void *a2, void *stream) {
    return pdl_launch(residual_ln_kernel, (unsigned)batch, stream, (const __nv_bfloat16 *)h, y, H,
                      (__nv_bfloat16 *)h1, g, b, (__nv_bfloat16 *)a2);
}

int launch_relu_bf16(const float *y, int64_t n, int batch, void *out, void *stream) {
    return pdl_launch(relu_bf16_kernel, grid_for(batch * n), stream, y, batch * n, (__nv_bfloat16 *)out);
}

int launch_residual(const void *h1, const float *y, int64_t H, int batch, void *out, void *stream) {
    return pdl_launch(residual_kernel, grid_for(batch * H), stream, (const __nv_bfloat16 *)h1, y, batch * H,
                      (__nv_bfloat16 *)out);
}

int launch_gather_permute(const float *gbuf, int P, int batch, int64_t n_local, float *y,
                          void *stream) {
    return pdl_launch(gather_permute_kernel, grid_for((int64_t)P * batch * n_local), stream, gbuf, P, batch,
                      n_local, y);
}

}  // namespace hg
