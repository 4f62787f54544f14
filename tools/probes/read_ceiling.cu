// read_ceiling.cu -- what a plain streaming read reaches per launch at the replay's sizes (development probe).
//
// The GEMV roofline in bench.py is the step's four per-linear launches (OPT-30B at alpha ~0.24, B = 1:
// 77.07 / 25.69 / 100.93 / 102.76 MB) back to back over a 4 GiB ring.  This probe times the simplest
// possible kernel over the same byte sequence -- every thread streams 16-byte ld.global.nc loads, eight
// in flight, XOR-reduced -- to separate the per-launch cost any kernel pays (launch, ramp to full
// bandwidth, drain) from what the GEMV adds, and tries two ways to hide it:
//   * programmatic dependent launch (griddepcontrol.launch_dependents first thing);
//   * + each CTA, once its own loads are issued, prefetches its share of the NEXT launch's first
//     `pf` bytes into L2 (cp.async.bulk.prefetch.L2), so the HBM pipe stays full across the boundary.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/rc tools/probes/read_ceiling.cu
//   /tmp/rc
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            return 1;                                                                           \
        }                                                                                       \
    } while (0)

__device__ __forceinline__ uint4 ldnc(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

struct Args {
    const uint4 *p;
    int64_t n16;
    const char *next;  // next launch's bytes (L2 prefetch) or null
    int64_t pf_bytes;
    uint32_t *out;
    int wait_mode;  // 0 none, 1 griddepcontrol.wait before any load, 2 after the first batch of loads
};

template <bool PDL>
__global__ void __launch_bounds__(512) read_kernel(const __grid_constant__ Args a) {
    if (PDL && threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    if (a.wait_mode == 1) asm volatile("griddepcontrol.wait;" ::: "memory");
    bool first = true;
    for (; i + 7 * stride < a.n16; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = ldnc(a.p + i + j * stride);
        if (first && a.wait_mode == 2) asm volatile("griddepcontrol.wait;" ::: "memory");
        first = false;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc ^= v[j].x ^ v[j].y ^ v[j].z ^ v[j].w;
    }
    for (; i < a.n16; i += stride) {
        const uint4 v = ldnc(a.p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (a.next && threadIdx.x == 0) {  // this CTA's share of the next launch's prefix, 64 KB per instruction
        const int64_t share = (a.pf_bytes / gridDim.x + 15) / 16 * 16;
        const int64_t b0 = share * blockIdx.x;
        for (int64_t o = b0; o < b0 + share && o < a.pf_bytes; o += 65536) {
            const int64_t len = (b0 + share < a.pf_bytes ? b0 + share : a.pf_bytes) - o;
            const uint32_t n = (uint32_t)(len < 65536 ? len : 65536);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.next + o), "r"(n) : "memory");
        }
    }
    if (acc == 0x12345678u) a.out[blockIdx.x] = acc;
}

// a warp per 14 KB row (K = 7168 bf16): lane l holds vectors l, l+32, ... (28 x 16 B in flight per lane),
// griddepcontrol.wait after the first row's loads are issued (where a GEMV would then read x)
template <int NV>
__global__ void __launch_bounds__(128) row_kernel(const __grid_constant__ Args a) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int64_t rows = a.n16 / (NV * 32);
    const int64_t gw = (int64_t)gridDim.x * 4, w = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    uint32_t acc = 0;
    bool waited = false;
    for (int64_t r = w; r < rows; r += gw) {
        uint4 v[NV];
        const uint4 *row = a.p + r * NV * 32;
#pragma unroll
        for (int j = 0; j < NV; ++j) v[j] = ldnc(row + lane + 32 * j);
        if (!waited && a.wait_mode) asm volatile("griddepcontrol.wait;" ::: "memory");
        waited = true;
#pragma unroll
        for (int j = 0; j < NV; ++j) acc ^= v[j].x ^ v[j].y ^ v[j].z ^ v[j].w;
    }
    if (!waited && a.wait_mode) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (acc == 0x12345678u) a.out[blockIdx.x] = acc;
}

// the GEMV's arithmetic on top of the row read: MODE 0 = x staging only (XOR), 1 = + fma8 in the
// library's order (one accumulator chain per lane), 2 = four accumulators (j mod 4), 3 = x staged as
// fp32 (converted once per CTA), one chain
__device__ __forceinline__ float lo_f(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float hi_f(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }
template <int MODE, int NV>
__global__ void __launch_bounds__(128, 3) gemv_like(const __grid_constant__ Args a, const uint4 *x, float *y) {
    extern __shared__ __align__(16) uint8_t sm[];
    if (a.pf_bytes != 1 || threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int64_t KV = NV * 32;
    const int64_t rows = a.n16 / KV;
    const int64_t gw = (int64_t)gridDim.x * 4, w0 = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    uint4 v[NV];
    int64_t r = w0;
    if (r < rows) {
#pragma unroll
        for (int j = 0; j < NV; ++j) v[j] = ldnc(a.p + r * KV + lane + 32 * j);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (MODE == 3) {
        float4 *xf = (float4 *)sm;
        for (int i = threadIdx.x; i < KV; i += 128) {
            const uint4 q = x[i];
            xf[2 * i] = make_float4(lo_f(q.x), hi_f(q.x), lo_f(q.y), hi_f(q.y));
            xf[2 * i + 1] = make_float4(lo_f(q.z), hi_f(q.z), lo_f(q.w), hi_f(q.w));
        }
    } else {
        for (int i = threadIdx.x; i < KV; i += 128)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(sm + 16 * i)),
                         "l"(x + i) : "memory");
        asm volatile("cp.async.commit_group;\n cp.async.wait_all;" ::: "memory");
    }
    __syncthreads();
    const uint4 *xs = (const uint4 *)sm;
    const float4 *xf4 = (const float4 *)sm;
    uint32_t accx = 0;
    for (; r < rows; r += gw) {
        if (r != w0) {
#pragma unroll
            for (int j = 0; j < NV; ++j) v[j] = ldnc(a.p + r * KV + lane + 32 * j);
        }
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const uint4 wv = v[j];
            if (MODE == 0) {
                const uint4 q = xs[lane + 32 * j];
                accx ^= wv.x ^ wv.y ^ wv.z ^ wv.w ^ q.x;
                continue;
            }
            float xv[8];
            if (MODE == 3) {
                const float4 p0 = xf4[2 * (lane + 32 * j)], p1 = xf4[2 * (lane + 32 * j) + 1];
                xv[0] = p0.x; xv[1] = p0.y; xv[2] = p0.z; xv[3] = p0.w; xv[4] = p1.x; xv[5] = p1.y; xv[6] = p1.z; xv[7] = p1.w;
            } else {
                const uint4 q = xs[lane + 32 * j];
                xv[0] = lo_f(q.x); xv[1] = hi_f(q.x); xv[2] = lo_f(q.y); xv[3] = hi_f(q.y);
                xv[4] = lo_f(q.z); xv[5] = hi_f(q.z); xv[6] = lo_f(q.w); xv[7] = hi_f(q.w);
            }
            float &c = acc[MODE == 2 ? (j & 3) : 0];
            c = fmaf(lo_f(wv.x), xv[0], c); c = fmaf(hi_f(wv.x), xv[1], c);
            c = fmaf(lo_f(wv.y), xv[2], c); c = fmaf(hi_f(wv.y), xv[3], c);
            c = fmaf(lo_f(wv.z), xv[4], c); c = fmaf(hi_f(wv.z), xv[5], c);
            c = fmaf(lo_f(wv.w), xv[6], c); c = fmaf(hi_f(wv.w), xv[7], c);
        }
        float t = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) y[r] = t + (float)(accx & 1);
    }
}


// thread-per-row: lane i of a warp streams row (32 w + i) in 64 B steps (4 x 16 B loads, all in flight
// for NS steps) -- the access pattern of loading a W tile row-per-thread for tcgen05.st (TMEM lane = row)
template <int NS, bool CACHE>
__global__ void __launch_bounds__(128) tpr_kernel(const __grid_constant__ Args a) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int64_t rowbytes = 14336;  // K = 7168 bf16
    const int64_t rows = a.n16 * 16 / rowbytes;
    const int64_t tiles = rows / 128;
    uint32_t acc = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const char *row = (const char *)a.p + (t * 128 + threadIdx.x) * rowbytes;
        for (int64_t k = 0; k < rowbytes; k += 64 * NS) {
            uint4 v[4 * NS];
#pragma unroll
            for (int j = 0; j < 4 * NS; ++j) {
                const uint4 *q = (const uint4 *)(row + k) + j;
                if (CACHE) v[j] = *q;
                else v[j] = ldnc(q);
            }
#pragma unroll
            for (int j = 0; j < 4 * NS; ++j) acc ^= v[j].x ^ v[j].w;
        }
        if (t == blockIdx.x) asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    if (acc == 0x12345678u) a.out[blockIdx.x] = acc;
}

__global__ void flush_kernel(uint4 *p, int64_t n16) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = make_uint4((uint32_t)i, 0, 0, 0);
}

float *g_y = nullptr;
const uint4 *g_x = nullptr;
int launch(bool pdl, const Args &a, int grid, int block, cudaStream_t s, bool rowk = false, int gmode = -1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    if (gmode >= 0 && gmode < 10) {
        cfg.dynamicSmemBytes = gmode == 3 ? 28672 : 14336;
        switch (gmode) {
            case 0: return (int)cudaLaunchKernelEx(&cfg, gemv_like<0, 28>, a, g_x, g_y);
            case 1: return (int)cudaLaunchKernelEx(&cfg, gemv_like<1, 28>, a, g_x, g_y);
            case 2: return (int)cudaLaunchKernelEx(&cfg, gemv_like<2, 28>, a, g_x, g_y);
            default: return (int)cudaLaunchKernelEx(&cfg, gemv_like<3, 28>, a, g_x, g_y);
        }
    }
    if (gmode == 10) return (int)cudaLaunchKernelEx(&cfg, tpr_kernel<2, false>, a);
    if (gmode == 11) return (int)cudaLaunchKernelEx(&cfg, tpr_kernel<2, true>, a);
    if (gmode == 12) return (int)cudaLaunchKernelEx(&cfg, tpr_kernel<4, true>, a);
    if (rowk) return (int)cudaLaunchKernelEx(&cfg, row_kernel<28>, a);
    return (int)(pdl ? cudaLaunchKernelEx(&cfg, read_kernel<true>, a) : cudaLaunchKernelEx(&cfg, read_kernel<false>, a));
}

int main() {
    const double peak = 6542.4;  // MEASURED_PEAKS.json hbm_gbs on this pool
    const int64_t ring = 4ll << 30;
    char *buf;
    uint32_t *out;
    uint4 *fl;
    CK(cudaMalloc(&buf, ring));
    CK(cudaMemset(buf, 1, ring));
    CK(cudaMalloc(&out, 1 << 20));
    CK(cudaMalloc(&fl, 256 << 20));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const double mb[4] = {77.07, 25.69, 100.93, 102.76};
    const int reps = 20;
    // the replay's sequence: 4 launches per rep, walking the ring (every launch at fresh addresses)
    std::vector<int64_t> off, len;
    int64_t o = 0;
    for (int r = 0; r < reps; ++r)
        for (int l = 0; l < 4; ++l) {
            const int64_t n = ((int64_t)(mb[l] * 1e6) + 4095) / 4096 * 4096;
            if (o + n > ring) o = 0;
            off.push_back(o);
            len.push_back(n);
            o += n;
        }
    double total = 0;
    for (size_t i = 0; i < len.size(); ++i) total += (double)len[i];
    if (getenv("RC_SINGLE")) {  // one launch per size and kernel, L2 flushed before each (for ncu)
        for (int k = 0; k < 2; ++k)
            for (int l = 0; l < 4; ++l) {
                flush_kernel<<<sms * 4, 512, 0, s>>>(fl, (256 << 20) / 16);
                Args a{(const uint4 *)(buf + off[l]), len[l] / 16, nullptr, 0, out, 0};
                CK((cudaError_t)launch(false, a, sms * 4, k == 0 ? 512 : 128, s, k == 1));
                CK(cudaStreamSynchronize(s));
            }
        printf("single launches done\n");
        return 0;
    }
    printf("sequence: %d launches, %.1f MB; SMs %d; peak %.1f GB/s\n", (int)len.size(), total / 1e6, sms, peak);
    struct V {
        const char *name;
        bool pdl;
        int64_t pf;
        int cps, block;
        int wait_mode;
        bool rowk;
        bool ev = false;  // an event record between launches (as the library's replay did)
        int gmode = -1;
    };
    const V vs[] = {
        {"plain 4x512", false, 0, 4, 512},   {"pdl 4x512", true, 0, 4, 512},
        {"pdl 2x512", true, 0, 2, 512},      {"pdl 8x256", true, 0, 8, 256},
        {"pdl+pf 4MB", true, 4 << 20, 4, 512}, {"pdl+pf 8MB", true, 8 << 20, 4, 512},
        {"pdl+pf 16MB", true, 16 << 20, 4, 512}, {"pdl+pf 32MB", true, 32 << 20, 4, 512},
        {"pdl+pf 16MB 2x512", true, 16 << 20, 2, 512},
        {"pdl wait-first 4x512", true, 0, 4, 512, 1}, {"pdl wait-after8 4x512", true, 0, 4, 512, 2},
        {"pdl wait-first 2x512", true, 0, 2, 512, 1}, {"pdl+pf16 wait-first", true, 16 << 20, 4, 512, 1},
        {"pdl+pf32 wait-first", true, 32 << 20, 4, 512, 1}, {"pdl+pf32 wait-after8", true, 32 << 20, 4, 512, 2},
        {"pdl wait-after8 8x256", true, 0, 8, 256, 2}, {"pdl wait-first 8x256", true, 0, 8, 256, 1},
        {"row 3x128 wait-row0", true, 0, 3, 128, 1, true}, {"row 4x128 wait-row0", true, 0, 4, 128, 1, true},
        {"row 6x128 wait-row0", true, 0, 6, 128, 1, true}, {"row 8x128 wait-row0", true, 0, 8, 128, 1, true},
        {"row 4x128 no wait", true, 0, 4, 128, 0, true},
        {"gemv-like xor+x 3x128", true, 0, 3, 128, 1, false, false, 0},
        {"gemv-like fma 3x128", true, 0, 3, 128, 1, false, false, 1},
        {"thread/row nc 2x64B 4x128", true, 0, 4, 128, 0, false, false, 10},
        {"thread/row L1 2x64B 4x128", true, 0, 4, 128, 0, false, false, 11},
        {"thread/row L1 4x64B 4x128", true, 0, 4, 128, 0, false, false, 12},
        {"thread/row L1 4x64B 8x128", true, 0, 8, 128, 0, false, false, 12},
        {"gemv-like fma4acc 3x128", true, 0, 3, 128, 1, false, false, 2},
        {"gemv-like fma xf32 3x128", true, 0, 3, 128, 1, false, false, 3},
        {"gemv-like fma 4x128", true, 0, 4, 128, 1, false, false, 1},
        {"gemv-like fma4acc 4x128", true, 0, 4, 128, 1, false, false, 2},
    };
    CK(cudaMalloc(&g_y, 64 << 20));
    CK(cudaMalloc((void **)&g_x, 1 << 20));
    CK(cudaMemset((void *)g_x, 0, 1 << 20));
    for (int m = 0; m < 4; ++m) {
        cudaError_t e = cudaSuccess;
        if (m == 0) e = cudaFuncSetAttribute(gemv_like<0, 28>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
        if (m == 1) e = cudaFuncSetAttribute(gemv_like<1, 28>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
        if (m == 2) e = cudaFuncSetAttribute(gemv_like<2, 28>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
        if (m == 3) e = cudaFuncSetAttribute(gemv_like<3, 28>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
        CK(e);
    }
    cudaEvent_t evd;
    CK(cudaEventCreateWithFlags(&evd, cudaEventDisableTiming));
    // warm up: ~0.5 s of streaming so clocks settle before anything is timed
    for (int w = 0; w < 400; ++w) {
        Args a{(const uint4 *)buf, (1ll << 30) / 16, nullptr, 0, out, 0};
        CK((cudaError_t)launch(true, a, sms * 4, 512, s));
    }
    CK(cudaStreamSynchronize(s));
    for (int round = 0; round < 1; ++round)
    for (const V &v : vs) {
        double best = 1e30;
        for (int t = 0; t < 5; ++t) {
            flush_kernel<<<sms * 4, 512, 0, s>>>(fl, (256 << 20) / 16);
            CK(cudaEventRecord(e0, s));
            for (size_t i = 0; i < len.size(); ++i) {
                Args a{(const uint4 *)(buf + off[i]), len[i] / 16, nullptr, 0, out, v.wait_mode};
                if (v.pf && i + 1 < len.size()) {
                    a.next = buf + off[i + 1];
                    a.pf_bytes = v.pf < len[i + 1] ? v.pf : len[i + 1];
                }
                CK((cudaError_t)launch(v.pdl, a, sms * v.cps, v.block, s, v.rowk, v.gmode));
                if (v.ev) CK(cudaEventRecord(evd, s));
            }
            CK(cudaEventRecord(e1, s));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < best) best = ms;
        }
        const double gbs = total / (best * 1e-3) / 1e9;
        printf("%-22s %8.1f us/launch  %7.1f GB/s  frac %.3f\n", v.name, best * 1e3 / len.size(), gbs, gbs / peak);
    }
    // the bench's replay order: 20 launches of ONE linear back to back, per linear
    for (int legacy = 0; legacy < 1; ++legacy)
    for (int gm = -2; gm < 3; ++gm) {
        if (legacy) s = 0;  // the legacy default stream (what torch.cuda.current_stream() is by default)
        double tb = 0, tt = 0;
        printf("%s per-linear x20 (%s):", legacy ? "LEGACY" : "own stream", gm == -2 ? "row xor 4x128" : gm == -1 ? "row xor 3x128" : gm == 0 ? "gemv-like x 3x128" : gm == 1 ? "gemv-like fma 3x128" : "gemv-like fma 3x128, launch_dependents by thread 0 only");
        for (int l = 0; l < 4; ++l) {
            const int64_t n = ((int64_t)(mb[l] * 1e6) + 4095) / 4096 * 4096;
            double best = 1e30;
            for (int t = 0; t < 5; ++t) {
                flush_kernel<<<sms * 4, 512, 0, s>>>(fl, (256 << 20) / 16);
                CK(cudaEventRecord(e0, s));
                int64_t oo = 0;
                for (int i = 0; i < reps; ++i) {
                    if (oo + n > ring) oo = 0;
                    Args a{(const uint4 *)(buf + oo), n / 16, nullptr, gm == 2 ? 1 : 0, out, 1};
                    oo += n;
                    if (gm < 0) CK((cudaError_t)launch(true, a, sms * (gm == -2 ? 4 : 3), 128, s, true));
                    else CK((cudaError_t)launch(true, a, sms * 3, 128, s, false, gm == 0 ? 0 : 1));
                    (void)0;
                }
                CK(cudaEventRecord(e1, s));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                if (ms < best) best = ms;
            }
            tb += (double)n * reps;
            tt += best * 1e-3;
            printf("  %.1f MB %.2f us", n / 1e6, best * 1e3 / reps);
        }
        printf("  -> frac %.3f\n", tb / tt / 1e9 / peak);
    }
    // one launch of each size after an L2 flush, event to event (includes launch + event latency)
    for (int l = 0; l < 4; ++l) {
        double best = 1e30;
        for (int t = 0; t < 5; ++t) {
            flush_kernel<<<sms * 4, 512, 0, s>>>(fl, (256 << 20) / 16);
            CK(cudaEventRecord(e0, s));
            Args a{(const uint4 *)(buf + off[l]), len[l] / 16, nullptr, 0, out, 0};
            CK((cudaError_t)launch(false, a, sms * 4, 512, s));
            CK(cudaEventRecord(e1, s));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < best) best = ms;
        }
        printf("single %6.2f MB: %7.2f us  %7.1f GB/s  frac %.3f\n", len[l] / 1e6, best * 1e3,
               len[l] / (best * 1e-3) / 1e9, len[l] / (best * 1e-3) / 1e9 / peak);
    }
    // one launch over the whole layer's bytes (the four linears' sizes summed)
    {
        int64_t n = 0;
        for (int l = 0; l < 4; ++l) n += len[l];
        double best = 1e30;
        for (int t = 0; t < 5; ++t) {
            flush_kernel<<<sms * 4, 512, 0, s>>>(fl, (256 << 20) / 16);
            CK(cudaEventRecord(e0, s));
            Args a{(const uint4 *)(buf + (1ll << 30)), n / 16, nullptr, 0, out, 0};
            CK((cudaError_t)launch(false, a, sms * 4, 512, s));
            CK(cudaEventRecord(e1, s));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < best) best = ms;
        }
        printf("single %6.2f MB (layer): %7.2f us  %7.1f GB/s  frac %.3f\n", n / 1e6, best * 1e3,
               n / (best * 1e-3) / 1e9, n / (best * 1e-3) / 1e9 / peak);
    }
    return 0;
}
