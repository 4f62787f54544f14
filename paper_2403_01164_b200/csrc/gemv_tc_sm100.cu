// gemv_tc_sm100.cu -- tcgen05 tensor-core GEMV for batch 2..8.
//
// Same contract as gemv_sm100.cu: y[b, j] = sum_k x[b,k] W[j,k] (+bias[j]) with
// fp32 accumulation.  From batch 2 the SIMT kernel is instruction-issue bound (per weight it
// converts bf16 -> fp32 and issues B FMAs, and x's conversion grows with B), measured at 0.43 of
// the copy peak at B = 2 and 0.37 at B = 4 against 0.58 / 0.55 here (profiles/r01/gemv_batches.md).
// Here the conversion and the multiply-adds run on the 5th-generation tensor cores and the kernel
// stays an HBM stream (the batch is padded to N = 16 inside the MMA, the weights are read once):
//
//   D[128 rows of W, 16] (TMEM, fp32) += A[128 x 16] (W tile, smem) . B[16 x 16] (x^T, smem)
//
// * one elected thread of warp 0 issues TMA (cp.async.bulk.tensor.2d) for a
//   [128 rows x 64 k] W tile (16 KB, 128-byte swizzle) and the [16 x 64] x tile
//   (rows >= B are out of bounds and zero-filled by TMA) into a ring of smem
//   stages guarded by full/empty mbarriers;
// * one elected thread of warp 1 issues tcgen05.mma.cta_group::1.kind::f16
//   (M=128, N=16, K=16; four per stage) into a TMEM accumulator and frees each
//   stage with tcgen05.commit;
// * warps 2-5 drain the accumulator with tcgen05.ld (32x32b.x16) and either keep a running sum
//   of the row's slice partials in registers or store the partial for a cross-CTA fold.  Four
//   accumulators (TMEM columns 0-63) let the MMAs of the next units run while one is drained.
// * persistent CTAs own CONTIGUOUS ranges of work units (row tile, k-slice): equal work to within
//   one unit whatever the linear's size (the old round-robin walk left a 52-CTA grid on the o
//   projection at B = 8 and a two-unit tail on the others); the k-slice geometry depends on K only
//   and every row is the left-to-right sum of its slice partials, so every launch reduces every row
//   identically (split invariance).
// * one kernel for everything: a single buffer (hg_gemv, the resident GEMV alone, the per-chunk
//   fallback) is a launch with one source; the persistent per-linear form covers the resident
//   block and every streamed chunk, gated by the chunk arrival tags, PDL-launched (see below).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "hg_internal.h"

namespace hg {
namespace {

// Named barrier among a subset of warps.  PTX bar.sync is barrier.sync.aligned, which requires the
// whole warp to execute it convergently; call sites follow lane-divergent code (a lane-0-only grid
// barrier, loops with lane-dependent trip counts), so reconverge first and use the non-aligned form.
__device__ __forceinline__ void named_barrier(int id, int nthreads) {
    __syncwarp();
    asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}


constexpr int kTileM = 128;        // W rows per tile (UMMA M)
constexpr int kTileK = 64;         // k per stage (one 128-byte swizzle atom of bf16)
constexpr int kUmmaN = 16;         // batch padded to N = 16
constexpr int kUmmaK = 16;         // k per tcgen05.mma (bf16)
constexpr int kWBytes = kTileM * kTileK * 2;  // 16 KB
constexpr int kXBytes = kUmmaN * kTileK * 2;  // 2 KB
constexpr int kThreads = 192;                 // warp0 TMA, warp1 MMA, warps2-5 epilogue
constexpr int kNAcc = 4;                      // TMEM accumulators of 16 columns: the MMA warp may run
                                              // up to three work units ahead of the epilogue
constexpr int64_t kSliceMin = 512;            // k per work unit: at least this ...
constexpr int kSliceMaxCount = 16;            // ... and at most this many slices per row

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!ok);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, uint32_t bar,
                                            int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

// K-major, 128-byte swizzled operand: 8-row core groups 1024 B apart (SBO), LBO
// unused (1), descriptor version 1 (sm_100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;            // LBO (16 B units), unused for swizzled K-major
    d |= (uint64_t)(1024 >> 4) << 32;  // SBO
    d |= (uint64_t)1 << 46;            // version
    d |= (uint64_t)2 << 61;            // SWIZZLE_128B
    return d;
}

// kind::f16 instruction descriptor: D fp32, A/B bf16, both K-major, N=16, M=128.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kUmmaN >> 3) << 17) |
                            ((uint32_t)(kTileM >> 4) << 24);

__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accum) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc), "r"(accum)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// smem: ST stages of [W tile | x tile], then full[ST] empty[ST] tfull[kNAcc] tempty[kNAcc], TMEM slot,
// last-arriver flag
constexpr size_t smem_for(int st) { return 1024 + st * (kWBytes + kXBytes) + 8 * (2 * st + 2 * kNAcc) + 16; }
// 6-stage CTAs, two per SM (measured against 11 stages x one per SM and 4 stages x three per SM: both
// slower, profiles/r01/gemv_batches.md)
constexpr int kStagesWide = 6;

// ---------------------------------------------------------------- persistent per-linear form
// One launch per linear covering the resident block and every streamed chunk (the SIMT kernel's
// structure, SURVEY 8(a) a3+a4).  Sources: [resident block] then chunk 0, 1, ... in arrival order;
// each has its own tensor map (a kernel parameter) over exactly its rows (rows past a source are
// zero-filled by TMA, never read from a neighbour).
//
// Work: unit u = (row tile t = u / S, k-slice s = u % S), U = tiles * S units in tile-major order.
// CTA c owns the CONTIGUOUS range [c U / G, (c+1) U / G) (G = grid): every CTA gets the same number
// of units to within one, whatever the linear's size, and most tiles lie wholly inside one CTA's
// range.  Each unit's slice partial p_s (a fresh TMEM accumulation over the slice's k) is what the
// row's result is built from, always as the left-to-right fp32 sum p_0 + p_1 + ... + p_{S-1} + bias
// (the slice geometry depends on K only): so every partition of a linear into resident rows and
// chunks, and every grid, gives the same bits (split invariance).
//   * the CTA holding slice 0 of a tile (its "prefix holder") keeps the running sum in registers
//     over its consecutive slices; if it holds the whole tile it writes y directly;
//   * otherwise the prefix sum goes to the workspace at its last slice's index, and every other CTA
//     touching the tile stores its slices' partials individually; each contributor then counts in
//     on the tile's counter, and the last one adds prefix + remaining partials in slice order.
// A CTA walks its units in order, so it meets the sources in arrival order and waits for a chunk's
// arrival tag before its first TMA from that chunk.  When every unit of a chunk has finished its
// MMAs (all TMA reads of the slot done), the last one writes the slot's `consumed` tag.
constexpr int kMaxSrc = 17;  // resident + up to 16 chunks per launch (else the per-chunk path)

struct TcArgs {
    CUtensorMap map_x;
    CUtensorMap maps[kMaxSrc];
    int64_t rows[kMaxSrc], g0[kMaxSrc], tile0[kMaxSrc + 1];
    int32_t slot[kMaxSrc];
    uint32_t tag[kMaxSrc];
    int n_src;
    int S;
    int cluster;     // 1: one unit per CTA, a tile's S slices are one thread-block cluster and its
                     // slice partials are added through distributed shared memory (no workspace)
    int64_t ks, K, n_total, U;
    const float *bias;
    float *y;
    int64_t ldy;
    float *ws;       // [S][B][n_total] slice partials of tiles split across CTAs (coalesced per b)
    int *counters;   // [tiles] contributors counted in (zero between launches)
    const uint32_t *arrived;  // null: every source present (resident / replay)
    uint32_t *consumed, *slot_cnt, *err;
    unsigned long long timeout_ns;
    unsigned long long *stamps;  // measurement: [CTA][8] globaltimer, see kStamp*
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t dsmem_addr(uint32_t local_addr, uint32_t rank) {
    uint32_t remote;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(rank));
    return remote;
}
// no memory clobber: the loads of one fold are independent and may all be in flight at once (they
// are ordered after the cluster barrier, which clobbers memory)
__device__ __forceinline__ float ld_dsmem_f32(uint32_t remote) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote));
    return v;
}

// the CTA whose range [c U / G, (c+1) U / G) holds unit u
__device__ __forceinline__ int64_t cta_of(int64_t u, int64_t U, int64_t G) { return ((u + 1) * G - 1) / U; }

template <int B, int ST>
__global__ void __launch_bounds__(kThreads, 2) gemv_tc_stream_kernel(const __grid_constant__ TcArgs a) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (base - raw);
    const uint32_t sW = base;
    const uint32_t sX = base + ST * kWBytes;
    const uint32_t bars = sX + ST * kXBytes;
    uint32_t *tmem_slot = (uint32_t *)(gbase + (bars - base) + 8 * (2 * ST + 2 * kNAcc));
    int *last_flag = (int *)(tmem_slot + 1);
    auto full = [&](int s) { return bars + 8 * s; };
    auto empty = [&](int s) { return bars + 8 * (ST + s); };
    auto tfull = [&](int q) { return bars + 8 * (2 * ST + q); };
    auto tempty = [&](int q) { return bars + 8 * (2 * ST + kNAcc + q); };

    // PDL: the next kernel may be scheduled once every CTA of this one runs; x (read by the
    // producer with every stage) is the only input of the previous kernel, so only the producer
    // waits (griddepcontrol.wait) before its first x TMA.
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (a.stamps && threadIdx.x == 0) a.stamps[blockIdx.x * 8 + 0] = gtimer();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full(s), 1);
            mbar_init(empty(s), 1);
        }
        for (int q = 0; q < kNAcc; ++q) {
            mbar_init(tfull(q), 1);
            mbar_init(tempty(q), 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();  // barriers initialised: the producer starts at once; TMEM is allocated meanwhile
    uint32_t tmem = 0;
    if (warp >= 1) {  // MMA warp allocates; warps 1-5 meet on named barrier 2 (the producer never waits)
        if (warp == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(kNAcc * kUmmaN)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        named_barrier(2, kThreads - 32);
        tc_fence_after();
        tmem = *tmem_slot;
    }

    const int S = a.S;
    const int64_t U = a.U, G = gridDim.x;
    const int64_t u0 = (int64_t)blockIdx.x * U / G, u1 = ((int64_t)blockIdx.x + 1) * U / G;
    auto src_of = [&](int64_t t) {
        int i = 0;
        while (t >= a.tile0[i + 1]) ++i;
        return i;
    };
    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            // descriptors: x and this CTA's first source now, each next source when the walk reaches the
            // one before it (a prefetch of every source up front held the first TMA back ~0.8 us)
            int pf = src_of(u0 / S);
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&a.maps[pf]) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&a.map_x) : "memory");
            if (a.stamps) a.stamps[blockIdx.x * 8 + 1] = gtimer();
            int stage = 0;
            uint32_t phase = 0;
            int ready = -1;  // highest source index known to have arrived
            // W does not depend on the previous kernel, x does: the first ST stages get their W tile at
            // once and their x tile after griddepcontrol.wait (each stage's barrier expects both)
            bool dep = false;
            int pend = 0, pst[ST];
            int32_t pk[ST];
            auto flush_x = [&]() {
                asm volatile("griddepcontrol.wait;" ::: "memory");
                for (int q = 0; q < pend; ++q) tma_load_2d(sX + pst[q] * kXBytes, &a.map_x, full(pst[q]), pk[q], 0);
                pend = 0;
                dep = true;
            };
            for (int64_t u = u0; u < u1; ++u) {
                const int64_t t = u / S;
                const int s = (int)(u - t * S);
                const int i = src_of(t);
                if (i == pf && pf + 1 < a.n_src) {
                    ++pf;
                    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&a.maps[pf]) : "memory");
                }
                if (a.arrived && a.slot[i] >= 0 && i > ready) {
                    if (!dep) flush_x();
                    const unsigned long long t0 = gtimer();
                    while ((int32_t)(ld_acquire_u32(a.arrived + a.slot[i]) - a.tag[i]) < 0) {
                        __nanosleep(64);
                        if (gtimer() - t0 > a.timeout_ns) {
                            *(volatile uint32_t *)a.err = 1u;  // mapped host word: a plain store (no PCIe atomic)
                            break;
                        }
                    }
                    ready = i;
                }
                const int32_t row0 = (int32_t)((t - a.tile0[i]) * kTileM);
                const int64_t k0 = (int64_t)s * a.ks;
                const int64_t k1 = k0 + a.ks < a.K ? k0 + a.ks : a.K;
                for (int64_t k = k0; k < k1; k += kTileK) {
                    mbar_wait(empty(stage), phase ^ 1);
                    mbar_expect_tx(full(stage), kWBytes + kXBytes);
                    tma_load_2d(sW + stage * kWBytes, &a.maps[i], full(stage), (int32_t)k, row0);
                    if (a.stamps && u == u0 && k == k0) a.stamps[blockIdx.x * 8 + 2] = gtimer();
                    if (dep) {
                        tma_load_2d(sX + stage * kXBytes, &a.map_x, full(stage), (int32_t)k, 0);
                    } else {
                        pst[pend] = stage;
                        pk[pend] = (int32_t)k;
                        if (++pend == ST) flush_x();  // before any stage could be waited on again
                    }
                    if (++stage == ST) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
            if (!dep) flush_x();
            if (a.stamps) a.stamps[blockIdx.x * 8 + 7] = gtimer();
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int64_t u = u0; u < u1; ++u, ++it) {
                const int acc = it % kNAcc;
                const uint32_t aphase = (uint32_t)((it / kNAcc) & 1);
                mbar_wait(tempty(acc), aphase ^ 1);
                tc_fence_after();
                const int64_t t = u / S;
                const int s = (int)(u - t * S);
                const int64_t k0 = (int64_t)s * a.ks;
                const int64_t k1 = k0 + a.ks < a.K ? k0 + a.ks : a.K;
                const uint32_t d = tmem + (uint32_t)(acc * kUmmaN);
                uint32_t accum = 0;
                for (int64_t k = k0; k < k1; k += kTileK) {
                    mbar_wait(full(stage), phase);
                    tc_fence_after();
                    if (a.stamps && it == 0 && k == k0) a.stamps[blockIdx.x * 8 + 3] = gtimer();
#pragma unroll
                    for (int kk = 0; kk < kTileK / kUmmaK; ++kk) {
                        const uint64_t da = sw128_desc(sW + stage * kWBytes + kk * kUmmaK * 2);
                        const uint64_t db = sw128_desc(sX + stage * kXBytes + kk * kUmmaK * 2);
                        umma(d, da, db, accum);
                        accum = 1;
                    }
                    umma_commit(empty(stage));
                    if (++stage == ST) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(tfull(acc));
            }
        }
    } else {  // ---------------- epilogue warps 2..5: TMEM lanes 32*quarter.. = the tile's rows
        const int quarter = warp & 3;
        const int et = (warp - 2) * 32 + lane;
        float r[B];
        bool prefix = false;
        int it = 0;
        for (int64_t u = u0; u < u1; ++u, ++it) {
            const int acc = it % kNAcc;
            const uint32_t aphase = (uint32_t)((it / kNAcc) & 1);
            const int64_t t = u / S;
            const int s = (int)(u - t * S);
            const int i = src_of(t);
            mbar_wait(tfull(acc), aphase);
            tc_fence_after();
            if (a.stamps && it == 0 && et == 0) a.stamps[blockIdx.x * 8 + 4] = gtimer();
            uint32_t p[16];
            const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * kUmmaN);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
                "%14,%15}, [%16];"
                : "=r"(p[0]), "=r"(p[1]), "=r"(p[2]), "=r"(p[3]), "=r"(p[4]), "=r"(p[5]), "=r"(p[6]),
                  "=r"(p[7]), "=r"(p[8]), "=r"(p[9]), "=r"(p[10]), "=r"(p[11]), "=r"(p[12]),
                  "=r"(p[13]), "=r"(p[14]), "=r"(p[15])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            tc_fence_before();
            mbar_arrive(tempty(acc));
            // every TMA read of this unit has landed (its MMAs completed): count it for the slot
            if (a.arrived && a.slot[i] >= 0 && et == 0) {
                const uint32_t units_i = (uint32_t)((a.tile0[i + 1] - a.tile0[i]) * S);
                const uint32_t old = atomicAdd(&a.slot_cnt[a.slot[i]], 1u);
                if (old == units_i - 1) {
                    atomicExch(&a.slot_cnt[a.slot[i]], 0u);
                    __threadfence();
                    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.consumed + a.slot[i]), "r"(a.tag[i])
                                 : "memory");
                }
            }
            const int64_t lrow = (t - a.tile0[i]) * kTileM + quarter * 32 + lane;
            const bool valid = lrow < a.rows[i];
            const int64_t g = a.g0[i] + lrow;
            if (a.cluster) {  // the tile's fold happens through DSMEM after the loop (one unit per CTA)
                float *red = (float *)gbase;  // stage 0's W tile: free once this unit's MMAs completed
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // (last written by TMA)
#pragma unroll
                for (int b = 0; b < B; ++b) red[b * kTileM + quarter * 32 + lane] = __uint_as_float(p[b]);
                continue;
            }
            const bool first = u == u0 || s == 0;      // this CTA's first unit of tile t
            const bool last = u == u1 - 1 || s == S - 1;  // ... and its last
            if (first) prefix = s == 0;
            if (prefix) {
#pragma unroll
                for (int b = 0; b < B; ++b) r[b] = first ? __uint_as_float(p[b]) : r[b] + __uint_as_float(p[b]);
            } else if (valid) {
#pragma unroll
                for (int b = 0; b < B; ++b) a.ws[((int64_t)s * B + b) * a.n_total + g] = __uint_as_float(p[b]);
            }
            if (!last) continue;
            if (prefix && s == S - 1) {  // the whole tile in this CTA: p_0 + ... + p_{S-1} + bias
                if (valid) {
                    const float bb = a.bias ? a.bias[g] : 0.f;
#pragma unroll
                    for (int b = 0; b < B; ++b) a.y[b * a.ldy + g] = r[b] + bb;
                }
                continue;
            }
            if (prefix && valid) {  // the prefix sum p_0 + ... + p_s, stored at slice index s
#pragma unroll
                for (int b = 0; b < B; ++b) a.ws[((int64_t)s * B + b) * a.n_total + g] = r[b];
            }
            // count in (the CUTLASS semaphore pattern): the four warps' partial stores are ordered before
            // one thread's gpu-scope acq_rel atomic by the barrier; the last contributor's acquire and
            // the second barrier order its warps' partial loads after every contributor's stores
            named_barrier(1, 128);
            const int64_t cf = cta_of(t * S, U, G), cl = cta_of(t * S + S - 1, U, G);
            if (et == 0) {
                int old;
                asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(a.counters + t) : "memory");
                *last_flag = old == (int)(cl - cf);
            }
            named_barrier(1, 128);
            if (*last_flag) {  // every contributor is in: prefix + the remaining partials, in slice order
                if (valid) {
                    const int64_t ce = (cf + 1) * U / G;
                    const int pe = (int)((ce < t * S + S ? ce : t * S + S) - t * S);  // prefix = slices [0, pe)
                    float sum[B];
#pragma unroll
                    for (int b = 0; b < B; ++b) sum[b] = __ldcg(&a.ws[((int64_t)(pe - 1) * B + b) * a.n_total + g]);
                    // kFold slices x B loads issued unconditionally (indices clamped to the last slice, which
                    // is always written), then added in slice order: no load waits behind a branch
                    constexpr int kFold = 8;
                    for (int q0 = pe; q0 < S; q0 += kFold) {
                        float part[kFold][B];
#pragma unroll
                        for (int q = 0; q < kFold; ++q) {
                            const int sq = q0 + q < S ? q0 + q : S - 1;
                            const float *src = &a.ws[(int64_t)sq * B * a.n_total + g];
#pragma unroll
                            for (int b = 0; b < B; ++b) part[q][b] = __ldcg(src + (int64_t)b * a.n_total);
                        }
#pragma unroll
                        for (int q = 0; q < kFold; ++q)
                            if (q0 + q < S) {
#pragma unroll
                                for (int b = 0; b < B; ++b) sum[b] += part[q][b];
                            }
                    }
                    const float bb = a.bias ? a.bias[g] : 0.f;
#pragma unroll
                    for (int b = 0; b < B; ++b) a.y[b * a.ldy + g] = sum[b] + bb;
                }
                if (et == 0) a.counters[t] = 0;
            }
            named_barrier(1, 128);
        }
    }
    if (a.cluster) {
        // cluster rank r holds slice r of tile blockIdx.x / S: rank 0 adds the S partials in slice order
        // (the same left-to-right sum as the register / workspace paths) once every rank stored its own
        __syncwarp();
        cluster_sync_all();
        if (warp >= 2 && (blockIdx.x % S) == 0) {
            const int quarter = warp & 3;
            const int64_t t = blockIdx.x / S;
            const int i = src_of(t);
            const int64_t lrow = (t - a.tile0[i]) * kTileM + quarter * 32 + lane;
            if (lrow < a.rows[i]) {
                const int64_t g = a.g0[i] + lrow;
                const float bb = a.bias ? a.bias[g] : 0.f;
                const uint32_t red = smem_u32(gbase) + (uint32_t)(quarter * 32 + lane) * 4;
                float part[kSliceMaxCount][B];
#pragma unroll
                for (int r = 0; r < kSliceMaxCount; ++r)
                    if (r < S) {
                        const uint32_t base = dsmem_addr(red, (uint32_t)r);
#pragma unroll
                        for (int b = 0; b < B; ++b) part[r][b] = ld_dsmem_f32(base + (uint32_t)(b * kTileM) * 4);
                    }
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    float sum = part[0][b];
#pragma unroll
                    for (int r = 1; r < kSliceMaxCount; ++r)
                        if (r < S) sum += part[r][b];
                    a.y[b * a.ldy + g] = sum + bb;
                }
            }
        }
        __syncwarp();
        cluster_sync_all();  // every rank's shared memory stays valid until rank 0 has read it
    }
    if (a.stamps && warp == 2 && lane == 0) a.stamps[blockIdx.x * 8 + 5] = gtimer();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kNAcc * kUmmaN)
                     : "memory");
    if (a.stamps && threadIdx.x == 0) a.stamps[blockIdx.x * 8 + 6] = gtimer();
}

// ---------------------------------------------------------------- host side
typedef CUresult (*encode_fn_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                CUtensorMapFloatOOBfill);

encode_fn_t encode_fn() {
    static encode_fn_t fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (encode_fn_t)p;
    });
    return fn;
}

bool make_map(CUtensorMap *m, const void *ptr, int64_t inner, int64_t outer, uint32_t box_inner,
              uint32_t box_outer) {
    encode_fn_t enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)inner * 2};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int g_num_sms = 0;

template <int B, int ST>
int launch_tc_stream_st(const TcArgs &a, cudaStream_t st) {
    const int sms = g_num_sms > 0 ? g_num_sms : 148;
    int grid = 2 * sms;  // two 6-stage CTAs per SM (2 x ~112 KB smem)
    if (a.U < grid) grid = (int)a.U;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem_for(ST);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    int na = 1;
    if (a.cluster) {  // grid = U = tiles x S, one cluster of S CTAs per tile
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = (unsigned)a.S;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaError_t e = cudaLaunchKernelEx(&cfg, gemv_tc_stream_kernel<B, ST>, a);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}
// From B = 5, 4-stage CTAs (2 x ~76 KB per SM) leave room for a CTA of the NEXT launch on every SM, so
// back-to-back launches overlap (programmatic dependent launch) and the HBM stream does not drain at the
// boundary: B = 6 / 8 0.63 / 0.62 -> 0.66 / 0.65; at B = 4 the extra bytes in flight of 6 stages win
// (0.65-0.67 vs 0.64; profiles/r02/tc_stages.md).  HG_TC_ST=4|6 forces one.
static const int g_tc_st = getenv("HG_TC_ST") ? atoi(getenv("HG_TC_ST")) : 0;
template <int B>
int launch_tc_stream_b(const TcArgs &a, cudaStream_t st) {
    const bool four = g_tc_st == 4 || (g_tc_st == 0 && B >= 5);
    return four ? launch_tc_stream_st<B, 4>(a, st) : launch_tc_stream_st<B, kStagesWide>(a, st);
}

template <int B>
int prepare_tc_b() {
    int e = (int)cudaFuncSetAttribute(gemv_tc_stream_kernel<B, kStagesWide>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_for(kStagesWide));
    // clusters of up to 16 CTAs (one per k-slice of a tile): above the portable 8
    e |= (int)cudaFuncSetAttribute(gemv_tc_stream_kernel<B, kStagesWide>,
                                   cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    e |= (int)cudaFuncSetAttribute(gemv_tc_stream_kernel<B, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem_for(4));
    e |= (int)cudaFuncSetAttribute(gemv_tc_stream_kernel<B, 4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return e;
}

}  // namespace

int64_t g_slice_min = kSliceMin;       // A/B (HG_TC_SLICE_MIN): smallest k per work unit
int g_tc_cluster = 1;                  // A/B (HG_TC_CLUSTER=0): workspace fold for every split tile
int g_slice_count = kSliceMaxCount;    // A/B (HG_TC_SLICE_COUNT): most slices per row

// k-slice geometry: a function of K only (split invariance): slices of ks = 64 * max(min/64,
// ceil(K / (64 * count))) k, the last one shorter.
GemvGeom gemv_tc_geom(int64_t K) {
    GemvGeom g;
    int64_t ks = (K + (int64_t)kTileK * g_slice_count - 1) / ((int64_t)kTileK * g_slice_count) * kTileK;
    if (ks < g_slice_min) ks = g_slice_min;
    g.ks = ks;
    g.s = (int)((K + ks - 1) / ks);
    g.rows_per_cta = kTileM;
    return g;
}

int gemv_tc_prepare() {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (const char *v = getenv("HG_TC_SLICE_MIN")) {
        const int64_t sl = atoll(v) / kTileK * kTileK;
        if (sl >= kTileK) g_slice_min = sl;
    }
    if (const char *v = getenv("HG_TC_CLUSTER")) g_tc_cluster = atoi(v) != 0;
    if (const char *v = getenv("HG_TC_SLICE_COUNT")) {
        const int c = atoi(v);
        if (c >= 1 && c <= 256) g_slice_count = c;
    }
    int e = 0;
    e |= prepare_tc_b<1>();
    e |= prepare_tc_b<2>();
    e |= prepare_tc_b<3>();
    e |= prepare_tc_b<4>();
    e |= prepare_tc_b<5>();
    e |= prepare_tc_b<6>();
    e |= prepare_tc_b<7>();
    e |= prepare_tc_b<8>();
    if (!encode_fn()) e |= 1;
    return e;
}

bool gemv_tc_stream_ok(int64_t n_res, int64_t n_chunks) {
    return (n_res > 0 ? 1 : 0) + n_chunks <= kMaxSrc;
}

int64_t gemv_tc_stream_tiles(int64_t n_res, int64_t n_str, int64_t chunk_rows, int64_t n_chunks) {
    int64_t t = (n_res + kTileM - 1) / kTileM;
    for (int64_t i = 0; i < n_chunks; ++i) {
        const int64_t r0 = i * chunk_rows;
        const int64_t rows = chunk_rows < n_str - r0 ? chunk_rows : n_str - r0;
        t += (rows + kTileM - 1) / kTileM;
    }
    return t;
}

int launch_gemv_tc_stream(const StreamLaunch &L, int *counters, void *stream) {
    const int B = L.batch;
    if (B < 1 || B > 8) return (int)cudaErrorInvalidValue;
    const int64_t n_chunks = L.n_str > 0 ? L.n_chunks : 0;
    if (!gemv_tc_stream_ok(L.n_res, n_chunks)) return (int)cudaErrorInvalidValue;
    static TcArgs a;  // ~2.5 KB: not on the stack; the launch copies it (one context per host thread)
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    std::memset(&a, 0, sizeof(a));
    const int64_t K = L.K;
    if (!make_map(&a.map_x, L.x, K, B, kTileK, kUmmaN)) return (int)cudaErrorInvalidValue;
    int ns = 0;
    a.tile0[0] = 0;
    if (L.n_res > 0) {
        if (!make_map(&a.maps[ns], L.W_res, K, L.n_res, kTileK, kTileM)) return (int)cudaErrorInvalidValue;
        a.rows[ns] = L.n_res;
        a.g0[ns] = 0;
        a.slot[ns] = -1;
        a.tag[ns] = 0;
        a.tile0[ns + 1] = a.tile0[ns] + (L.n_res + kTileM - 1) / kTileM;
        ++ns;
    }
    for (int64_t i = 0; i < n_chunks; ++i) {
        const int64_t seq = L.seq0 + i;
        const int64_t slot = seq % (L.nslots > 0 ? L.nslots : 1);
        const int64_t r0 = i * L.chunk_rows;
        const int64_t rows = L.chunk_rows < L.n_str - r0 ? L.chunk_rows : L.n_str - r0;
        if (!make_map(&a.maps[ns], L.ring + slot * L.slot_bytes, K, rows, kTileK, kTileM))
            return (int)cudaErrorInvalidValue;
        a.rows[ns] = rows;
        a.g0[ns] = L.n_res + r0;
        a.slot[ns] = L.arrived ? (int32_t)slot : -1;
        a.tag[ns] = (uint32_t)(seq + 1);
        a.tile0[ns + 1] = a.tile0[ns] + (rows + kTileM - 1) / kTileM;
        ++ns;
    }
    a.n_src = ns;
    if (ns == 0) return 0;
    const GemvGeom g = gemv_tc_geom(K);
    a.S = g.s;
    a.ks = g.ks;
    a.K = K;
    a.U = a.tile0[ns] * a.S;
    // few units (at most two per SM): one unit per CTA and a tile's slices as one cluster, folded
    // through distributed shared memory instead of the workspace + counter round trip
    const int sms = g_num_sms > 0 ? g_num_sms : 148;
    a.cluster = (g_tc_cluster && a.S > 1 && a.S <= kSliceMaxCount && a.U <= 2 * sms) ? 1 : 0;
    a.n_total = L.n_res + L.n_str;
    a.bias = L.bias;
    a.y = L.y;
    a.ldy = L.ldy;
    a.ws = L.ws;
    a.counters = counters;
    a.arrived = L.arrived;
    a.consumed = L.consumed;
    a.slot_cnt = L.slot_cnt;
    a.err = L.err;
    a.timeout_ns = (unsigned long long)(L.timeout_s * 1e9 * dev_timeout_scale());
    a.stamps = gemv_stamps_dev();
    if (a.S > 1 && (!a.ws || !counters)) return (int)cudaErrorInvalidValue;
    if (a.arrived && (!a.consumed || !a.slot_cnt || !a.err)) return (int)cudaErrorInvalidValue;
    cudaStream_t st = (cudaStream_t)stream;
    switch (B) {
        case 1: return launch_tc_stream_b<1>(a, st);
        case 2: return launch_tc_stream_b<2>(a, st);
        case 3: return launch_tc_stream_b<3>(a, st);
        case 4: return launch_tc_stream_b<4>(a, st);
        case 5: return launch_tc_stream_b<5>(a, st);
        case 6: return launch_tc_stream_b<6>(a, st);
        case 7: return launch_tc_stream_b<7>(a, st);
        default: return launch_tc_stream_b<8>(a, st);
    }
}

// One buffer (the resident GEMV alone, hg_gemv, and the per-chunk fallback): the same kernel with a
// single source, so its rows get the same bits as in any persistent launch.
int launch_gemv_tc(const void *x, int batch, int64_t K, const void *W, int64_t n, const float *bias,
                   float *y, int64_t ldy, float *ws, int *counters, void *stream) {
    if (n <= 0) return 0;
    StreamLaunch L{};
    L.x = x;
    L.batch = batch;
    L.K = K;
    L.W_res = W;
    L.n_res = n;
    L.bias = bias;
    L.y = y;
    L.ldy = ldy;
    L.ws = ws;
    L.timeout_s = 60.0;
    return launch_gemv_tc_stream(L, counters, stream);
}

}  // namespace hg
