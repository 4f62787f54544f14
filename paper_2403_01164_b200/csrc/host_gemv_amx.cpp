// host_gemv_amx.cpp -- the CPU lane's GEMV on AMX tiles for batch >= 4.
//
// At batch 1-2 the CPU lane is bound by host DRAM and AVX512-BF16 keeps up; from batch ~4 the
// vdpbf16ps count per weight byte (B per 64 B) makes it ALU-heavy (v_cpu falls ~25% at B=8).  The
// B200 box's host has AMX-BF16: one TDPBF16PS multiplies a 16-row x 32-k bf16 tile of W by a
// 32-k x B tile of x (pairs interleaved, "VNNI" layout) into a 16 x B fp32 accumulator tile --
// 16*B*32 multiply-adds per instruction -- so the lane is memory-bound again.
//
// Rows are done 16 at a time (a tail of < 16 rows, or K % 32 != 0, goes to the AVX-512 path);
// x is packed once per job into the pair-interleaved layout.  Every call loads the tile configuration
// (LDTILECFG) and releases it at the end; the process asks the kernel for AMX state once (arch_prctl).  fp32
// accumulation of bf16 products like the other lanes; the order of the sums differs from the
// AVX-512 path, which the CPU rows' tolerance comparison allows.
#include <immintrin.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include "hg_internal.h"

namespace hg {
namespace {

struct alignas(64) TileCfg {
    uint8_t palette = 1;
    uint8_t start_row = 0;
    uint8_t reserved[14] = {};
    uint16_t colsb[16] = {};
    uint8_t rows[16] = {};
};

// tmm0: C [16 rows][B fp32]; tmm1: A = W [16 rows][32 bf16]; tmm2: B = x pairs [16][B][2 bf16].
// Loaded at the start of every call and released at its end: the thread may be the API caller's,
// where other code (e.g. a oneDNN bf16 kernel) can run AMX with its own configuration and
// TILERELEASE it in between; a cached "already configured" flag would then run tile instructions
// on an unconfigured (#UD) or foreign configuration.  LDTILECFG costs ~100 cycles against the
// ~20 us a call's 16-row blocks take.
void config_tiles(int B) {
    TileCfg cfg;
    cfg.rows[0] = 16;
    cfg.colsb[0] = (uint16_t)(B * 4);
    cfg.rows[1] = 16;
    cfg.colsb[1] = 64;
    cfg.rows[2] = 16;
    cfg.colsb[2] = (uint16_t)(B * 4);
    _tile_loadconfig(&cfg);
}

// x [B][K] bf16 -> xp[kb][r][b][2]: pair r of k-block kb for batch row b
void pack_x(const uint16_t *x, int B, int64_t K, std::vector<uint16_t> &xp) {
    const int64_t nkb = K / 32;
    xp.resize((size_t)nkb * 16 * B * 2);
    for (int64_t kb = 0; kb < nkb; ++kb)
        for (int r = 0; r < 16; ++r)
            for (int b = 0; b < B; ++b) {
                uint16_t *d = &xp[(((size_t)kb * 16 + r) * B + b) * 2];
                d[0] = x[b * K + kb * 32 + 2 * r];
                d[1] = x[b * K + kb * 32 + 2 * r + 1];
            }
}

std::atomic<uint64_t> g_job_gen{1};  // bumped for every CPU-lane job (host_gemv_new_job)

struct PackCache {  // per worker thread: x packed once per job
    const uint16_t *x = nullptr;
    int B = 0;
    int64_t K = 0;
    uint64_t gen = 0;
    std::vector<uint16_t> xp;
};
thread_local PackCache t_pack;

const uint16_t *packed_x(const uint16_t *x, int B, int64_t K) {
    PackCache &pc = t_pack;
    const uint64_t gen = g_job_gen.load(std::memory_order_acquire);
    if (pc.x == x && pc.B == B && pc.K == K && pc.gen == gen) return pc.xp.data();
    pc.x = x;
    pc.B = B;
    pc.K = K;
    pc.gen = gen;
    pack_x(x, B, K, pc.xp);
    return pc.xp.data();
}

template <int B>
void rows16(const uint16_t *xp, int64_t K, const uint16_t *W, int64_t r, const float *bias, float *y, int64_t ldy) {
    alignas(64) float c[16 * B];
    _tile_zero(0);
    const int64_t nkb = K / 32;
    const uint16_t *w0 = W + r * K;
    for (int64_t kb = 0; kb < nkb; ++kb) {
        if (kb + 8 < nkb)
            for (int q = 0; q < 16; ++q) _mm_prefetch((const char *)(w0 + q * K + (kb + 8) * 32), _MM_HINT_T0);
        _tile_loadd(1, w0 + kb * 32, K * 2);
        _tile_loadd(2, xp + (size_t)kb * 16 * B * 2, B * 4);
        _tile_dpbf16ps(0, 1, 2);
    }
    _tile_stored(0, c, B * 4);
    for (int q = 0; q < 16; ++q) {
        const float bb = bias ? bias[r + q] : 0.f;
        for (int b = 0; b < B; ++b) y[b * ldy + r + q] = c[q * B + b] + bb;
    }
}

template <int B>
void rows_amx(const uint16_t *x, int64_t K, const uint16_t *W, int64_t r0, int64_t r1, const float *bias,
              float *y, int64_t ldy) {
    config_tiles(B);
    const uint16_t *xp = packed_x(x, B, K);
    int64_t r = r0;
    for (; r + 16 <= r1; r += 16) rows16<B>(xp, K, W, r, bias, y, ldy);
    _tile_release();
    if (r < r1) host_rows_avx512bf16(x, B, K, W, r, r1, bias, y, ldy);
}

bool g_amx_ok = false;

}  // namespace

// A new CPU-lane job begins (its x may reuse a buffer with new contents): repack x lazily.
void host_gemv_new_job() { g_job_gen.fetch_add(1, std::memory_order_acq_rel); }

// Ask the OS for the AMX tile state once per process; false when unavailable.
bool host_amx_enable() {
    static std::once_flag once;
    std::call_once(once, [] {
        __builtin_cpu_init();
        if (!__builtin_cpu_supports("amx-bf16") || !__builtin_cpu_supports("amx-tile") ||
            !__builtin_cpu_supports("avx512bf16"))
            return;
        constexpr long kArchReqXcompPerm = 0x1023, kXfeatureXtiledata = 18;
        g_amx_ok = syscall(SYS_arch_prctl, kArchReqXcompPerm, kXfeatureXtiledata) == 0;
    });
    return g_amx_ok;
}

void host_rows_amx(const uint16_t *x, int batch, int64_t K, const uint16_t *W, int64_t r0, int64_t r1,
                   const float *bias, float *y, int64_t ldy) {
    if (K % 32 != 0 || batch < 1 || batch > 8) {
        host_rows_avx512bf16(x, batch, K, W, r0, r1, bias, y, ldy);
        return;
    }
    switch (batch) {
        case 1: rows_amx<1>(x, K, W, r0, r1, bias, y, ldy); break;
        case 2: rows_amx<2>(x, K, W, r0, r1, bias, y, ldy); break;
        case 3: rows_amx<3>(x, K, W, r0, r1, bias, y, ldy); break;
        case 4: rows_amx<4>(x, K, W, r0, r1, bias, y, ldy); break;
        case 5: rows_amx<5>(x, K, W, r0, r1, bias, y, ldy); break;
        case 6: rows_amx<6>(x, K, W, r0, r1, bias, y, ldy); break;
        case 7: rows_amx<7>(x, K, W, r0, r1, bias, y, ldy); break;
        default: rows_amx<8>(x, K, W, r0, r1, bias, y, ldy); break;
    }
}

}  // namespace hg
