// cpu_lane_prefetch.cpp -- per-core memory parallelism of the CPU lane's B=1 GEMV (development probe).
//
// The CPU lane reads its weight rows once per token; with 14 threads it runs at ~11.4 GB/s per thread,
// close to a plain streaming read on one core, i.e. bound by how many cache-line misses a core keeps in
// flight, not by VDPBF16PS.  This probe times the lane's inner loop (R rows x 32 k per VDPBF16PS step)
// over a weight matrix larger than the LLC under software-prefetch variants (hint level and distance),
// at several thread counts, to see whether prefetching into L2 further ahead raises the per-core rate.
//
//   g++ -O3 -std=c++17 -mavx512f -mavx512bw -mavx512bf16 -pthread cpu_lane_prefetch.cpp -o /tmp/clp
//   /tmp/clp [GB=2] [threads list, e.g. 1,8,14,16]
#include <immintrin.h>
#include <sys/mman.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

constexpr int64_t K = 7168;

// HINT: 0 none, 1 T0, 2 T1, 3 T2, 4 NTA.  DIST in bytes ahead of the current load, per row stream.
template <int R, int HINT, int DIST>
void lane_rows(const uint16_t *x, const uint16_t *W, int64_t r0, int64_t r1, float *y) {
    for (int64_t r = r0; r + R <= r1; r += R) {
        __m512 acc[R];
        for (int i = 0; i < R; ++i) acc[i] = _mm512_setzero_ps();
        const uint16_t *w[R];
        for (int i = 0; i < R; ++i) w[i] = W + (r + i) * K;
        for (int64_t k = 0; k < K; k += 32) {
            __m512i wv[R];
#pragma GCC unroll 16
            for (int i = 0; i < R; ++i) {
                wv[i] = _mm512_loadu_si512((const void *)(w[i] + k));
                if constexpr (HINT == 1) _mm_prefetch((const char *)(w[i] + k) + DIST, _MM_HINT_T0);
                if constexpr (HINT == 2) _mm_prefetch((const char *)(w[i] + k) + DIST, _MM_HINT_T1);
                if constexpr (HINT == 3) _mm_prefetch((const char *)(w[i] + k) + DIST, _MM_HINT_T2);
                if constexpr (HINT == 4) _mm_prefetch((const char *)(w[i] + k) + DIST, _MM_HINT_NTA);
            }
            const __m512i xv = _mm512_loadu_si512((const void *)(x + k));
#pragma GCC unroll 16
            for (int i = 0; i < R; ++i) acc[i] = _mm512_dpbf16_ps(acc[i], (__m512bh)wv[i], (__m512bh)xv);
        }
        for (int i = 0; i < R; ++i) y[r + i] = _mm512_reduce_add_ps(acc[i]);
    }
}

// plain streaming read (the hg_measure probe's loop)
template <int HINT, int DIST>
void readonly(const uint16_t *, const uint16_t *W, int64_t r0, int64_t r1, float *y) {
    const char *c = (const char *)(W + r0 * K);
    const int64_t bytes = (r1 - r0) * K * 2;
    __m512i a0 = _mm512_setzero_si512(), a1 = a0, a2 = a0, a3 = a0;
    for (int64_t i = 0; i + 256 <= bytes; i += 256) {
        if constexpr (HINT == 2) {
            _mm_prefetch(c + i + DIST, _MM_HINT_T1);
            _mm_prefetch(c + i + DIST + 128, _MM_HINT_T1);
        }
        a0 = _mm512_xor_si512(a0, _mm512_loadu_si512(c + i));
        a1 = _mm512_xor_si512(a1, _mm512_loadu_si512(c + i + 64));
        a2 = _mm512_xor_si512(a2, _mm512_loadu_si512(c + i + 128));
        a3 = _mm512_xor_si512(a3, _mm512_loadu_si512(c + i + 192));
    }
    a0 = _mm512_xor_si512(_mm512_xor_si512(a0, a1), _mm512_xor_si512(a2, a3));
    y[r0] = (float)_mm512_reduce_add_epi64(a0);
}

using Fn = void (*)(const uint16_t *, const uint16_t *, int64_t, int64_t, float *);

struct Variant {
    const char *name;
    Fn fn;
};

double run(Fn fn, int threads, const uint16_t *x, const uint16_t *W, int64_t rows, float *y, int reps) {
    // dynamic blocks of 16 rows, like the lane's host_job_run
    double best = 1e30;
    for (int rep = 0; rep < reps; ++rep) {
        std::atomic<int64_t> next{0};
        std::atomic<int> ready{0};
        std::atomic<bool> go{false};
        std::vector<std::thread> ts;
        for (int t = 0; t < threads; ++t)
            ts.emplace_back([&, t] {
                (void)t;
                ready.fetch_add(1);
                while (!go.load(std::memory_order_acquire)) {
                }
                for (;;) {
                    const int64_t b = next.fetch_add(16);
                    if (b >= rows) break;
                    fn(x, W, b, b + 16 < rows ? b + 16 : rows, y);
                }
            });
        while (ready.load() < threads) {
        }
        const auto t0 = std::chrono::steady_clock::now();
        go.store(true, std::memory_order_release);
        for (auto &t : ts) t.join();
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (s < best) best = s;
    }
    return (double)rows * K * 2 / best / 1e9;
}

}  // namespace

int main(int argc, char **argv) {
    const double gb = argc > 1 ? atof(argv[1]) : 2.0;
    std::vector<int> tl = {1, 8, 14, 16};
    if (argc > 2) {
        tl.clear();
        std::string s = argv[2];
        size_t p = 0;
        while (p < s.size()) {
            tl.push_back(atoi(s.c_str() + p));
            p = s.find(',', p);
            if (p == std::string::npos) break;
            ++p;
        }
    }
    const int64_t rows = ((int64_t)(gb * 1e9) / (K * 2)) & ~int64_t(127);
    const size_t bytes = (size_t)rows * K * 2;
    uint16_t *W = (uint16_t *)mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    for (size_t i = 0; i < bytes / 2; ++i) W[i] = (uint16_t)(0x3c00 + (i * 2654435761u >> 20) % 512);
    std::vector<uint16_t> x(K, 0x3f80);
    std::vector<float> y(rows + 64);
    const Variant vs[] = {
        {"read (probe loop)", readonly<0, 0>},
        {"read +T1 4KB", readonly<2, 4096>},
        {"read +T1 16KB", readonly<2, 16384>},
        {"R8 T0 2KB (lane now)", lane_rows<8, 1, 2048>},
        {"R8 none", lane_rows<8, 0, 0>},
        {"R8 T1 2KB", lane_rows<8, 2, 2048>},
        {"R8 T1 4KB", lane_rows<8, 2, 4096>},
        {"R8 T1 8KB", lane_rows<8, 2, 8192>},
        {"R8 T2 4KB", lane_rows<8, 3, 4096>},
        {"R8 NTA 2KB", lane_rows<8, 4, 2048>},
        {"R4 T1 4KB", lane_rows<4, 2, 4096>},
        {"R4 T1 8KB", lane_rows<4, 2, 8192>},
        {"R16 T1 2KB", lane_rows<16, 2, 2048>},
        {"R16 T1 4KB", lane_rows<16, 2, 4096>},
    };
    printf("weights %.2f GB (%lld rows x %lld), best of 3, GB/s (per thread in brackets)\n", bytes / 1e9,
           (long long)rows, (long long)K);
    printf("%-22s", "variant");
    for (int t : tl) printf(" | %4d thr       ", t);
    printf("\n");
    for (const Variant &v : vs) {
        printf("%-22s", v.name);
        for (int t : tl) {
            const double g = run(v.fn, t, x.data(), W, rows, y.data(), 3);
            printf(" | %6.1f (%5.2f)", g, g / t);
            fflush(stdout);
        }
        printf("\n");
    }
    munmap(W, bytes);
    return 0;
}
