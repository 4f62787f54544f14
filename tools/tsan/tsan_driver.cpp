// tsan_driver.cpp -- ThreadSanitizer run of the library's host-side concurrency (SURVEY 4 tier 4, 5
// "race detection"): the CPU lane's thread pool (post / join / run, many generations, the futex sleep
// path) and the pin lane (coordinator + memcpy pool + tag hand-off), with a "copy engine" thread that
// plays the copy stream: waits for each slot's pinned tag, checks the bytes, then writes its freed tag.
// Built and run by tools/tsan/run.sh (g++ -fsanitize=thread, host only, no CUDA).
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "hg_internal.h"

using namespace hg;

namespace {
struct SumJob {
    const int *data;
    int n;
    std::atomic<long long> sum{0};
    std::atomic<int> next{0};
};
void sum_fn(void *a, int) {
    SumJob *j = (SumJob *)a;
    for (;;) {
        const int i = j->next.fetch_add(64);
        if (i >= j->n) break;
        long long s = 0;
        for (int k = i; k < i + 64 && k < j->n; ++k) s += j->data[k];
        j->sum += s;
    }
}
}  // namespace

int main() {
    int bad = 0;
    // ---- thread pool: 2000 dispatches, some after the workers went to sleep (> 2 ms idle)
    {
        ThreadPool *pool = pool_create(6, -1);
        std::vector<int> data(100000);
        for (size_t i = 0; i < data.size(); ++i) data[i] = (int)(i % 97);
        long long want = 0;
        for (int v : data) want += v;
        for (int it = 0; it < 2000; ++it) {
            SumJob j;
            j.data = data.data();
            j.n = (int)data.size();
            if (it % 2) {
                pool_post(pool, sum_fn, &j);
                pool_join(pool);
            } else {
                pool_run(pool, sum_fn, &j);
            }
            if (j.sum != want) ++bad;
            if (it % 500 == 499) std::this_thread::sleep_for(std::chrono::milliseconds(5));
        }
        pool_destroy(pool);
        printf("pool: %d bad sums\n", bad);
    }
    // ---- pin lane: 4 staging slots, 200 chunks of 64 KB from a "pageable" source
    {
        const int nslots = 4, nchunks = 200;
        const int64_t slot_bytes = 64 << 10;
        std::vector<uint8_t> staging((size_t)nslots * slot_bytes), src((size_t)nchunks * slot_bytes);
        for (size_t i = 0; i < src.size(); ++i) src[i] = (uint8_t)(i * 131 + 7);
        std::vector<uint32_t> flags(2 * nslots, 0);
        volatile uint32_t *pinned = flags.data(), *freed = flags.data() + nslots;
        PinLane *lane = pinlane_create(3, staging.data(), slot_bytes, nslots, pinned, freed, 30.0);
        std::atomic<int> copy_bad{0};
        std::thread engine([&] {  // the copy stream: wait pinned >= tag, read the slot, free it
            for (int c = 0; c < nchunks; ++c) {
                const int slot = c % nslots;
                const uint32_t tag = (uint32_t)(c + 1);
                while ((int32_t)(__atomic_load_n(&pinned[slot], __ATOMIC_ACQUIRE) - tag) < 0) std::this_thread::yield();
                if (std::memcmp(staging.data() + (size_t)slot * slot_bytes, src.data() + (size_t)c * slot_bytes,
                                (size_t)slot_bytes) != 0)
                    ++copy_bad;
                __atomic_store_n(&freed[slot], tag, __ATOMIC_RELEASE);
            }
        });
        for (int c = 0; c < nchunks; ++c)
            pinlane_submit(lane, src.data() + (size_t)c * slot_bytes, slot_bytes, c % nslots, (uint32_t)(c + 1));
        engine.join();
        double busy;
        int64_t bytes;
        pinlane_stats(lane, &busy, &bytes, false);
        printf("pin lane: %d bad chunks, %lld bytes, error %d\n", copy_bad.load(), (long long)bytes,
               (int)pinlane_error(lane));
        bad += copy_bad.load() + (bytes != (int64_t)nchunks * slot_bytes) + pinlane_error(lane);
        pinlane_destroy(lane);
    }
    printf("%s\n", bad ? "FAIL" : "OK");
    return bad ? 1 : 0;
}
