// pinlane.cpp -- the pin lane of the asynchronous parameter manager.
//
// HeteGen overlaps three things for a weight that is not page-locked: pinning it ("the CPU
// pin[s] the next weight"), transferring it, and computing (Sec. 4.2-4.3, Fig. 5c, P:227-246;
// Eq. (8)/(9) put T_COM = max(T_PIN, T_TRANS)).  Here a coordinator thread copies each
// pageable chunk into a slot of a bounded pinned staging ring with a small memcpy pool, then
// publishes the slot's tag in mapped host memory; the copy stream waits for that tag with
// cuStreamWaitValue32, DMAs the staging slot to the device ring and writes the slot's `free` tag
// back, which the coordinator waits for before refilling the slot.  Neither the API thread nor the
// copy stream ever blocks on host work they could overlap.
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>

#include "hg_internal.h"

namespace hg {

namespace {
struct PinJob {
    const uint8_t *src;
    int64_t bytes;
    int slot;
    uint32_t tag;
};

struct CopyPart {
    const uint8_t *src;
    uint8_t *dst;
    int64_t bytes;
    int parts;
};

void copy_part(void *a, int w) {
    const CopyPart *cp = (const CopyPart *)a;
    const int64_t per = (cp->bytes / cp->parts + 63) / 64 * 64;
    const int64_t off = (int64_t)w * per;
    if (off < cp->bytes) std::memcpy(cp->dst + off, cp->src + off, (size_t)std::min(per, cp->bytes - off));
    _mm_sfence();  // non-temporal stores of a large memcpy are visible before the tag
}
}  // namespace

struct PinLane {
    ThreadPool *pool = nullptr;
    int threads = 1;
    uint8_t *staging = nullptr;
    int64_t slot_bytes = 0;
    int nslots = 0;
    volatile uint32_t *pinned = nullptr;  // [nslots] written here: staging slot holds tag's bytes
    volatile uint32_t *freed = nullptr;   // [nslots] written by the copy stream after its DMA
    double timeout_s = 60.0;
    std::thread th;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<PinJob> q;
    bool stop = false;
    std::atomic<bool> error{false};
    std::atomic<int64_t> busy_ns{0}, bytes{0};

    void loop() {
        for (;;) {
            PinJob j;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return stop || !q.empty(); });
                if (q.empty()) return;  // stop requested and drained
                j = q.front();
                q.pop_front();
            }
            // the slot's previous occupant (tag - nslots) must have left for the device.  After a
            // timeout the lane is failed: it writes no staging slot any more (one may still be under
            // DMA), but it still publishes every tag so the copy stream's device-side waits drain
            // instead of hanging the GPU; the context reports HG_ETIMEOUT at its next call.
            if (!error && j.tag > (uint32_t)nslots) {
                const uint32_t need = j.tag - (uint32_t)nslots;
                const auto t0 = std::chrono::steady_clock::now();
                for (int spin = 0; (int32_t)(__atomic_load_n(&freed[j.slot], __ATOMIC_ACQUIRE) - need) < 0; ++spin) {
                    _mm_pause();
                    if ((spin & 4095) == 4095) {
                        std::this_thread::yield();
                        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
                            error = true;
                            break;
                        }
                    }
                }
            }
            const auto t1 = std::chrono::steady_clock::now();
            if (!error) {
                CopyPart cp{j.src, staging + (int64_t)j.slot * slot_bytes, j.bytes, threads};
                pool_run(pool, copy_part, &cp);
            }
            // the memcpy pool's writes happen-before the join; the release store publishes them to the
            // copy stream (device memops on mapped memory) or any host reader (tools/tsan)
            __atomic_store_n(&pinned[j.slot], j.tag, __ATOMIC_RELEASE);
            _mm_sfence();
            busy_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t1).count();
            bytes += j.bytes;
        }
    }
};

PinLane *pinlane_create(int threads, uint8_t *staging, int64_t slot_bytes, int nslots, volatile uint32_t *pinned,
                        volatile uint32_t *freed, double timeout_s) {
    PinLane *p = new PinLane;
    p->threads = threads < 1 ? 1 : threads;
    p->pool = pool_create(p->threads, -1);
    p->staging = staging;
    p->slot_bytes = slot_bytes;
    p->nslots = nslots;
    p->pinned = pinned;
    p->freed = freed;
    p->timeout_s = timeout_s;
    p->th = std::thread([p] { p->loop(); });
    return p;
}

void pinlane_destroy(PinLane *p) {
    if (!p) return;
    {
        std::lock_guard<std::mutex> lk(p->mu);
        p->stop = true;
    }
    p->cv.notify_all();
    p->th.join();
    pool_destroy(p->pool);
    delete p;
}

void pinlane_submit(PinLane *p, const void *src, int64_t bytes, int slot, uint32_t tag) {
    {
        std::lock_guard<std::mutex> lk(p->mu);
        p->q.push_back({(const uint8_t *)src, bytes, slot, tag});
    }
    p->cv.notify_one();
}

bool pinlane_error(const PinLane *p) { return p && p->error.load(); }

void pinlane_stats(PinLane *p, double *busy_s, int64_t *bytes, bool reset) {
    if (!p) {
        *busy_s = 0;
        *bytes = 0;
        return;
    }
    *busy_s = p->busy_ns.load() * 1e-9;
    *bytes = p->bytes.load();
    if (reset) {
        p->busy_ns = 0;
        p->bytes = 0;
    }
}

// One-off parallel copy on the lane's pool (hg_measure's V_PIN probe); returns seconds.
double pinlane_copy_timed(PinLane *p, void *dst, const void *src, int64_t bytes) {
    const auto t0 = std::chrono::steady_clock::now();
    CopyPart cp{(const uint8_t *)src, (uint8_t *)dst, bytes, p->threads};
    pool_run(p->pool, copy_part, &cp);
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace hg
