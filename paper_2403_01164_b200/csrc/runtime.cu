// runtime.cu -- the heterogeneous offloaded linear on one B200.
//
// Per linear (Fig. 5c "hybrid heterogeneous parallelism"):
//   a2  x -> pinned host bounce (D2H on the caller's stream, event ev_x)
//   a3  resident GEMV over W_dev rows [0, n_res)                       (HBM-bound)
//   a4  streamed rows: the copy stream moves chunk c of W_host into a slot of a
//       device ring (cudaMemcpyAsync, copy engine) while the compute stream
//       runs the GEMV of chunk c-1; per-slot events order arrival -> GEMV ->
//       slot reuse.  The copy stream runs ahead across linears (prefetching,
//       P:127; "pin the next weight in the upcoming layer").
//   a5  CPU rows: once x is on the host, the thread pool computes them
//       ("while CPU computation is underway, model parameters are
//       conveyed to the GPU")
//   a6  join: y_cpu -> device, added with bias into its columns of y (concat)
//   a7  layer glue on the GPU between linears
//   a8  (P>1) all-gather of the row shards over NVLink (NCCL)
#include <cuda_runtime.h>
#include <immintrin.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "hg.h"
#include "hg_internal.h"

namespace hg {

static thread_local char g_err[512] = "";

hg_status set_error(hg_status st, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return st;
}

namespace {

using clk = std::chrono::steady_clock;
inline double secs(clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double>(b - a).count();
}

struct ChunkReq {
    const uint8_t *src;
    int64_t bytes;
    bool operator==(const ChunkReq &o) const { return src == o.src && bytes == o.bytes; }
};

struct Inflight {
    ChunkReq req;
    int slot;
    int64_t seq;
};

// cuStreamWaitValue32 / cuStreamWriteValue32 (driver entry points; stream memory operations)
typedef int (*memop_fn_t)(void *stream, unsigned long long addr, uint32_t value, unsigned int flags);
constexpr unsigned kWaitGeq = 0x0;      // CU_STREAM_WAIT_VALUE_GEQ: (int32)(*addr - value) >= 0
constexpr unsigned kWriteDefault = 0x0; // CU_STREAM_WRITE_VALUE_DEFAULT: fence before the write
memop_fn_t g_wait_value = nullptr, g_write_value = nullptr;

bool load_memops() {
    static int state = -1;
    if (state >= 0) return state == 1;
    void *w = nullptr, *v = nullptr;
    cudaDriverEntryPointQueryResult q1, q2;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &w, cudaEnableDefault, &q1) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess &&
        cudaGetDriverEntryPoint("cuStreamWriteValue32", &v, cudaEnableDefault, &q2) == cudaSuccess &&
        q2 == cudaDriverEntryPointSuccess) {
        g_wait_value = (memop_fn_t)w;
        g_write_value = (memop_fn_t)v;
        state = 1;
    } else {
        cudaGetLastError();
        state = 0;
    }
    return state == 1;
}

struct HostJob {
    host_rows_fn fn;
    const uint16_t *x;
    int batch;
    int64_t K, n;
    const uint16_t *W;
    const float *bias;
    float *y;
    int64_t ldy;
    int64_t block;
    std::atomic<int64_t> next;
};

void host_job_run(void *a, int) {
    HostJob *j = (HostJob *)a;
    const int64_t nblk = (j->n + j->block - 1) / j->block;
    for (;;) {
        const int64_t b = j->next.fetch_add(1, std::memory_order_relaxed);
        if (b >= nblk) break;
        const int64_t r0 = b * j->block;
        const int64_t r1 = r0 + j->block < j->n ? r0 + j->block : j->n;
        j->fn(j->x, j->batch, j->K, j->W, r0, r1, j->bias, j->y, j->ldy);
    }
}

// Fig. 5a transfer thread (hg_config.strategy = HG_STRATEGY_NAIVE): chunks of a pageable weight are
// copied straight from the un-pinned rows with cudaMemcpyAsync -- the driver stages them through its
// own pinned buffer and the call returns only when the source is consumed -- so the copies run on this
// thread and its own stream, beside the CPU lane.  Per chunk, in order on the stream: wait until the
// ring slot's previous occupant was consumed, copy, write the slot's arrival tag.
struct NaiveLane {
    struct Job {
        const uint32_t *consumed;
        uint32_t wait_val;  // 0: no wait
        uint32_t *arrived;
        uint32_t arrived_val;
        void *dst;
        const void *src;
        int64_t bytes;
    };
    int device = 0;
    cudaStream_t st = nullptr;
    std::thread th;
    std::mutex mu;
    std::condition_variable cv, idle;
    std::deque<Job> q;
    int busy = 0;
    bool stop = false;
    std::atomic<int> err{0};
    std::atomic<int64_t> busy_ns{0}, bytes{0};  // host time inside the staged copies (the link time)

    void loop() {
        cudaSetDevice(device);
        for (;;) {
            Job j;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return stop || !q.empty(); });
                if (q.empty()) return;
                j = q.front();
                q.pop_front();
                ++busy;
            }
            if (!err) {
                int e = 0;
                if (j.wait_val) e = g_wait_value((void *)st, (unsigned long long)(uintptr_t)j.consumed, j.wait_val, kWaitGeq);
                const auto t0 = std::chrono::steady_clock::now();
                if (!e && cudaMemcpyAsync(j.dst, j.src, (size_t)j.bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) e = 1;
                busy_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
                bytes += j.bytes;
                if (!e) e = g_write_value((void *)st, (unsigned long long)(uintptr_t)j.arrived, j.arrived_val, kWriteDefault);
                if (e) err = 1;
            }
            {
                std::lock_guard<std::mutex> lk(mu);
                --busy;
            }
            idle.notify_all();
        }
    }
    void submit(const Job &j) {
        {
            std::lock_guard<std::mutex> lk(mu);
            q.push_back(j);
        }
        cv.notify_one();
    }
    void drain() {  // every submitted copy has been enqueued on the stream
        std::unique_lock<std::mutex> lk(mu);
        idle.wait(lk, [&] { return q.empty() && busy == 0; });
    }
};

NaiveLane *naive_create(int device) {
    NaiveLane *n = new NaiveLane;
    n->device = device;
    if (cudaStreamCreateWithFlags(&n->st, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        delete n;
        return nullptr;
    }
    n->th = std::thread([n] { n->loop(); });
    return n;
}

void naive_destroy(NaiveLane *n) {
    if (!n) return;
    {
        std::lock_guard<std::mutex> lk(n->mu);
        n->stop = true;
    }
    n->cv.notify_all();
    n->th.join();
    cudaStreamSynchronize(n->st);
    cudaStreamDestroy(n->st);
    delete n;
}

// Parallel memcpy on a thread pool (Fig. 5b's blocking pin runs on the CPU lane's own threads).
struct PoolCopy {
    uint8_t *dst;
    const uint8_t *src;
    int64_t bytes;
    int parts;
};
void pool_copy_part(void *a, int w) {
    const PoolCopy *pc = (const PoolCopy *)a;
    const int64_t per = (pc->bytes / pc->parts + 63) / 64 * 64;
    const int64_t off = (int64_t)w * per;
    if (off < pc->bytes) std::memcpy(pc->dst + off, pc->src + off, (size_t)std::min(per, pc->bytes - off));
    _mm_sfence();
}

}  // namespace
}  // namespace hg
struct hg_ctx;
namespace hg {
namespace {
host_rows_fn host_fn_for(hg_ctx *c, int batch);
}  // namespace
}  // namespace hg
namespace hg {
namespace {

// One heterogeneous linear, internal form.
struct Lin {
    hg_plan_t plan;
    const void *x;      // device bf16 [B, K]
    const void *W_dev;  // device [n_res, K]
    const uint8_t *W_host;  // pinned [N - n_res, K]
    const float *bias;  // device [N] or null
    float *y;           // device, row stride ldy
    int64_t ldy;
};

}  // namespace
}  // namespace hg

using namespace hg;

struct hg_ctx {
    int device = -1;
    hg_config cfg;
    ThreadPool *pool = nullptr;
    host_rows_fn host_fn = nullptr;
    int amx_min_batch = 0;  // batches >= this use AMX tiles on the CPU lane (0: never)
    bool error = false;

    // ---- CUDA resources (device contexts only)
    cudaStream_t copy = nullptr;
    uint8_t *ring = nullptr;
    int64_t slot_bytes = 0;
    int nslots = 0;
    std::vector<cudaEvent_t> ev_arrived, ev_free;
    std::vector<char> slot_used;
    std::deque<Inflight> inflight;
    int64_t next_seq = 0;
    int64_t prebound = 0;   // upcoming future chunks already bound to an enqueued GEMV (tags mode)
    bool tags = false;      // cfg.handshake == 1 and stream memory operations available
    bool tc_stream = true;  // tcgen05 batches: one persistent launch per linear (HG_TC_STREAM=0: per chunk)
    uint32_t *tagmem = nullptr;  // device: arrived[nslots] consumed[nslots] slot_cnt[nslots] err[4] gbar[4 + kGroupCounters]
    uint32_t *arrived = nullptr, *consumed = nullptr, *slot_cnt = nullptr, *err = nullptr, *gbar = nullptr;
    volatile uint32_t *err_host = nullptr;  // mapped pinned [4]: host view of `err` (read without a sync)
    std::vector<ChunkReq> future;
    size_t fpos = 0;
    bool fwrap = false;

    uint16_t *x_host = nullptr;   // pinned [max_batch, max_k]
    // CPU-lane results: two mapped pinned buffers [max_batch, max_n] used alternately; the join
    // kernel reads them in place (zero-copy).  A cudaMemcpyAsync H2D here would queue behind every
    // chunk copy already in the copy engine's queue (measured: 2 GiB queued -> 39 ms), draining the
    // link's run-ahead at every linear boundary.
    float *ycpu_host[2] = {nullptr, nullptr};
    float *ycpu_map[2] = {nullptr, nullptr};  // device addresses of the same buffers
    float *ycpu_dev = nullptr;    // device [max_batch, max_n] (HG_JOIN_MEMCPY=1 A/B path only)
    int ybuf = 0;
    cudaEvent_t ev_x = nullptr, ev_ycpu[2] = {nullptr, nullptr}, ev_done = nullptr;
    std::vector<uint16_t> hh, hh1, xchk;          // mirrored glue: host residual stream, check buffer
    // mirrored glue ring (kMirrorRing linears deep): device y per linear, its host copy (mapped
    // pinned; the CPU lane's rows land there too), and the events ordering them
    static constexpr int kMirrorRing = 8;
    float *yring = nullptr;                        // device [kMirrorRing][max_batch * max_n]
    float *yhost[kMirrorRing] = {};                // mapped pinned [max_batch * max_n]
    float *ymap[kMirrorRing] = {};
    cudaEvent_t ev_g[kMirrorRing] = {}, ev_yg[kMirrorRing] = {}, ev_use[kMirrorRing] = {};
    cudaStream_t d2h = nullptr;                    // side stream for the GPU rows' D2H
    // pin lane (pageable weights, Sec. 4.3): pinned staging ring + mapped tag words
    PinLane *pin = nullptr;
    NaiveLane *naive = nullptr;  // strategy NAIVE: transfer thread + stream for pageable chunks
    uint8_t *staging = nullptr;
    int nstage = 0;
    uint32_t *pinflags = nullptr;       // mapped host: pinned[nstage], freed[nstage]
    uint32_t *pinflags_dev = nullptr;   // device address of the same words (stream memops)
    int64_t pin_seq = 0;
    uint32_t *trace = nullptr;                     // HG_SYNC_DEBUG=3: mapped host trace words
    uint64_t trace_seq = 0;
    struct TraceLin { uint32_t id; int64_t seq0, n_chunks, n_res, n_str, K; };
    std::vector<TraceLin> trace_lin;
    cudaStream_t last_stream = nullptr;
    bool have_last = false;

    float *ws = nullptr;
    int64_t ws_floats = 0;
    int *counters = nullptr;
    int64_t n_counters = 0;
    float *sink = nullptr;

    // layer scratch
    void *act = nullptr;
    float *yscr = nullptr;
    void *h1 = nullptr;
    int64_t act_elems = 0, yscr_elems = 0, h1_elems = 0;

    // multi-GPU: NCCL all-gather (hg_dist_init) or the peer-memory exchange (hg_peer_open, peer.cu)
    Dist *dist = nullptr;
    PeerGroup *peer = nullptr, *peer_pending = nullptr;
    float *ylring = nullptr;  // P > 1 mirrored stack: this rank's rows per linear, device [kMirrorRing][...]
    int64_t hseq = 0;         // linears run through the mirrored stack so far (host-segment index)
    std::vector<void *> retired;  // outgrown scratch buffers (freed by hg_destroy)
    float *ylocal = nullptr, *gbuf = nullptr;
    int64_t ylocal_elems = 0, gbuf_elems = 0;

    // stats
    hg_stats_t st;
    std::vector<cudaEvent_t> tev;
    size_t tev_used = 0;
    std::vector<std::pair<size_t, size_t>> copy_ev, gemv_ev;
    std::vector<int64_t> copy_bytes;  // bytes of each timed chunk copy (copy_ev order)
    cudaEvent_t ev_call0 = nullptr, ev_call1 = nullptr;
    bool call_timed = false;
    bool stats_open = false;  // ev_call0 recorded since the last reset
};

namespace hg {
namespace {
int nranks_of(const hg_ctx *c) { return c->peer ? peer_nranks(c->peer) : dist_nranks(c->dist); }
host_rows_fn host_fn_for(hg_ctx *c, int batch) {
    return (c->amx_min_batch > 0 && batch >= c->amx_min_batch) ? host_rows_amx : c->host_fn;
}
}  // namespace
}  // namespace hg

namespace {

// ---------------------------------------------------------------- helpers
#define HG_CK(ctx, expr)                                                                     \
    do {                                                                                     \
        cudaError_t e_ = (cudaError_t)(expr);                                                \
        if (e_ != cudaSuccess) {                                                             \
            (ctx)->error = true;                                                             \
            return set_error(HG_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,            \
                             cudaGetErrorString(e_));                                        \
        }                                                                                    \
    } while (0)

#define HG_TRY(expr)                      \
    do {                                  \
        hg_status s_ = (expr);            \
        if (s_ != HG_OK) return s_;       \
    } while (0)

inline bool aligned(const void *p, size_t a) { return ((uintptr_t)p % a) == 0; }

hg_status check_ptr(hg_ctx *c, const void *p, bool want_device, const char *what) {
    if (!p) return set_error(HG_EINVAL, "%s is NULL", what);
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (!want_device && c->cfg.pageable) return HG_OK;
        return set_error(want_device ? HG_ENOTDEVICE : HG_ENOTPINNED, "%s: %s", what,
                         cudaGetErrorString(e));
    }
    if (want_device) {
        if (at.type != cudaMemoryTypeDevice || at.device != c->device)
            return set_error(HG_ENOTDEVICE, "%s is not device memory of device %d", what, c->device);
    } else {
        if (at.type == cudaMemoryTypeUnregistered && c->cfg.pageable) return HG_OK;  // pin lane stages it
        if (at.type != cudaMemoryTypeHost)
            return set_error(HG_ENOTPINNED, "%s is not page-locked host memory", what);
    }
    return HG_OK;
}

// true when p is host memory that is not page-locked (pageable); such weights need the pin lane
bool is_pageable(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
}

hg_status kerr(hg_ctx *c, int e, const char *what) {
    if (e != 0) {
        c->error = true;
        return set_error(HG_ECUDA, "%s: %s", what, cudaGetErrorString((cudaError_t)e));
    }
    return HG_OK;
}

// HG_SYNC_DEBUG=3: GEMV launches record their id and CTA progress in mapped host words.
volatile uint32_t *dbg_trace(hg_ctx *c) {
    static const int mode = getenv("HG_SYNC_DEBUG") ? atoi(getenv("HG_SYNC_DEBUG")) : 0;
    if (mode != 3) return nullptr;
    if (!c->trace) {
        if (cudaHostAlloc((void **)&c->trace, 64, cudaHostAllocMapped) != cudaSuccess) return nullptr;
        std::memset(c->trace, 0, 64);
    }
    return c->trace;
}

void dbg_trace_report(hg_ctx *c) {
    if (!c->trace) return;
    const uint32_t id = c->trace[1], ctas_done = c->trace[2];
    fprintf(stderr, "hg trace: last GEMV started id=%u, last past its groups (CTA 0) id=%u, launches=%zu\n", id,
            ctas_done, c->trace_lin.size());
    for (const auto &t : c->trace_lin)
        if (t.id + 3 >= id && t.id <= id + 1)
            fprintf(stderr, "  id %u: seq0=%lld n_chunks=%lld n_res=%lld n_str=%lld K=%lld (slots %lld..)\n", t.id,
                    (long long)t.seq0, (long long)t.n_chunks, (long long)t.n_res, (long long)t.n_str, (long long)t.K,
                    (long long)(t.seq0 % c->nslots));
}

// A tag wait inside a kernel that timed out leaves err != 0 (mapped host word; also polled by
// begin_call / end_call).
hg_status check_device_error(hg_ctx *c) {
    if (!c->err_host) return HG_OK;
    const uint32_t e = c->err_host[0];
    if (e) {
        c->error = true;
        return set_error(HG_ETIMEOUT, "a GEMV waited longer than %.1f s for a streamed chunk", c->cfg.timeout_s);
    }
    return HG_OK;
}

hg_status wait_event(hg_ctx *c, cudaEvent_t ev, double *waited) {
    const auto t0 = clk::now();
    for (int spin = 0;; ++spin) {
        cudaError_t e = cudaEventQuery(ev);
        if (e == cudaSuccess) break;
        if (e != cudaErrorNotReady) {
            c->error = true;
            return set_error(HG_ECUDA, "event wait: %s", cudaGetErrorString(e));
        }
        for (int i = 0; i < 16; ++i) _mm_pause();
        if ((spin & 1023) == 1023 && secs(t0, clk::now()) > c->cfg.timeout_s) {
            c->error = true;
            if (getenv("HG_PEER_DEBUG"))
                fprintf(stderr, "hg: event wait timeout: next_seq %lld inflight %zu (front seq %lld) prebound %lld "
                        "fpos %zu/%zu err %u\n", (long long)c->next_seq, c->inflight.size(),
                        c->inflight.empty() ? -1ll : (long long)c->inflight.front().seq, (long long)c->prebound, c->fpos,
                        c->future.size(), c->err_host ? c->err_host[0] : 0u);
            return set_error(HG_ETIMEOUT, "event wait exceeded %.1f s", c->cfg.timeout_s);
        }
    }
    if (waited) *waited += secs(t0, clk::now());
    return HG_OK;
}

// timing events (collect_stats)
cudaEvent_t tev_get(hg_ctx *c, size_t *idx) {
    if (c->tev_used == c->tev.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        c->tev.push_back(e);
    }
    *idx = c->tev_used;
    return c->tev[c->tev_used++];
}

// ---------------------------------------------------------------- chunk ring
hg_status memop(hg_ctx *c, memop_fn_t fn, cudaStream_t s, const uint32_t *addr, uint32_t v, unsigned flags) {
    const int e = fn((void *)s, (unsigned long long)(uintptr_t)addr, v, flags);
    if (e != 0) {
        c->error = true;
        return set_error(HG_ECUDA, "stream memory operation failed (CUresult %d)", e);
    }
    return HG_OK;
}

hg_status ensure_pinlane(hg_ctx *c) {
    if (c->pin) return HG_OK;
    c->nstage = (int)std::max<int64_t>(2, c->cfg.staging_bytes / c->slot_bytes);
    HG_CK(c, cudaHostAlloc((void **)&c->staging, (size_t)c->nstage * c->slot_bytes, cudaHostAllocDefault));
    HG_CK(c, cudaHostAlloc((void **)&c->pinflags, (size_t)2 * c->nstage * 4, cudaHostAllocMapped));
    std::memset(c->pinflags, 0, (size_t)2 * c->nstage * 4);
    HG_CK(c, cudaHostGetDevicePointer((void **)&c->pinflags_dev, c->pinflags, 0));
    c->pin = pinlane_create(c->cfg.pin_threads, c->staging, c->slot_bytes, c->nstage, c->pinflags,
                            c->pinflags + c->nstage, c->cfg.timeout_s);
    return HG_OK;
}

// Enqueue chunk `r` into the next ring slot on the copy stream.  `bound`: a GEMV that consumes
// it is already enqueued (tags mode), so it is not tracked as in flight.
hg_status issue_copy(hg_ctx *c, const ChunkReq &r, bool bound = false) {
    const int64_t seq = c->next_seq;
    const int slot = (int)(seq % c->nslots);
    const bool pageable = c->cfg.pageable && is_pageable(r.src);
    if (pageable && c->cfg.strategy == HG_STRATEGY_NAIVE) {
        // Fig. 5a: the transfer thread copies straight from the pageable rows on its own stream; the
        // slot-reuse wait and the arrival tag travel with the copy, in order on that stream
        if (!c->tags) return set_error(HG_EUNSUPPORTED, "pageable weights need the device-tag pipeline");
        if (!c->naive && !(c->naive = naive_create(c->device))) {
            c->error = true;
            return set_error(HG_ECUDA, "cannot create the naive-strategy transfer thread");
        }
        NaiveLane::Job j;
        j.consumed = c->consumed + slot;
        j.wait_val = seq >= c->nslots ? (uint32_t)(seq - c->nslots + 1) : 0u;
        j.arrived = c->arrived + slot;
        j.arrived_val = (uint32_t)(seq + 1);
        j.dst = c->ring + (int64_t)slot * c->slot_bytes;
        j.src = r.src;
        j.bytes = r.bytes;
        c->naive->submit(j);
        c->slot_used[slot] = 1;
        if (!bound) c->inflight.push_back({r, slot, seq});
        ++c->next_seq;
        return HG_OK;
    }
    if (c->tags) {
        // The slot's previous occupant (seq - nslots) must have been drained by its GEMV.  ev_free
        // follows that GEMV (or the drop): when the host already sees it complete, the device-side
        // wait (which costs the copy engine a few microseconds) is skipped.
        if (seq >= c->nslots) {
            const cudaError_t q = cudaEventQuery(c->ev_free[slot]);
            if (q != cudaSuccess) {
                if (q != cudaErrorNotReady) HG_CK(c, q);
                HG_TRY(memop(c, g_wait_value, c->copy, c->consumed + slot, (uint32_t)(seq - c->nslots + 1),
                             kWaitGeq));
            }
        }
    } else if (c->slot_used[slot]) {
        HG_CK(c, cudaStreamWaitEvent(c->copy, c->ev_free[slot], 0));
    }
    size_t i0 = 0, i1 = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->cfg.collect_stats) {
        e0 = tev_get(c, &i0);
        if (e0) HG_CK(c, cudaEventRecord(e0, c->copy));
    }
    const void *src = r.src;
    int pslot = -1;
    uint32_t ptag = 0;
    if (pageable) {  // pageable chunk -> pinned staging slot
        if (!c->tags) return set_error(HG_EUNSUPPORTED, "pageable weights need the device-tag pipeline");
        HG_TRY(ensure_pinlane(c));
        const int64_t ps = c->pin_seq++;
        pslot = (int)(ps % c->nstage);
        ptag = (uint32_t)(ps + 1);
        src = c->staging + (int64_t)pslot * c->slot_bytes;
        if (c->cfg.strategy == HG_STRATEGY_PINNED_BLOCKING) {
            // Fig. 5b: pin now, on the CPU lane's own threads, before anything else of this linear runs
            // (the caller posts the CPU rows only after the linear's chunks are issued); the staging
            // slot's previous DMA must have left it (freed tag, written by the copy stream)
            if (ps >= c->nstage) {
                const uint32_t need = (uint32_t)(ps - c->nstage + 1);
                const auto t0 = clk::now();
                for (int spin = 0; (int32_t)(__atomic_load_n(&c->pinflags[c->nstage + pslot], __ATOMIC_ACQUIRE) - need) < 0;
                     ++spin) {
                    _mm_pause();
                    if ((spin & 4095) == 4095 && secs(t0, clk::now()) > c->cfg.timeout_s) {
                        c->error = true;
                        return set_error(HG_ETIMEOUT, "pinned-blocking: staging slot not freed within %.1f s",
                                         c->cfg.timeout_s);
                    }
                }
            }
            const auto t1 = clk::now();
            PoolCopy pc{(uint8_t *)src, (const uint8_t *)r.src, r.bytes, pool_size(c->pool)};
            pool_run(c->pool, pool_copy_part, &pc);
            c->st.pin_busy_s += secs(t1, clk::now());
            c->st.bytes_pinned += r.bytes;
        } else {  // Fig. 5c: the pin lane pins ahead; the copy stream waits for the slot's pinned tag
            pinlane_submit(c->pin, r.src, r.bytes, pslot, ptag);
            HG_TRY(memop(c, g_wait_value, c->copy, c->pinflags_dev + pslot, ptag, kWaitGeq));
        }
    }
    HG_CK(c, cudaMemcpyAsync(c->ring + (int64_t)slot * c->slot_bytes, src, (size_t)r.bytes,
                             cudaMemcpyHostToDevice, c->copy));
    if (pslot >= 0)  // the staging slot may be refilled
        HG_TRY(memop(c, g_write_value, c->copy, c->pinflags_dev + c->nstage + pslot, ptag, kWriteDefault));
    if (c->tags) HG_TRY(memop(c, g_write_value, c->copy, c->arrived + slot, (uint32_t)(seq + 1), kWriteDefault));
    else HG_CK(c, cudaEventRecord(c->ev_arrived[slot], c->copy));
    if (c->cfg.collect_stats && e0) {
        e1 = tev_get(c, &i1);
        if (e1) {
            HG_CK(c, cudaEventRecord(e1, c->copy));
            c->copy_ev.push_back({i0, i1});
            c->copy_bytes.push_back(r.bytes);
        }
    }
    c->slot_used[slot] = 1;
    if (!bound) c->inflight.push_back({r, slot, seq});
    ++c->next_seq;
    return HG_OK;
}

// Give up prefetched chunks nobody will consume (the call sequence changed): release their slots.
hg_status drop_front(hg_ctx *c) {
    const Inflight &f = c->inflight.front();
    if (c->tags) HG_TRY(memop(c, g_write_value, c->copy, c->consumed + f.slot, (uint32_t)(f.seq + 1), kWriteDefault));
    HG_CK(c, cudaEventRecord(c->ev_free[f.slot], c->copy));
    c->inflight.pop_front();
    return HG_OK;
}

hg_status drop_inflight(hg_ctx *c) {
    while (!c->inflight.empty()) HG_TRY(drop_front(c));
    return HG_OK;
}

bool future_next(hg_ctx *c, ChunkReq *out) {
    if (c->future.empty()) return false;
    if (c->fpos >= c->future.size()) {
        if (!c->fwrap) return false;
        c->fpos = 0;
    }
    *out = c->future[c->fpos++];
    return true;
}

hg_status pump(hg_ctx *c) {
    ChunkReq r;
    while (c->prebound > 0) {  // chunks an enqueued GEMV waits for: issue unconditionally
        if (!future_next(c, &r)) return set_error(HG_ESTATE, "bound chunk missing from the schedule");
        HG_TRY(issue_copy(c, r, true));
        --c->prebound;
    }
    // speculative run-ahead into later linears: the hybrid strategy's "pin the next weight";
    // the naive and pinned-blocking strategies (Fig. 5a/5b) move a linear's rows only while it runs
    if (c->cfg.pageable && c->cfg.strategy != HG_STRATEGY_HYBRID) return HG_OK;
    while ((int)c->inflight.size() < c->nslots && future_next(c, &r)) HG_TRY(issue_copy(c, r));
    return HG_OK;
}

// Tags mode: bind the chunks of one linear to the GEMV about to be enqueued.  They must occupy
// consecutive sequence numbers (the kernel derives slot = (seq0 + c) % nslots): the in-flight
// prefix followed by the next entries of the schedule.  Anything else is dropped and the
// schedule restarts with this linear.
hg_status bind_chunks(hg_ctx *c, const std::vector<ChunkReq> &mine, int64_t *seq0) {
    const size_t n = mine.size();
    size_t m = std::min(n, c->inflight.size());
    bool ok = true;
    for (size_t i = 0; i < m && ok; ++i) ok = c->inflight[i].req == mine[i];
    if (ok && m < n) {  // the rest must be next in the schedule
        size_t pos = c->fpos;
        for (size_t i = m; i < n && ok; ++i) {
            if (pos >= c->future.size()) {
                if (!c->fwrap || c->future.empty()) { ok = false; break; }
                pos = 0;
            }
            ok = c->future[pos++] == mine[i];
        }
    }
    if (!ok) {
        HG_TRY(drop_inflight(c));
        c->future = mine;
        c->fpos = 0;
        c->fwrap = false;
        m = 0;
    }
    *seq0 = m > 0 ? c->inflight.front().seq : c->next_seq;
    for (size_t i = 0; i < m; ++i) c->inflight.pop_front();
    c->prebound += (int64_t)(n - m);
    return HG_OK;
}

// The slot holding `r`, with `stream` ordered after its arrival.
hg_status acquire(hg_ctx *c, const ChunkReq &r, cudaStream_t stream, int *slot) {
    while (!c->inflight.empty() && !(c->inflight.front().req == r)) HG_TRY(drop_front(c));
    int64_t seq = 0;
    if (c->inflight.empty()) {
        // not prefetched: the planned sequence diverged -> restart it here
        c->future.clear();
        c->fpos = 0;
        HG_TRY(issue_copy(c, r));
    }
    *slot = c->inflight.front().slot;
    seq = c->inflight.front().seq;
    if (c->tags) HG_TRY(memop(c, g_wait_value, stream, c->arrived + *slot, (uint32_t)(seq + 1), kWaitGeq));
    else HG_CK(c, cudaStreamWaitEvent(stream, c->ev_arrived[*slot], 0));
    return HG_OK;
}

hg_status release(hg_ctx *c, int slot, cudaStream_t stream) {
    if (c->tags)
        HG_TRY(memop(c, g_write_value, stream, c->consumed + slot, (uint32_t)(c->inflight.front().seq + 1),
                     kWriteDefault));
    HG_CK(c, cudaEventRecord(c->ev_free[slot], stream));
    c->inflight.pop_front();
    return HG_OK;
}

void push_chunks(std::vector<ChunkReq> &v, const hg_plan_t &p, const void *W_host) {
    const uint8_t *base = (const uint8_t *)W_host;
    const int64_t row = 2 * p.K;
    for (int64_t i = 0; i < p.n_chunks; ++i) {
        const int64_t r0 = i * p.chunk_rows;
        const int64_t r1 = (i + 1) * p.chunk_rows < p.n_str ? (i + 1) * p.chunk_rows : p.n_str;
        v.push_back({base + r0 * row, (r1 - r0) * row});
    }
}

void set_future(hg_ctx *c, std::vector<ChunkReq> &&list, bool wrap) {
    if (c->cfg.stream_mode == 1) {  // zero-copy streaming: nothing for the copy engine
        c->future.clear();
        c->fpos = 0;
        c->fwrap = false;
        return;
    }
    if (wrap && c->fwrap && list.size() == c->future.size() &&
        std::equal(list.begin(), list.end(), c->future.begin()))
        return;  // same stack as last call: keep streaming where we are
    c->future = std::move(list);
    c->fpos = 0;
    c->fwrap = wrap;
}

// ---------------------------------------------------------------- GEMV launch
hg_status gemv(hg_ctx *c, const void *x, int B, int64_t K, const void *W, int64_t n,
               const float *bias, float *y, int64_t ldy, cudaStream_t s) {
    if (n <= 0) return HG_OK;
    if (gemv_ws_floats(n, K, B) > c->ws_floats || gemv_counters(n, K, B) > c->n_counters)
        return set_error(HG_EINVAL, "GEMV of %lld rows x K=%lld exceeds the context workspace "
                                    "(raise max_n / max_k)", (long long)n, (long long)K);
    size_t i0 = 0, i1 = 0;
    cudaEvent_t e0 = nullptr;
    if (c->cfg.collect_stats && (e0 = tev_get(c, &i0))) HG_CK(c, cudaEventRecord(e0, s));
    HG_TRY(kerr(c, launch_gemv(x, B, K, W, n, bias, y, ldy, c->ws, c->counters, c->gbar, c->err, s), "gemv launch"));
    c->st.gpu_launches++;
    if (e0) {
        cudaEvent_t e1 = tev_get(c, &i1);
        if (e1) {
            HG_CK(c, cudaEventRecord(e1, s));
            c->gemv_ev.push_back({i0, i1});
        }
    }
    return HG_OK;
}

// ---------------------------------------------------------------- one linear
hg_status stream_guard(hg_ctx *c, cudaStream_t s) {
    if (c->have_last && c->last_stream != s) HG_CK(c, cudaStreamWaitEvent(s, c->ev_done, 0));
    c->last_stream = s;
    c->have_last = true;
    return HG_OK;
}

// GPU lanes of one linear: a3 resident GEMV, a4 streamed chunk GEMVs.
hg_status enqueue_gpu_lanes(hg_ctx *c, const Lin &L, cudaStream_t s) {
    const hg_plan_t &p = L.plan;
    const int B = (int)p.batch;
    const int64_t K = p.K;
    const bool direct = c->cfg.stream_mode == 1 && !gemv_use_tc(B, K);
    // tcgen05 batches take the persistent per-linear launch too when the linear's sources fit
    // its parameter block (resident + <= 16 chunks) and no chunk reuses a slot of the same launch
    const bool tc = gemv_use_tc(B, K);
    const bool tc_stream = tc && c->tags && c->tc_stream &&
                           gemv_tc_stream_ok(p.n_res, p.n_str > 0 ? p.n_chunks : 0) && p.n_chunks <= c->nslots;
    if ((c->tags || direct) && (!tc || tc_stream)) {
        // a3 + a4 in ONE persistent launch: resident rows, then each chunk as its arrival tag lands
        // (stream_mode 1: the streamed rows are read by the kernel itself over the link, zero-copy)
        std::vector<ChunkReq> mine;
        int64_t seq0 = 0;
        if (!direct) {
            push_chunks(mine, p, L.W_host);
            if (p.n_str > 0) HG_TRY(bind_chunks(c, mine, &seq0));
        }
        const int64_t n = p.n_res + p.n_str;
        if (gemv_ws_floats(n, K, B) > c->ws_floats || gemv_counters(n, K, B) > c->n_counters)
            return set_error(HG_EINVAL, "GEMV of %lld rows x K=%lld exceeds the context workspace", (long long)n,
                             (long long)K);
        StreamLaunch S{};
        S.x = L.x;
        S.batch = B;
        S.K = K;
        S.W_res = L.W_dev;
        S.n_res = p.n_res;
        S.ring = c->ring;
        S.slot_bytes = c->slot_bytes;
        S.nslots = c->nslots;
        S.seq0 = seq0;
        S.n_chunks = (p.n_str > 0 && !direct) ? p.n_chunks : 0;
        S.chunk_rows = p.chunk_rows;
        S.n_str = direct ? 0 : p.n_str;
        const void *wdir = nullptr;
        if (direct && p.n_str > 0) {  // the device address of the pinned host rows (UVA mapping; checked
                                      // by validate_lin / validate_layer before anything was enqueued)
            cudaPointerAttributes at;
            HG_CK(c, cudaPointerGetAttributes(&at, L.W_host));
            wdir = at.devicePointer;
        }
        S.W_dir = wdir;
        S.n_dir = direct ? p.n_str : 0;
        S.arrived = direct ? nullptr : c->arrived;
        S.consumed = c->consumed;
        S.slot_cnt = c->slot_cnt;
        S.bias = L.bias;
        S.y = L.y;
        S.ldy = L.ldy;
        S.ws = c->ws;
        S.gbar = c->gbar;
        S.err = c->err;
        S.timeout_s = c->cfg.timeout_s;
        S.trace = dbg_trace(c);
        S.trace_id = (uint32_t)(c->trace_seq++);
        if (S.trace) {
            c->trace_lin.push_back({S.trace_id, (int64_t)seq0, (int64_t)S.n_chunks, p.n_res, p.n_str, p.K});
        }
        if (tc_stream &&
            gemv_tc_stream_tiles(p.n_res, p.n_str, p.chunk_rows, S.n_chunks) > c->n_counters)
            return set_error(HG_EINVAL, "tcgen05 GEMV: %lld rows need more tile counters than the context has",
                             (long long)n);
        if (n > 0) {
            size_t i0 = 0, i1 = 0;
            cudaEvent_t e0 = nullptr;
            if (c->cfg.collect_stats && (e0 = tev_get(c, &i0))) HG_CK(c, cudaEventRecord(e0, s));
            if (tc_stream) {
                HG_TRY(kerr(c, launch_gemv_tc_stream(S, c->counters, s), "gemv tcgen05 stream launch"));
            }
            else
                HG_TRY(kerr(c, launch_gemv_stream(S, s), "gemv stream launch"));
            c->st.gpu_launches++;
            for (int64_t i = 0; i < S.n_chunks; ++i)  // the slots are free once this GEMV is done
                HG_CK(c, cudaEventRecord(c->ev_free[(seq0 + i) % c->nslots], s));
            if (e0) {
                cudaEvent_t e1 = tev_get(c, &i1);
                if (e1) {
                    HG_CK(c, cudaEventRecord(e1, s));
                    c->gemv_ev.push_back({i0, i1});
                }
            }
        }
        c->st.bytes_res += 2 * K * p.n_res;
        c->st.bytes_str += 2 * K * p.n_str;
        if (p.n_str > 0 && !direct) c->st.n_chunks += p.n_chunks;
        return direct ? HG_OK : pump(c);
    }
    if (p.n_res > 0) {  // a3
        HG_TRY(gemv(c, L.x, B, K, L.W_dev, p.n_res, L.bias, L.y, L.ldy, s));
        c->st.bytes_res += 2 * K * p.n_res;
    }
    if (p.n_str > 0) {  // a4
        std::vector<ChunkReq> mine;
        push_chunks(mine, p, L.W_host);
        for (int64_t i = 0; i < p.n_chunks; ++i) {
            int slot = 0;
            HG_TRY(acquire(c, mine[i], s, &slot));
            const int64_t r0 = p.n_res + i * p.chunk_rows;
            const int64_t rows = mine[i].bytes / (2 * K);
            HG_TRY(gemv(c, L.x, B, K, c->ring + (int64_t)slot * c->slot_bytes, rows,
                        L.bias ? L.bias + r0 : nullptr, L.y + r0, L.ldy, s));
            HG_TRY(release(c, slot, s));
            HG_TRY(pump(c));
        }
        c->st.bytes_str += 2 * K * p.n_str;
        c->st.n_chunks += p.n_chunks;
    }
    return HG_OK;
}

bool blocking_pin(const hg_ctx *c) { return c->cfg.pageable && c->cfg.strategy == HG_STRATEGY_PINNED_BLOCKING; }

hg_status run_linear(hg_ctx *c, const Lin &L, cudaStream_t s) {
    const hg_plan_t &p = L.plan;
    const int B = (int)p.batch;
    const int64_t K = p.K;
    HG_TRY(pump(c));
    if (p.n_cpu == 0) {
        HG_TRY(enqueue_gpu_lanes(c, L, s));
        c->st.n_linears++;
        return HG_OK;
    }
    // a2: activation to the host first; the CPU lane is the long pole
    HG_CK(c, cudaMemcpyAsync(c->x_host, L.x, (size_t)B * K * 2, cudaMemcpyDeviceToHost, s));
    HG_CK(c, cudaEventRecord(c->ev_x, s));
    {  // a5 + a3/a4: workers start on the CPU rows the moment x lands, while this thread
       // enqueues the GPU lanes behind the D2H and then joins the CPU rows itself
       // (HG_ASYNC_POST=0: enqueue the GPU lanes first, then compute -- A/B switch).
        static const bool async_post_env = !getenv("HG_ASYNC_POST") || atoi(getenv("HG_ASYNC_POST")) != 0;
        // pinned-blocking (Fig. 5b) pins the linear's streamed rows on the pool threads before the CPU rows
        const bool async_post = async_post_env && !blocking_pin(c);
        hg_status gst = HG_OK;
        if (!async_post) HG_TRY(enqueue_gpu_lanes(c, L, s));
        HG_TRY(wait_event(c, c->ev_x, &c->st.x_wait_s));
        const int yb = c->ybuf;
        c->ybuf ^= 1;
        HG_TRY(wait_event(c, c->ev_ycpu[yb], nullptr));  // this buffer's previous join has read it
        const auto t0 = clk::now();
        HostJob job;
        job.fn = host_fn_for(c, B);
        job.x = c->x_host;
        job.batch = B;
        job.K = K;
        job.n = p.n_cpu;
        job.W = (const uint16_t *)(L.W_host + 2 * K * p.n_str);
        job.bias = nullptr;  // bias joins on the device
        job.y = c->ycpu_host[yb];
        job.ldy = p.n_cpu;
        job.block = 16;
        job.next.store(0);
        if (async_post) {
            host_gemv_new_job();
            pool_post(c->pool, host_job_run, &job);
            gst = enqueue_gpu_lanes(c, L, s);
            pool_join(c->pool);  // always: workers reference `job`
        } else {
            host_gemv_new_job();
            pool_run(c->pool, host_job_run, &job);
        }
        if (gst != HG_OK) return gst;
        c->st.cpu_busy_s += secs(t0, clk::now());
        c->st.bytes_cpu += 2 * K * p.n_cpu;
        static const bool join_memcpy = getenv("HG_JOIN_MEMCPY") && atoi(getenv("HG_JOIN_MEMCPY")) != 0;
        const float *ysrc = c->ycpu_map[yb];
        if (join_memcpy) {  // A/B reference: H2D copy engine (queues behind the chunk stream)
            HG_CK(c, cudaMemcpyAsync(c->ycpu_dev, c->ycpu_host[yb], (size_t)B * p.n_cpu * 4,
                                     cudaMemcpyHostToDevice, s));
            ysrc = c->ycpu_dev;
        }
        const int64_t col0 = p.n_res + p.n_str;
        HG_TRY(kerr(c, launch_join(L.y, L.ldy, col0, p.n_cpu, B, ysrc, p.n_cpu, L.bias, s), "join"));
        HG_CK(c, cudaEventRecord(c->ev_ycpu[yb], s));
        c->st.gpu_launches++;
    }
    c->st.n_linears++;
    return HG_OK;
}


hg_status validate_plan(hg_ctx *c, const hg_plan_t &p) {
    if (p.batch < 1 || p.batch > HG_MAX_BATCH) return set_error(HG_EINVAL, "batch %lld", (long long)p.batch);
    if (p.K <= 0 || p.K % 8) return set_error(HG_EALIGN, "K=%lld must be a positive multiple of 8", (long long)p.K);
    if (p.K > c->cfg.max_k || p.N > c->cfg.max_n)
        return set_error(HG_EINVAL, "N=%lld K=%lld exceed context max_n/max_k", (long long)p.N, (long long)p.K);
    if (p.granule < 1 || p.N % p.granule || p.n_res % p.granule || p.n_res < 0 || p.n_str < 0 ||
        p.n_cpu < 0 || p.n_res + p.n_str + p.n_cpu != p.N || p.chunk_rows < 1 ||
        p.n_chunks != (p.n_str + p.chunk_rows - 1) / p.chunk_rows)
        return set_error(HG_EINVAL, "inconsistent plan");
    if (p.chunk_rows * p.K * 2 > c->slot_bytes)
        return set_error(HG_EINVAL, "chunk of %lld rows x K=%lld exceeds the ring slot (%lld B)",
                         (long long)p.chunk_rows, (long long)p.K, (long long)c->slot_bytes);
    return HG_OK;
}

// stream_mode 1 (zero-copy streaming) reads the streamed rows through the host pointer's device
// mapping: checked with the other arguments, before anything is enqueued.
hg_status check_mapped(hg_ctx *c, const hg_plan_t &p, const void *W_host) {
    if (c->cfg.stream_mode != 1 || p.n_str <= 0 || gemv_use_tc((int)p.batch, p.K)) return HG_OK;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, W_host) != cudaSuccess || !at.devicePointer) {
        cudaGetLastError();
        return set_error(HG_ENOTPINNED, "stream_mode 1: W_host is not mapped into the device address space");
    }
    return HG_OK;
}

hg_status validate_lin(hg_ctx *c, const hg_plan_t &p, const void *x, const void *W_dev,
                       const void *W_host, const float *bias, const float *y) {
    HG_TRY(validate_plan(c, p));
    HG_TRY(check_ptr(c, x, true, "x"));
    if (!aligned(x, 16)) return set_error(HG_EALIGN, "x not 16-byte aligned");
    if (p.n_res > 0) {
        HG_TRY(check_ptr(c, W_dev, true, "W_dev"));
        if (!aligned(W_dev, 16)) return set_error(HG_EALIGN, "W_dev not 16-byte aligned");
    }
    if (p.n_res < p.N) {
        HG_TRY(check_ptr(c, W_host, false, "W_host"));
        if (!aligned(W_host, 16)) return set_error(HG_EALIGN, "W_host not 16-byte aligned");
        HG_TRY(check_mapped(c, p, W_host));
    }
    if (bias) {
        HG_TRY(check_ptr(c, bias, true, "bias"));
        if (!aligned(bias, 4)) return set_error(HG_EALIGN, "bias not 4-byte aligned");
    }
    HG_TRY(check_ptr(c, y, true, "y"));
    if (!aligned(y, 4)) return set_error(HG_EALIGN, "y not 4-byte aligned");
    return HG_OK;
}

// Asynchronous failures found without synchronising: a GEMV's bounded wait for a streamed chunk
// (the kernel sets the mapped err word) or the pin lane's bounded wait for a staging slot.  Both
// leave the results of the call in flight undefined, so the context enters its error state.
hg_status check_async_errors(hg_ctx *c) {
    if (c->err_host && c->err_host[0]) {
        c->error = true;
        return set_error(HG_ETIMEOUT, c->err_host[0] == 2u ? "a peer exchange waited longer than %.1f s for another rank"
                                                           : "a GEMV waited longer than %.1f s for a streamed chunk",
                         c->cfg.timeout_s);
    }
    if (c->pin && pinlane_error(c->pin)) {
        c->error = true;
        return set_error(HG_ETIMEOUT, "the pin lane waited longer than %.1f s for a staging slot", c->cfg.timeout_s);
    }
    if (c->naive && c->naive->err) {
        c->error = true;
        return set_error(HG_ECUDA, "the naive-strategy transfer thread failed to enqueue a copy");
    }
    return HG_OK;
}

// Every copy the naive-strategy transfer thread was handed is enqueued on its stream, and that stream
// has finished (synchronising points: stats, measurement, reallocation).
hg_status sync_naive(hg_ctx *c) {
    if (!c->naive) return HG_OK;
    c->naive->drain();
    HG_CK(c, cudaStreamSynchronize(c->naive->st));
    return HG_OK;
}

hg_status begin_call(hg_ctx *c, cudaStream_t s) {
    if (c->error) return set_error(HG_ESTATE, "context is in an error state");
    if (c->device < 0) return set_error(HG_ESTATE, "host-only context");
    HG_TRY(check_async_errors(c));
    HG_CK(c, cudaSetDevice(c->device));
    gemv_set_tc_min_batch(c->cfg.gemv_tc_min_batch);
    HG_TRY(stream_guard(c, s));
    // Stats accumulate over all calls since hg_reset_stats (no per-call sync, so the
    // copy stream keeps running ahead across calls while statistics are collected).
    if (!c->stats_open) {
        HG_CK(c, cudaEventRecord(c->ev_call0, s));
        c->stats_open = true;
    }
    return HG_OK;
}

hg_status end_call(hg_ctx *c, cudaStream_t s) {
    HG_TRY(check_async_errors(c));
    HG_CK(c, cudaEventRecord(c->ev_call1, s));
    HG_CK(c, cudaEventRecord(c->ev_done, s));
    c->call_timed = true;
    return HG_OK;
}

// Grow a scratch buffer.  The old one may still be read by queued work, and freeing it would
// synchronise the whole device (cudaFree) -- a deadlock when other ranks share the device and spin on
// this rank's next exchange -- so it is retired and freed with the context.
hg_status ensure(hg_ctx *c, void **p, int64_t *have, int64_t need_bytes) {
    if (*have >= need_bytes) return HG_OK;
    if (*p) {
        c->retired.push_back(*p);
        *p = nullptr;
    }
    HG_CK(c, cudaMalloc(p, (size_t)need_bytes));
    *have = need_bytes;
    return HG_OK;
}

// all-gather this rank's [B, n_local] shard into y [B, P*n_local]
hg_status gather(hg_ctx *c, const float *ylocal, int B, int64_t n_local, float *y, cudaStream_t s) {
    const int P = nranks_of(c);
    if (c->peer) {  // peer-memory exchange: pushes + flags, the full y in global column order
        HG_TRY(kerr(c, peer_exchange(c->peer, ylocal, B, n_local, y, (int64_t)P * n_local, c->err, c->cfg.timeout_s, s),
                    "peer exchange"));
        c->st.gpu_launches += 2;
        return HG_OK;
    }
    if (B == 1) return dist_allgather(c->dist, ylocal, y, (size_t)n_local, s);
    HG_TRY(ensure(c, (void **)&c->gbuf, &c->gbuf_elems, (int64_t)P * B * n_local * 4));
    HG_TRY(dist_allgather(c->dist, ylocal, c->gbuf, (size_t)B * n_local, s));
    HG_TRY(kerr(c, launch_gather_permute(c->gbuf, P, B, n_local, y, s), "gather permute"));
    c->st.gpu_launches++;
    return HG_OK;
}

// all-reduce of a row-parallel linear's partial [B, N] into y [B, N] (+ bias once), peer group only
hg_status reduce(hg_ctx *c, const float *partial, int B, int64_t N, const float *bias, float *y, cudaStream_t s) {
    if (!c->peer) return set_error(HG_EUNSUPPORTED, "row-parallel linears need the peer group (hg_peer_open)");
    HG_TRY(kerr(c, peer_reduce(c->peer, partial, B, N, bias, y, N, c->err, c->cfg.timeout_s, s), "peer reduce"));
    c->st.gpu_launches += 2;
    return HG_OK;
}

// How a layer's linear meets the other ranks' shards (hg_tp; one rank: kLocal).
enum class Xchg { kGather, kLocal, kReduce };

// One linear of a layer: kGather (P > 1: local rows, then all-gather into y [B, P*N]), kLocal (this
// rank's rows only, y [B, N]), kReduce (partial without bias, then all-reduce + bias into y [B, N]).
hg_status layer_linear(hg_ctx *c, const hg_linear_desc &d, const void *x, float *y, int64_t N_full,
                       cudaStream_t s, Xchg kind = Xchg::kGather) {
    const int P = nranks_of(c);
    Lin L{d.plan, x, d.W_dev, (const uint8_t *)d.W_host, d.bias, y, N_full};
    if (P == 1 || kind == Xchg::kLocal) {
        L.ldy = d.plan.N;
        return run_linear(c, L, s);
    }
    HG_TRY(ensure(c, (void **)&c->ylocal, &c->ylocal_elems, d.plan.batch * d.plan.N * 4));
    L.y = c->ylocal;
    L.ldy = d.plan.N;
    if (kind == Xchg::kReduce) {
        L.bias = nullptr;  // added once, after the sum
        HG_TRY(run_linear(c, L, s));
        return reduce(c, c->ylocal, (int)d.plan.batch, d.plan.N, d.bias, y, s);
    }
    HG_TRY(run_linear(c, L, s));
    return gather(c, c->ylocal, (int)d.plan.batch, d.plan.N, y, s);
}

// Megatron pairing in force for this layer (HG_TP_MEGATRON with more than one rank).
bool megatron(const hg_ctx *c, const hg_opt_layer &l) { return l.tp == HG_TP_MEGATRON && nranks_of(c) > 1; }

hg_status validate_layer(hg_ctx *c, const hg_opt_layer &l, int B) {
    const int P = nranks_of(c);
    const int64_t H = l.hidden, F = l.ffn;
    if (H <= 0 || F <= 0) return set_error(HG_EINVAL, "layer: hidden/ffn must be > 0");
    if (l.tp != HG_TP_COLUMN && l.tp != HG_TP_MEGATRON) return set_error(HG_EINVAL, "layer: tp %d", l.tp);
    const bool mg = megatron(c, l);
    if (mg && (H % P || F % P)) return set_error(HG_EINVAL, "layer: Megatron needs H and F divisible by P");
    if (mg && !c->peer) return set_error(HG_EUNSUPPORTED, "layer: Megatron pairing needs the peer group");
    // expected (N, K) of this rank's descriptors: column shards (N_full / P rows), or the Megatron
    // shapes (hg_tp)
    const int64_t Nfull[4] = {3 * H, H, F, H};
    const int64_t Ns[4] = {3 * H / P, mg ? H : H / P, F / P, mg ? H : H / P};
    const int64_t Ks[4] = {H, mg ? H / P : H, H, mg ? F / P : F};
    for (int i = 0; i < 4; ++i) {
        const hg_linear_desc &d = l.lin[i];
        const bool rows_split = !mg || i == 0 || i == 2;  // this linear's output columns are sharded
        if (d.plan.N != Ns[i] || d.plan.K != Ks[i] || d.plan.batch != B || (rows_split && Nfull[i] % P))
            return set_error(HG_EINVAL, "layer linear %d: plan (N=%lld K=%lld B=%lld) does not match "
                                        "(N=%lld K=%lld B=%d; %d ranks, %s)", i, (long long)d.plan.N,
                             (long long)d.plan.K, (long long)d.plan.batch, (long long)Ns[i], (long long)Ks[i], B,
                             P, mg ? "Megatron" : "column shards");
        HG_TRY(validate_plan(c, d.plan));
        if (d.plan.n_res > 0) HG_TRY(check_ptr(c, d.W_dev, true, "layer W_dev"));
        if (d.plan.n_res < d.plan.N) {
            HG_TRY(check_ptr(c, d.W_host, false, "layer W_host"));
            HG_TRY(check_mapped(c, d.plan, d.W_host));
        }
        if (d.bias) HG_TRY(check_ptr(c, d.bias, true, "layer bias"));
    }
    return HG_OK;
}

hg_status trace_copy(hg_ctx *c, void *dst, const void *src, size_t bytes, cudaStream_t s) {
    if (dst) HG_CK(c, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
    return HG_OK;
}

hg_status run_layer(hg_ctx *c, const hg_opt_layer &l, void *h, int B, hg_layer_trace *tr,
                    cudaStream_t s) {
    const int64_t H = l.hidden, F = l.ffn;
    // Megatron pairing (hg_tp): qkv / fc1 stay local ([B, 3H/P], [B, F/P]; the V slice and the ReLU
    // act on this rank's columns), o / fc2 are all-reduced; otherwise every linear is all-gathered
    const bool mg = megatron(c, l);
    const int P = nranks_of(c);
    const int64_t Hl = mg ? H / P : H, Fl = mg ? F / P : F;
    const Xchg col = mg ? Xchg::kLocal : Xchg::kGather, row = mg ? Xchg::kReduce : Xchg::kGather;
    HG_TRY(ensure(c, &c->act, &c->act_elems, (int64_t)B * (F > H ? F : H) * 2));
    HG_TRY(ensure(c, (void **)&c->yscr, &c->yscr_elems, (int64_t)B * (F > 3 * H ? F : 3 * H) * 4));
    HG_TRY(ensure(c, &c->h1, &c->h1_elems, (int64_t)B * H * 2));
    // a = LN1(h)
    HG_TRY(kerr(c, launch_layernorm(h, H, B, l.ln1_g, l.ln1_b, c->act, s), "ln1"));
    if (tr) HG_TRY(trace_copy(c, tr->a, c->act, (size_t)B * H * 2, s));
    // qkv
    HG_TRY(layer_linear(c, l.lin[0], c->act, c->yscr, 3 * H, s, col));
    if (tr && tr->y_qkv) HG_TRY(trace_copy(c, tr->y_qkv, c->yscr, (size_t)B * 3 * Hl * 4, s));
    // attention at decode position 0: context = v
    HG_TRY(kerr(c, launch_slice_to_bf16(c->yscr, 3 * Hl, 2 * Hl, Hl, B, c->act, s), "v"));
    if (tr) HG_TRY(trace_copy(c, tr->v, c->act, (size_t)B * Hl * 2, s));
    // o
    HG_TRY(layer_linear(c, l.lin[1], c->act, c->yscr, H, s, row));
    if (tr) HG_TRY(trace_copy(c, tr->y_o, c->yscr, (size_t)B * H * 4, s));
    // h1 = h + o ; a2 = LN2(h1)
    HG_TRY(kerr(c, launch_residual_ln(h, c->yscr, H, B, c->h1, l.ln2_g, l.ln2_b, c->act, s), "res+ln2"));
    if (tr) {
        HG_TRY(trace_copy(c, tr->h1, c->h1, (size_t)B * H * 2, s));
        HG_TRY(trace_copy(c, tr->a2, c->act, (size_t)B * H * 2, s));
    }
    // fc1 + ReLU
    HG_TRY(layer_linear(c, l.lin[2], c->act, c->yscr, F, s, col));
    if (tr) HG_TRY(trace_copy(c, tr->y_fc1, c->yscr, (size_t)B * Fl * 4, s));
    HG_TRY(kerr(c, launch_relu_bf16(c->yscr, Fl, B, c->act, s), "relu"));
    if (tr) HG_TRY(trace_copy(c, tr->u, c->act, (size_t)B * Fl * 2, s));
    // fc2 + residual
    HG_TRY(layer_linear(c, l.lin[3], c->act, c->yscr, H, s, row));
    if (tr) HG_TRY(trace_copy(c, tr->y_fc2, c->yscr, (size_t)B * H * 4, s));
    HG_TRY(kerr(c, launch_residual(c->h1, c->yscr, H, B, h, s), "residual"));
    c->st.gpu_launches += 5;
    return HG_OK;
}

// ---------------------------------------------------------------- mirrored glue (reading R24)
//
// At P > 1 every rank must take the same decision: the mirrored ranks publish their rows of every
// linear into the shared host segment and wait for everybody else's, so one rank on the plain path
// would leave the others waiting.  The decision then depends only on what all ranks pass alike (the
// configuration and which host copies the descriptors carry), not on this rank's own plans: a rank
// whose shards have no CPU rows still mirrors (it publishes its GPU rows and keeps its host copy of
// the residual stream up to date).
bool can_mirror(hg_ctx *c, const hg_opt_layer *layers, int n) {
    // P > 1 mirrors only through the peer group's shared host segment (not with NCCL)
    const bool multi = nranks_of(c) != 1;
    if (!c->cfg.mirror_glue || (multi && !c->peer) || !hglue_supported()) return false;
    for (int l = 0; l < n; ++l)  // the Megatron pairing takes the plain path (tp is alike on every rank)
        if (megatron(c, layers[l])) return false;
    bool any_cpu = false;  // without CPU rows nobody needs the glue on the host
    for (int l = 0; l < n; ++l)
        for (int i = 0; i < 4; ++i) any_cpu |= layers[l].lin[i].plan.n_cpu > 0;
    if (!any_cpu && !multi) return false;
    for (int l = 0; l < n; ++l) {
        const hg_opt_layer &L = layers[l];
        if ((L.ln1_g && !L.ln1_g_host) || (L.ln1_b && !L.ln1_b_host) || (L.ln2_g && !L.ln2_g_host) ||
            (L.ln2_b && !L.ln2_b_host))
            return false;
        for (int i = 0; i < 4; ++i)
            if (L.lin[i].bias && !L.lin[i].bias_host && (multi || L.lin[i].plan.n_cpu > 0)) return false;
    }
    return true;
}

// Compare the host activation with the device one (verify_mirror; synchronises).
hg_status verify_act(hg_ctx *c, const uint16_t *xh, const void *xd, int64_t n, cudaStream_t s) {
    c->xchk.resize((size_t)n);
    HG_CK(c, cudaMemcpyAsync(c->xchk.data(), xd, (size_t)n * 2, cudaMemcpyDeviceToHost, s));
    HG_CK(c, cudaStreamSynchronize(s));
    for (int64_t i = 0; i < n; ++i) c->st.mirror_mismatch += c->xchk[i] != xh[i];
    return HG_OK;
}

// HG_SYNC_DEBUG=1: synchronise after every GPU step of the mirrored stack and name the one that
// failed (development aid for asynchronous device faults).
hg_status dbg_sync(hg_ctx *c, cudaStream_t s, const char *what, int k) {
    static const int mode = getenv("HG_SYNC_DEBUG") ? atoi(getenv("HG_SYNC_DEBUG")) : 0;
    if (!mode) return HG_OK;
    if (mode == 2) {  // no synchronisation: report the first sticky error seen after this step
        const cudaError_t e = cudaPeekAtLastError();
        if (e != cudaSuccess) {
            fprintf(stderr, "hg debug: error seen after %s (linear %d): %s\n", what, k, cudaGetErrorString(e));
            return set_error(HG_ECUDA, "%s (linear %d): %s", what, k, cudaGetErrorString(e));
        }
        const cudaError_t q = cudaStreamQuery(s);
        if (q != cudaSuccess && q != cudaErrorNotReady) {
            fprintf(stderr, "hg debug: stream error after %s (linear %d): %s\n", what, k, cudaGetErrorString(q));
            return set_error(HG_ECUDA, "%s (linear %d): %s", what, k, cudaGetErrorString(q));
        }
        return HG_OK;
    }
    cudaError_t e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->copy);
    if (e == cudaSuccess && c->d2h) e = cudaStreamSynchronize(c->d2h);
    if (e != cudaSuccess) {
        c->error = true;
        fprintf(stderr, "hg debug: %s (linear %d): %s\n", what, k, cudaGetErrorString(e));
        return set_error(HG_ECUDA, "%s (linear %d): %s", what, k, cudaGetErrorString(e));
    }
    return HG_OK;
}

hg_status ensure_mirror(hg_ctx *c) {
    if (c->yring) return HG_OK;
    const size_t per = (size_t)HG_MAX_BATCH * c->cfg.max_n;
    HG_CK(c, cudaMalloc((void **)&c->yring, per * 4 * hg_ctx::kMirrorRing));
    for (int r = 0; r < hg_ctx::kMirrorRing; ++r) {
        HG_CK(c, cudaHostAlloc((void **)&c->yhost[r], per * 4, cudaHostAllocMapped));
        HG_CK(c, cudaHostGetDevicePointer((void **)&c->ymap[r], c->yhost[r], 0));
        HG_CK(c, cudaEventCreateWithFlags(&c->ev_g[r], cudaEventDisableTiming));
        HG_CK(c, cudaEventCreateWithFlags(&c->ev_yg[r], cudaEventDisableTiming));
        HG_CK(c, cudaEventCreateWithFlags(&c->ev_use[r], cudaEventDisableTiming));
    }
    HG_CK(c, cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    if (c->peer) HG_CK(c, cudaMalloc((void **)&c->ylring, per * 4 * hg_ctx::kMirrorRing));
    return HG_OK;
}

// One decode step over n layers (P = 1) with the glue mirrored on the host (reading R24).
//
// GPU stream: per linear [glue kernel -> act] [GEMV lanes -> y ring slot] [join of the CPU rows];
// the GPU rows of every y go D2H on a side stream into the matching host slot.  The host never
// waits for the GPU to enqueue: a linear without CPU rows is enqueued and passed, and the host
// brings its copy of the residual stream up to date ("catches up") only when a linear with CPU
// rows needs its input -- from each linear's full y (its CPU rows were written there by the CPU
// lane itself, its GPU rows arrive D2H while the CPU lane is busy).  So neither a D2H of x nor the
// zero-copy join sits on the CPU lane's critical path, and fully resident linears run back to back.
hg_status run_stack_mirror(hg_ctx *c, const hg_opt_layer *layers, int nl, void *h, int B, hg_layer_trace *trs,
                           cudaStream_t s) {
    constexpr int R = hg_ctx::kMirrorRing;
    const int64_t H = layers[0].hidden;
    int64_t maxF = 0;
    for (int l = 0; l < nl; ++l) maxF = std::max(maxF, layers[l].ffn);
    const int64_t ystride = (int64_t)HG_MAX_BATCH * c->cfg.max_n;
    if (std::max(maxF, 3 * H) > c->cfg.max_n) return set_error(HG_EINVAL, "layer width exceeds max_n");
    HG_TRY(ensure_mirror(c));
    HG_TRY(ensure(c, &c->act, &c->act_elems, (int64_t)B * std::max(maxF, H) * 2));
    HG_TRY(ensure(c, &c->h1, &c->h1_elems, (int64_t)B * H * 2));
    c->hh.resize((size_t)B * H);
    c->hh1.resize((size_t)B * H);
    HG_CK(c, cudaMemcpyAsync(c->hh.data(), h, (size_t)B * H * 2, cudaMemcpyDeviceToHost, s));
    HG_CK(c, cudaStreamSynchronize(s));
    uint16_t *xh = c->x_host;
    const int total = 4 * nl;
    auto lin_of = [&](int k) -> const hg_linear_desc & { return layers[k / 4].lin[k % 4]; };
    auto ydev = [&](int k) { return c->yring + (int64_t)(k % R) * ystride; };
    // P > 1 (peer group, peer.cu): linear k's full y lives in the host segment shared by all ranks (this
    // rank's columns start at pr * n_local); the device computes its rows into a local ring slot and the
    // peer exchange assembles the full y in ydev(k)
    PeerGroup *g = c->peer;
    const int Pn = g ? peer_nranks(g) : 1, pr = g ? peer_rank(g) : 0;
    const int64_t hk0 = c->hseq;  // host-segment index of linear 0 of this call
    c->hseq += total;
    auto ylocal = [&](int k) { return Pn > 1 ? c->ylring + (int64_t)(k % R) * ystride : ydev(k); };
    auto yhost_of = [&](int k) { return Pn > 1 ? peer_host_y(g, hk0 + k) : c->yhost[k % R]; };
    auto yhost_dev_of = [&](int k) { return Pn > 1 ? peer_host_y_dev(g, hk0 + k) : c->ymap[k % R]; };
    // this rank's part of linear j in the host segment: CPU rows written (its CPU job was joined in
    // iteration j) and GPU rows' D2H landed; published in order, eagerly when the D2H is already done
    int published = -1;
    auto publish_upto = [&](int j, bool block) -> hg_status {
        while (published < j) {
            const int q = published + 1;
            if (block) HG_TRY(wait_event(c, c->ev_yg[q % R], &c->st.x_wait_s));
            else if (cudaEventQuery(c->ev_yg[q % R]) != cudaSuccess) {
                cudaGetLastError();
                return HG_OK;
            }
            peer_host_publish(g, hk0 + q);
            published = q;
        }
        return HG_OK;
    };
    // host catch-up: apply the glue of linears (done, upto] to the host residual stream; the input
    // x itself is produced only for `upto` (the linear whose CPU rows are about to run)
    int done = -1;
    auto catch_up = [&](int upto) -> hg_status {
        for (int k = done + 1; k <= upto; ++k) {
            const int l = k / 4, i = k % 4;
            const hg_opt_layer &L = layers[l];
            const bool want_x = k == upto;
            const float *yp = nullptr;  // previous linear's full y on the host
            if (k > 0) {
                if (Pn > 1) {  // every rank's rows of linear k-1 in the shared segment
                    HG_TRY(publish_upto(k - 1, true));
                    const auto tw = clk::now();
                    HG_TRY(peer_host_wait_ready(g, hk0 + k - 1, c->cfg.timeout_s));
                    c->st.x_wait_s += secs(tw, clk::now());
                } else {
                    HG_TRY(wait_event(c, c->ev_yg[(k - 1) % R], &c->st.x_wait_s));
                }
                yp = yhost_of(k - 1);
            }
            const auto tg = clk::now();
            if (i == 0) {
                if (l > 0) hglue_residual(c->hh1.data(), yp, H, H, B, c->hh.data());  // h = h1 + y_fc2
                if (want_x) hglue_layernorm(c->hh.data(), H, B, L.ln1_g_host, L.ln1_b_host, xh);
            } else if (i == 1) {
                if (want_x) hglue_slice_bf16(yp, 3 * H, 2 * H, H, B, xh);
            } else if (i == 2) {
                if (want_x) hglue_residual_ln(c->hh.data(), yp, H, H, B, c->hh1.data(), L.ln2_g_host, L.ln2_b_host, xh);
                else hglue_residual(c->hh.data(), yp, H, H, B, c->hh1.data());  // h1 = h + y_o
            } else {
                if (want_x) hglue_relu_bf16(yp, L.ffn, L.ffn, B, xh);
            }
            c->st.glue_s += secs(tg, clk::now());
            if (Pn > 1 && k > 0) peer_host_consumed(g, hk0 + k - 1);
            done = k;
        }
        return HG_OK;
    };
    for (int k = 0; k < total; ++k) {
        const int l = k / 4, i = k % 4;
        const hg_opt_layer &L = layers[l];
        const int64_t F = L.ffn;
        const hg_linear_desc &d = lin_of(k);
        const hg_plan_t &p = d.plan;
        const int64_t N = p.N, K = p.K, n_gpu = p.n_res + p.n_str;
        const int64_t N_full = N * Pn, col0 = (int64_t)pr * N;  // this rank's columns of the full y
        const int slot = k % R;
        float *yd = ydev(k);          // full y on the device
        float *yl = ylocal(k);        // this rank's rows (== yd at P = 1)
        float *yh = yhost_of(k);      // full y on the host (ld N_full)
        const float *yprev_d = k > 0 ? ydev(k - 1) : nullptr;
        HG_TRY(pump(c));
        // ---- GPU glue -> act (run_layer's kernels, reading the previous linear's ring slot)
        if (i == 0) {
            HG_TRY(kerr(c, launch_layernorm(h, H, B, L.ln1_g, L.ln1_b, c->act, s), "ln1"));
        } else if (i == 1) {
            HG_TRY(kerr(c, launch_slice_to_bf16(yprev_d, 3 * H, 2 * H, H, B, c->act, s), "v"));
        } else if (i == 2) {
            HG_TRY(kerr(c, launch_residual_ln(h, yprev_d, H, B, c->h1, L.ln2_g, L.ln2_b, c->act, s), "res+ln2"));
        } else {
            HG_TRY(kerr(c, launch_relu_bf16(yprev_d, F, B, c->act, s), "relu"));
        }
        c->st.gpu_launches++;
        hg_layer_trace *tr = trs ? &trs[l] : nullptr;
        if (tr) {  // the linear's input as the GPU computed it (stream-ordered device copies)
            void *xin = i == 0 ? tr->a : i == 1 ? tr->v : i == 2 ? tr->a2 : tr->u;
            HG_TRY(trace_copy(c, xin, c->act, (size_t)B * K * 2, s));
            if (i == 2) HG_TRY(trace_copy(c, tr->h1, c->h1, (size_t)B * H * 2, s));
        }
        HG_TRY(dbg_sync(c, s, "glue", k));
        // ---- this slot's previous occupant (k - R): its D2H must be done before y is overwritten,
        // and the host must have consumed its host copy before the new D2H / CPU rows land there
        if (k >= R) {
            HG_CK(c, cudaStreamWaitEvent(s, c->ev_yg[slot], 0));
            if (done < k - R + 1) HG_TRY(catch_up(k - R + 1));
        }
        if (Pn > 1) {  // the shared host slot's previous occupant has been read by every rank
            HG_TRY(publish_upto(k - 1, false));
            const auto tw = clk::now();
            HG_TRY(peer_host_wait_free(g, hk0 + k, c->cfg.timeout_s));
            c->st.x_wait_s += secs(tw, clk::now());
        }
        HostJob job;
        auto t0 = clk::now();
        // pinned-blocking (Fig. 5b): this linear's streamed rows are pinned on the pool threads first,
        // so its GPU lanes are enqueued before the CPU rows are posted
        const bool gpu_first = blocking_pin(c);
        hg_status gst = HG_OK;
        bool gpu_done = false;
        auto gpu_lanes = [&]() {
            Lin lin{p, c->act, d.W_dev, (const uint8_t *)d.W_host, d.bias, yl, N};
            gst = enqueue_gpu_lanes(c, lin, s);
            if (gst == HG_OK && n_gpu > 0) {
                cudaError_t e = cudaEventRecord(c->ev_g[slot], s);
                if (e == cudaSuccess) e = cudaStreamWaitEvent(c->d2h, c->ev_g[slot], 0);
                if (e == cudaSuccess) e = cudaStreamWaitEvent(c->d2h, c->ev_use[slot], 0);
                if (e == cudaSuccess)
                    e = cudaMemcpy2DAsync(yh + col0, (size_t)N_full * 4, yl, (size_t)N * 4, (size_t)n_gpu * 4,
                                          (size_t)B, cudaMemcpyDeviceToHost, c->d2h);
                if (e != cudaSuccess) gst = kerr(c, (int)e, "y D2H");
            }
            if (gst == HG_OK) {
                cudaError_t e = cudaEventRecord(c->ev_yg[slot], c->d2h);
                if (e != cudaSuccess) gst = kerr(c, (int)e, "y D2H event");
            }
            gpu_done = true;
        };
        if (gpu_first) {  // (the host is already past slot k - R: caught up above)
            gpu_lanes();
            if (gst != HG_OK) return gst;
        }
        if (p.n_cpu > 0) {
            HG_TRY(catch_up(k));
            c->st.mirror_linears++;
            if (c->cfg.verify_mirror) HG_TRY(verify_act(c, xh, c->act, (int64_t)B * K, s));
            HG_TRY(wait_event(c, c->ev_use[slot], nullptr));  // the join that read this slot is done
            job.fn = host_fn_for(c, B);
            job.x = xh;
            job.batch = B;
            job.K = K;
            job.n = p.n_cpu;
            job.W = (const uint16_t *)((const uint8_t *)d.W_host + 2 * K * p.n_str);
            job.bias = d.bias_host ? d.bias_host + n_gpu : nullptr;
            job.y = yh + col0 + n_gpu;
            job.ldy = N_full;
            job.block = 16;
            job.next.store(0);
            t0 = clk::now();  // CPU-lane busy time starts here (catch-up waits are x_wait)
            host_gemv_new_job();
            pool_post(c->pool, host_job_run, &job);
        }
        // ---- GPU rows into the ring slot, then (side stream) their copy to the host slot
        if (!gpu_done) gpu_lanes();
        if (p.n_cpu > 0) {
            pool_join(c->pool);  // always: workers reference `job`
            c->st.cpu_busy_s += secs(t0, clk::now());
            c->st.bytes_cpu += 2 * K * p.n_cpu;
        }
        if (gst != HG_OK) return gst;
        HG_TRY(dbg_sync(c, s, "gemv + y D2H", k));
        // ---- join: the CPU rows (bias already added on the host) into the ring slot on the device
        if (p.n_cpu > 0) {
            HG_TRY(kerr(c, launch_join(yl, N, n_gpu, p.n_cpu, B, yhost_dev_of(k) + col0 + n_gpu, N_full,
                                       d.bias_host ? nullptr : d.bias, s), "join"));
            c->st.gpu_launches++;
            HG_TRY(dbg_sync(c, s, "join", k));
        }
        if (Pn > 1) {  // a8: every rank's rows into every rank's y (peer stores), full y in yd
            HG_TRY(kerr(c, peer_exchange(g, yl, B, N, yd, N_full, c->err, c->cfg.timeout_s, s), "peer exchange"));
            c->st.gpu_launches += 2;
            if (Pn > 1) HG_TRY(publish_upto(k, false));
        }
        if (tr) {  // the linear's full output y (GPU rows + joined CPU rows)
            float *yt = i == 0 ? tr->y_qkv : i == 1 ? tr->y_o : i == 2 ? tr->y_fc1 : tr->y_fc2;
            HG_TRY(trace_copy(c, yt, yd, (size_t)B * N_full * 4, s));
        }
        HG_CK(c, cudaEventRecord(c->ev_use[slot], s));
        c->st.n_linears++;
        if (i == 3) {  // h = h1 + y_fc2 on the GPU (the host does the same when it catches up)
            HG_TRY(kerr(c, launch_residual(c->h1, yd, H, B, h, s), "residual"));
            c->st.gpu_launches++;
        }
    }
    // every rank may be waiting on this rank's last rows: publish them before returning; and this rank
    // reads none of this call's host slots any more (the next call starts from the device's h), so it
    // releases them all -- the last linear's y is read by nobody, and a rank whose shards have no CPU
    // rows has read only the slots its ring forced it to catch up on
    if (Pn > 1) {
        HG_TRY(publish_upto(total - 1, true));
        peer_host_consumed(g, hk0 + total - 1);
    }
    // the d2h stream must not run past this call's buffers unseen: order it before the caller's next work
    HG_CK(c, cudaEventRecord(c->ev_x, c->d2h));
    HG_CK(c, cudaStreamWaitEvent(s, c->ev_x, 0));
    return HG_OK;
}

}  // namespace

// =====================================================================================
// ABI
// =====================================================================================
extern "C" {

HG_API int hg_abi_version(void) { return HG_ABI_VERSION; }

HG_API size_t hg_struct_size(int which) {
    switch (which) {
        case 0: return sizeof(hg_rates);
        case 1: return sizeof(hg_plan_t);
        case 2: return sizeof(hg_config);
        case 3: return sizeof(hg_stats_t);
        case 4: return sizeof(hg_linear_desc);
        case 5: return sizeof(hg_opt_layer);
        case 6: return sizeof(hg_layer_trace);
        case 7: return sizeof(hg_abench_cfg);
        case 8: return sizeof(hg_abench_result);
        case 9: return sizeof(hg_module);
        default: return 0;
    }
}
HG_API const char *hg_last_error(void) { return g_err; }

HG_API hg_status hg_config_default(hg_config *cfg) {
    if (!cfg) return set_error(HG_EINVAL, "NULL cfg");
    std::memset(cfg, 0, sizeof *cfg);
    cfg->granule = 128;
    cfg->chunk_bytes = 16ll << 20;
    cfg->ring_bytes = 1ll << 30;
    cfg->max_k = 65536;
    cfg->max_n = 131072;
    cfg->cpu_threads = 0;
    cfg->cpu_first = -1;
    cfg->collect_stats = 0;
    cfg->wrap_prefetch = 0;
    cfg->timeout_s = 60.0;
    cfg->gemv_tc_min_batch = 2;  // measured: SIMT is issue-bound from B = 2 (profiles/r01/gemv_batches.md)
    if (const char *v = getenv("HG_GEMV_TC_MIN_BATCH")) cfg->gemv_tc_min_batch = atoi(v);
    cfg->handshake = 1;
    if (const char *v = getenv("HG_HANDSHAKE")) cfg->handshake = atoi(v);
    cfg->mirror_glue = 1;
    if (const char *v = getenv("HG_MIRROR_GLUE")) cfg->mirror_glue = atoi(v);
    cfg->stream_mode = 0;
    if (const char *v = getenv("HG_STREAM_MODE")) cfg->stream_mode = atoi(v);
    cfg->pageable = 0;
    cfg->pin_threads = 4;
    cfg->staging_bytes = 512ll << 20;
    cfg->verify_mirror = 0;
    cfg->numa_node = -1;
    return HG_OK;
}

HG_API const char *hg_host_isa(void) {
    const char *name = "?";
    host_rows_select(&name);
    return name;
}

HG_API hg_status hg_create(hg_ctx **out, int device, const hg_config *cfg_in) {
    if (!out) return set_error(HG_EINVAL, "NULL ctx pointer");
    *out = nullptr;
    hg_config cfg;
    if (cfg_in) cfg = *cfg_in;
    else hg_config_default(&cfg);
    if (cfg.granule < 1 || cfg.chunk_bytes < 1 || cfg.max_k < 8 || cfg.max_n < 1 ||
        !(cfg.timeout_s > 0))
        return set_error(HG_EINVAL, "bad config");
    if (cfg.strategy < HG_STRATEGY_HYBRID || cfg.strategy > HG_STRATEGY_PINNED_BLOCKING)
        return set_error(HG_EINVAL, "bad strategy %d", cfg.strategy);
    if (cfg.pageable && cfg.stream_mode == 1)  // zero-copy reads need page-locked, mapped rows
        return set_error(HG_EINVAL, "pageable weights cannot be streamed zero-copy (stream_mode 1)");
    hg_ctx *c = new hg_ctx;
    c->cfg = cfg;
    c->device = device;
    std::memset(&c->st, 0, sizeof c->st);
    // auto: leave cores to the CUDA driver's threads (and whatever else the process runs) -- with
    // every core in the pool a preempted worker stalls the lane now and then (profiles/r01/threads.md)
    const int ncpu = (int)sysconf(_SC_NPROCESSORS_ONLN);
    int nthr = cfg.cpu_threads > 0 ? cfg.cpu_threads : ncpu - (ncpu >= 12 ? 2 : ncpu >= 4 ? 1 : 0);
    // NUMA placement: pool threads on the cores of the GPU's node, from cpu_first on
    const int node = cfg.numa_node == -2 ? (device >= 0 ? numa_node_of_device(device) : -1) : cfg.numa_node;
    std::vector<int> cpus = numa_cpus(node);
    if (!cpus.empty()) {
        const size_t first = cfg.cpu_first > 0 ? (size_t)cfg.cpu_first % cpus.size() : 0;
        std::rotate(cpus.begin(), cpus.begin() + first, cpus.end());
        c->pool = pool_create_cpus(nthr, cpus);
    } else {
        c->pool = pool_create(nthr, cfg.cpu_first);
    }
    c->host_fn = host_rows_select(nullptr);
    {
        const char *v = getenv("HG_AMX_MIN_BATCH");
        const int want = v ? atoi(v) : 4;
        c->amx_min_batch = (want > 0 && !getenv("HG_HOST_ISA") && host_amx_enable()) ? want : 0;
    }
    if (device < 0) {
        *out = c;
        return HG_OK;
    }
    hg_status st = HG_OK;
    auto fail = [&](hg_status s) {
        hg_destroy(c);
        return s;
    };
#define CREATE_CK(expr)                                                                        \
    do {                                                                                       \
        cudaError_t e_ = (expr);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            st = set_error(e_ == cudaErrorMemoryAllocation ? HG_ENOMEM : HG_ECUDA, "%s: %s",    \
                           #expr, cudaGetErrorString(e_));                                     \
            return fail(st);                                                                   \
        }                                                                                      \
    } while (0)
    CREATE_CK(cudaSetDevice(device));
    if (gemv_prepare() != 0) return fail(set_error(HG_ECUDA, "gemv attributes"));
    CREATE_CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    c->slot_bytes = cfg.chunk_bytes;
    const int64_t min_slot = cfg.granule * cfg.max_k * 2;
    if (c->slot_bytes < min_slot) c->slot_bytes = min_slot;
    c->slot_bytes = (c->slot_bytes + 255) / 256 * 256;
    c->nslots = (int)(cfg.ring_bytes / c->slot_bytes);
    if (c->nslots < 2) c->nslots = 2;
    CREATE_CK(cudaMalloc((void **)&c->ring, (size_t)c->nslots * c->slot_bytes));
    c->ev_arrived.resize(c->nslots);
    c->ev_free.resize(c->nslots);
    c->slot_used.assign(c->nslots, 0);
    for (int i = 0; i < c->nslots; ++i) {
        CREATE_CK(cudaEventCreateWithFlags(&c->ev_arrived[i], cudaEventDisableTiming));
        CREATE_CK(cudaEventCreateWithFlags(&c->ev_free[i], cudaEventDisableTiming));
    }
    CREATE_CK(cudaHostAlloc((void **)&c->x_host, (size_t)HG_MAX_BATCH * cfg.max_k * 2, cudaHostAllocDefault));
    for (int i = 0; i < 2; ++i) {
        CREATE_CK(cudaHostAlloc((void **)&c->ycpu_host[i], (size_t)HG_MAX_BATCH * cfg.max_n * 4,
                                cudaHostAllocMapped));
        CREATE_CK(cudaHostGetDevicePointer((void **)&c->ycpu_map[i], c->ycpu_host[i], 0));
        CREATE_CK(cudaEventCreateWithFlags(&c->ev_ycpu[i], cudaEventDisableTiming));
    }
    CREATE_CK(cudaMalloc((void **)&c->ycpu_dev, (size_t)HG_MAX_BATCH * cfg.max_n * 4));
    CREATE_CK(cudaEventCreateWithFlags(&c->ev_x, cudaEventDisableTiming));
    CREATE_CK(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
    CREATE_CK(cudaEventCreate(&c->ev_call0));
    CREATE_CK(cudaEventCreate(&c->ev_call1));
    // workspace / counters: the largest any batch needs on either GEMV (SIMT stream, tcgen05)
    c->ws_floats = 1;
    c->n_counters = 1;
    for (int tcmin : {1, 0})
        for (int b = 1; b <= HG_MAX_BATCH; ++b) {
            gemv_set_tc_min_batch(tcmin);
            c->ws_floats = std::max(c->ws_floats, gemv_ws_floats(cfg.max_n, cfg.max_k, b));
            c->n_counters = std::max(c->n_counters, gemv_counters(cfg.max_n, cfg.max_k, b) + 1);
        }
    gemv_set_tc_min_batch(cfg.gemv_tc_min_batch);
    // the persistent tcgen05 launch has up to one partial tile per chunk on top
    c->n_counters = std::max(c->n_counters, (cfg.max_n + 127) / 128 + (int64_t)c->nslots + 2);
    CREATE_CK(cudaMalloc((void **)&c->ws, (size_t)c->ws_floats * 4));
    CREATE_CK(cudaMalloc((void **)&c->counters, (size_t)c->n_counters * 4));
    CREATE_CK(cudaMemset(c->counters, 0, (size_t)c->n_counters * 4));
    CREATE_CK(cudaMalloc((void **)&c->sink, 256));
    c->tags = cfg.handshake != 0 && load_memops();
    if (const char *v = getenv("HG_TC_STREAM")) c->tc_stream = atoi(v) != 0;
    CREATE_CK(cudaMalloc((void **)&c->tagmem, (size_t)(3 * c->nslots + 8 + kGroupCounters) * 4));
    CREATE_CK(cudaMemset(c->tagmem, 0, (size_t)(3 * c->nslots + 8 + kGroupCounters) * 4));
    c->arrived = c->tagmem;
    c->consumed = c->tagmem + c->nslots;
    c->slot_cnt = c->tagmem + 2 * c->nslots;
    c->gbar = c->tagmem + 3 * c->nslots + 4;
    {  // the kernels' timeout word lives in mapped host memory: begin_call/end_call poll it for free
        uint32_t *eh = nullptr;
        CREATE_CK(cudaHostAlloc((void **)&eh, 64, cudaHostAllocMapped));
        std::memset(eh, 0, 64);
        c->err_host = eh;
        CREATE_CK(cudaHostGetDevicePointer((void **)&c->err, eh, 0));
    }
    CREATE_CK(cudaDeviceSynchronize());
#undef CREATE_CK
    *out = c;
    return HG_OK;
}

HG_API hg_status hg_destroy(hg_ctx *c) {
    if (!c) return HG_OK;
    if (c->device >= 0) {
        cudaSetDevice(c->device);
        cudaDeviceSynchronize();
        if (c->dist) dist_destroy(c->dist);
        if (c->peer_pending) peer_destroy(c->peer_pending);
        if (c->ylring) cudaFree(c->ylring);
        for (auto e : c->ev_arrived) if (e) cudaEventDestroy(e);
        for (auto e : c->ev_free) if (e) cudaEventDestroy(e);
        for (auto e : c->tev) cudaEventDestroy(e);
        for (int r = 0; r < hg_ctx::kMirrorRing; ++r) {
            for (cudaEvent_t e : {c->ev_g[r], c->ev_yg[r], c->ev_use[r]})
                if (e) cudaEventDestroy(e);
            if (c->yhost[r]) cudaFreeHost(c->yhost[r]);
        }
        if (c->yring) cudaFree(c->yring);
        if (c->pin) pinlane_destroy(c->pin);
        if (c->naive) naive_destroy(c->naive);
        if (c->staging) cudaFreeHost(c->staging);
        if (c->pinflags) cudaFreeHost(c->pinflags);
        if (c->d2h) cudaStreamDestroy(c->d2h);
        for (cudaEvent_t e : {c->ev_x, c->ev_ycpu[0], c->ev_ycpu[1], c->ev_done, c->ev_call0, c->ev_call1})
            if (e) cudaEventDestroy(e);
        if (c->copy) cudaStreamDestroy(c->copy);
        for (void *p : {(void *)c->ring, (void *)c->ycpu_dev, (void *)c->ws, (void *)c->counters,
                        (void *)c->sink, c->act, (void *)c->yscr, c->h1, (void *)c->ylocal,
                        (void *)c->gbuf, (void *)c->tagmem})
            if (p) cudaFree(p);
        if (c->x_host) cudaFreeHost(c->x_host);
        for (void *q : c->retired) cudaFree(q);
        if (c->err_host) cudaFreeHost((void *)c->err_host);
        for (float *p : c->ycpu_host)
            if (p) cudaFreeHost(p);
    }
    if (c->pool) pool_destroy(c->pool);
    delete c;
    return HG_OK;
}

HG_API hg_status hg_linear_planned(hg_ctx *c, const hg_plan_t *p, const void *x, const void *W_dev,
                                   const void *W_host, const float *bias, float *y, void *stream) {
    if (!c || !p) return set_error(HG_EINVAL, "NULL argument");
    if (c->error) return set_error(HG_ESTATE, "context is in an error state");
    if (c->device < 0) return set_error(HG_ESTATE, "host-only context");
    HG_CK(c, cudaSetDevice(c->device));
    HG_TRY(validate_lin(c, *p, x, W_dev, W_host, bias, y));
    cudaStream_t s = (cudaStream_t)stream;
    HG_TRY(begin_call(c, s));
    std::vector<ChunkReq> list;
    push_chunks(list, *p, W_host);
    set_future(c, std::move(list), false);
    Lin L{*p, x, W_dev, (const uint8_t *)W_host, bias, y, p->N};
    HG_TRY(run_linear(c, L, s));
    return end_call(c, s);
}

HG_API hg_status hg_linear(hg_ctx *c, const void *x, int batch, int64_t N, int64_t K,
                           const void *W_dev, int64_t n_res, const void *W_host, double alpha,
                           const float *bias, float *y, void *stream) {
    if (!c) return set_error(HG_EINVAL, "NULL ctx");
    if (K % 8) return set_error(HG_EALIGN, "K %% 8 != 0");
    hg_rates r = {1, 1, 1, 1, 1, 1, 1};
    hg_plan_t p;
    HG_TRY(hg_plan(&r, N, K, batch, n_res, HG_ALPHA_FIXED, alpha, c->cfg.granule, c->cfg.chunk_bytes, &p));
    return hg_linear_planned(c, &p, x, W_dev, W_host, bias, y, stream);
}

HG_API hg_status hg_linear_sharded(hg_ctx *c, const hg_plan_t *p, const void *x, const void *W_dev,
                                   const void *W_host, const float *bias, float *y_full,
                                   void *stream) {
    if (!c || !p) return set_error(HG_EINVAL, "NULL argument");
    if (!c->dist && !c->peer) return set_error(HG_ESTATE, "neither hg_dist_init nor hg_peer_open called");
    if (c->error) return set_error(HG_ESTATE, "context is in an error state");
    HG_CK(c, cudaSetDevice(c->device));
    HG_TRY(validate_lin(c, *p, x, W_dev, W_host, bias, y_full));
    cudaStream_t s = (cudaStream_t)stream;
    HG_TRY(begin_call(c, s));
    std::vector<ChunkReq> list;
    push_chunks(list, *p, W_host);
    set_future(c, std::move(list), false);
    hg_linear_desc d{W_dev, W_host, bias, *p};
    HG_TRY(layer_linear(c, d, x, y_full, p->N * nranks_of(c), s));
    return end_call(c, s);
}

HG_API hg_status hg_linear_rowpar(hg_ctx *c, const hg_plan_t *p, const void *x, const void *W_dev,
                                  const void *W_host, const float *bias, float *y_full, void *stream) {
    if (!c || !p) return set_error(HG_EINVAL, "NULL argument");
    if (!c->peer) return set_error(HG_ESTATE, "hg_peer_open not called");
    if (c->error) return set_error(HG_ESTATE, "context is in an error state");
    HG_CK(c, cudaSetDevice(c->device));
    HG_TRY(validate_lin(c, *p, x, W_dev, W_host, bias, y_full));
    cudaStream_t s = (cudaStream_t)stream;
    HG_TRY(begin_call(c, s));
    std::vector<ChunkReq> list;
    push_chunks(list, *p, W_host);
    set_future(c, std::move(list), false);
    hg_linear_desc d{W_dev, W_host, bias, *p};
    HG_TRY(layer_linear(c, d, x, y_full, p->N, s, nranks_of(c) > 1 ? Xchg::kReduce : Xchg::kLocal));
    return end_call(c, s);
}

HG_API hg_status hg_layer(hg_ctx *c, const hg_opt_layer *l, void *h, int batch,
                          hg_layer_trace *trace, void *stream) {
    if (!c || !l) return set_error(HG_EINVAL, "NULL argument");
    if (c->error) return set_error(HG_ESTATE, "context is in an error state");
    if (c->device < 0) return set_error(HG_ESTATE, "host-only context");
    HG_CK(c, cudaSetDevice(c->device));
    HG_TRY(validate_layer(c, *l, batch));
    HG_TRY(check_ptr(c, h, true, "h"));
    cudaStream_t s = (cudaStream_t)stream;
    HG_TRY(begin_call(c, s));
    std::vector<ChunkReq> list;
    for (int i = 0; i < 4; ++i) push_chunks(list, l->lin[i].plan, l->lin[i].W_host);
    set_future(c, std::move(list), false);
    if (can_mirror(c, l, 1)) HG_TRY(run_stack_mirror(c, l, 1, h, batch, trace, s));
    else HG_TRY(run_layer(c, *l, h, batch, trace, s));
    return end_call(c, s);
}

HG_API hg_status hg_stack_trace(hg_ctx *c, const hg_opt_layer *layers, int n_layers, void *h, int batch,
                                hg_layer_trace *traces, void *stream) {
    if (!c || !layers || n_layers < 1) return set_error(HG_EINVAL, "bad arguments");
    if (c->error) return set_error(HG_ESTATE, "context is in an error state");
    if (c->device < 0) return set_error(HG_ESTATE, "host-only context");
    HG_CK(c, cudaSetDevice(c->device));
    for (int l = 0; l < n_layers; ++l) HG_TRY(validate_layer(c, layers[l], batch));
    HG_TRY(check_ptr(c, h, true, "h"));
    cudaStream_t s = (cudaStream_t)stream;
    HG_TRY(begin_call(c, s));
    std::vector<ChunkReq> list;
    for (int l = 0; l < n_layers; ++l)
        for (int i = 0; i < 4; ++i) push_chunks(list, layers[l].lin[i].plan, layers[l].lin[i].W_host);
    set_future(c, std::move(list), c->cfg.wrap_prefetch != 0);
    if (can_mirror(c, layers, n_layers)) {
        for (int l = 1; l < n_layers; ++l)
            if (layers[l].hidden != layers[0].hidden) return set_error(HG_EINVAL, "layers differ in hidden size");
        HG_TRY(run_stack_mirror(c, layers, n_layers, h, batch, traces, s));
    } else {
        for (int l = 0; l < n_layers; ++l) HG_TRY(run_layer(c, layers[l], h, batch, traces ? &traces[l] : nullptr, s));
    }
    return end_call(c, s);
}

HG_API hg_status hg_stack(hg_ctx *c, const hg_opt_layer *layers, int n_layers, void *h, int batch,
                          void *stream) {
    return hg_stack_trace(c, layers, n_layers, h, batch, nullptr, stream);
}

HG_API hg_status hg_gemv(hg_ctx *c, const void *x, int batch, int64_t n, int64_t K, const void *W,
                         const float *bias, float *y, int64_t ldy, void *stream) {
    if (!c) return set_error(HG_EINVAL, "NULL ctx");
    if (c->error) return set_error(HG_ESTATE, "context is in an error state");
    if (c->device < 0) return set_error(HG_ESTATE, "host-only context");
    if (batch < 1 || batch > HG_MAX_BATCH || n < 0 || K <= 0 || ldy < n)
        return set_error(HG_EINVAL, "hg_gemv: bad shape");
    if (K % 8) return set_error(HG_EALIGN, "K %% 8 != 0");
    HG_CK(c, cudaSetDevice(c->device));
    HG_TRY(check_ptr(c, x, true, "x"));
    HG_TRY(check_ptr(c, W, true, "W"));
    HG_TRY(check_ptr(c, y, true, "y"));
    if (bias) HG_TRY(check_ptr(c, bias, true, "bias"));
    if (!aligned(x, 16) || !aligned(W, 16)) return set_error(HG_EALIGN, "x/W not 16-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    gemv_set_tc_min_batch(c->cfg.gemv_tc_min_batch);
    HG_TRY(stream_guard(c, s));
    HG_TRY(gemv(c, x, batch, K, W, n, bias, y, ldy, s));
    HG_CK(c, cudaEventRecord(c->ev_done, s));
    return HG_OK;
}

HG_API hg_status hg_gemv_replay(hg_ctx *c, const hg_plan_t *p, const void *x, const void *W_dev,
                                const float *bias, float *y, int64_t seq0, void *stream) {
    if (!c || !p) return set_error(HG_EINVAL, "NULL argument");
    if (c->error) return set_error(HG_ESTATE, "context is in an error state");
    if (c->device < 0) return set_error(HG_ESTATE, "host-only context");
    HG_CK(c, cudaSetDevice(c->device));
    HG_TRY(validate_plan(c, *p));
    HG_TRY(check_ptr(c, x, true, "x"));
    HG_TRY(check_ptr(c, y, true, "y"));
    if (p->n_res > 0) HG_TRY(check_ptr(c, W_dev, true, "W_dev"));
    if (bias) HG_TRY(check_ptr(c, bias, true, "bias"));
    const int B = (int)p->batch;
    gemv_set_tc_min_batch(c->cfg.gemv_tc_min_batch);
    if (p->n_chunks > c->nslots) return set_error(HG_EINVAL, "plan has more chunks than ring slots");
    if (seq0 < 0) return set_error(HG_EINVAL, "seq0 < 0");
    if (gemv_use_tc(B, p->K) && !(c->tc_stream && gemv_tc_stream_ok(p->n_res, p->n_str > 0 ? p->n_chunks : 0))) {
        // tcgen05 batches without the persistent launch: the step launches the resident block,
        // then one GEMV per chunk (each gated by stream memops, skipped here)
        cudaStream_t s = (cudaStream_t)stream;
        HG_TRY(stream_guard(c, s));
        if (p->n_res > 0) HG_TRY(gemv(c, x, B, p->K, W_dev, p->n_res, bias, y, p->N, s));
        for (int64_t i = 0; p->n_str > 0 && i < p->n_chunks; ++i) {
            const int64_t r0 = i * p->chunk_rows;
            const int64_t rows = std::min(p->chunk_rows, p->n_str - r0);
            const int64_t g0 = p->n_res + r0;
            HG_TRY(gemv(c, x, B, p->K, c->ring + ((seq0 + i) % c->nslots) * c->slot_bytes, rows,
                        bias ? bias + g0 : nullptr, y + g0, p->N, s));
        }
        HG_CK(c, cudaEventRecord(c->ev_done, s));
        return HG_OK;
    }
    const int64_t n = p->n_res + p->n_str;
    if (gemv_ws_floats(n, p->K, B) > c->ws_floats) return set_error(HG_EINVAL, "workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    HG_TRY(stream_guard(c, s));
    StreamLaunch S{};
    S.x = x;
    S.batch = B;
    S.K = p->K;
    S.W_res = W_dev;
    S.n_res = p->n_res;
    S.ring = c->ring;
    S.slot_bytes = c->slot_bytes;
    S.nslots = c->nslots;
    S.seq0 = seq0;
    S.n_chunks = p->n_str > 0 ? p->n_chunks : 0;
    S.chunk_rows = p->chunk_rows;
    S.n_str = p->n_str;
    S.arrived = nullptr;  // chunks taken as present: no tags, nothing signalled
    S.bias = bias;
    S.y = y;
    S.ldy = p->N;
    S.ws = c->ws;
    S.gbar = c->gbar;
    S.err = c->err;
    S.timeout_s = c->cfg.timeout_s;
    if (gemv_use_tc(B, p->K)) {
        if (gemv_tc_stream_tiles(p->n_res, p->n_str, p->chunk_rows, S.n_chunks) > c->n_counters)
            return set_error(HG_EINVAL, "tcgen05 GEMV: too many tiles for the context's counters");
        HG_TRY(kerr(c, launch_gemv_tc_stream(S, c->counters, s), "gemv tcgen05 replay"));
    } else {
        HG_TRY(kerr(c, launch_gemv_stream(S, s), "gemv replay"));
    }
    HG_CK(c, cudaEventRecord(c->ev_done, s));
    return HG_OK;
}

HG_API hg_status hg_debug_gemv_stamps(uint64_t **out) {
    if (!out) {
        gemv_stamps_enable(false);
        return HG_OK;
    }
    unsigned long long *p = gemv_stamps_enable(true);
    if (!p) return set_error(HG_ECUDA, "cannot allocate mapped stamp memory");
    *out = (uint64_t *)p;
    return HG_OK;
}

HG_API hg_status hg_host_gemv(hg_ctx *c, const void *x, int batch, int64_t n, int64_t K,
                              const void *W, const float *bias, float *y) {
    if (!c || !x || !W || !y) return set_error(HG_EINVAL, "NULL argument");
    if (batch < 1 || batch > HG_MAX_BATCH || n < 0 || K <= 0)
        return set_error(HG_EINVAL, "hg_host_gemv: bad shape");
    if (K % 8) return set_error(HG_EALIGN, "K %% 8 != 0");
    HostJob job;
    job.fn = host_fn_for(c, batch);
    job.x = (const uint16_t *)x;
    job.batch = batch;
    job.K = K;
    job.n = n;
    job.W = (const uint16_t *)W;
    job.bias = bias;
    job.y = y;
    job.ldy = n;
    job.block = 16;
    job.next.store(0);
    host_gemv_new_job();
    pool_run(c->pool, host_job_run, &job);
    return HG_OK;
}

HG_API hg_status hg_gather_permute(hg_ctx *c, const float *gathered, int nranks, int batch, int64_t n_local,
                                   float *y, void *stream) {
    if (!c || !gathered || !y) return set_error(HG_EINVAL, "NULL argument");
    if (c->error) return set_error(HG_ESTATE, "context is in an error state");
    if (c->device < 0) return set_error(HG_ESTATE, "host-only context");
    if (nranks < 1 || batch < 1 || batch > HG_MAX_BATCH || n_local < 0)
        return set_error(HG_EINVAL, "hg_gather_permute: bad shape");
    HG_CK(c, cudaSetDevice(c->device));
    HG_TRY(check_ptr(c, gathered, true, "gathered"));
    HG_TRY(check_ptr(c, y, true, "y"));
    cudaStream_t s = (cudaStream_t)stream;
    HG_TRY(stream_guard(c, s));
    if (n_local > 0) HG_TRY(kerr(c, launch_gather_permute(gathered, nranks, batch, n_local, y, s), "gather permute"));
    c->st.gpu_launches++;
    HG_CK(c, cudaEventRecord(c->ev_done, s));
    return HG_OK;
}

HG_API hg_status hg_peer_export(hg_ctx *c, int nranks, int rank, void *blob) {
    if (!c || !blob) return set_error(HG_EINVAL, "NULL argument");
    if (c->device < 0) return set_error(HG_ESTATE, "host-only context");
    if (c->dist) return set_error(HG_ESTATE, "NCCL group already initialised (hg_dist_init)");
    if (c->peer && (peer_nranks(c->peer) != nranks || peer_rank(c->peer) != rank))
        return set_error(HG_ESTATE, "peer group already exported with another shape");
    HG_CK(c, cudaSetDevice(c->device));
    // device box: a gathered y [B, N] or the P partials [P][B][N] of an all-reduce; host slot: a y
    const int64_t floats = (int64_t)HG_MAX_BATCH * c->cfg.max_n;
    PeerGroup *g = c->peer;
    HG_TRY(peer_export(&g, c->device, nranks, rank, floats * nranks, floats, blob));
    c->peer_pending = g;
    return HG_OK;
}

HG_API hg_status hg_peer_open(hg_ctx *c, const void *blobs) {
    if (!c || !blobs) return set_error(HG_EINVAL, "NULL argument");
    if (!c->peer_pending) return set_error(HG_ESTATE, "hg_peer_export not called");
    HG_CK(c, cudaSetDevice(c->device));
    HG_TRY(peer_open(c->peer_pending, blobs));
    c->peer = c->peer_pending;
    // every buffer a call may need, allocated now: an allocation inside a call (cudaMalloc,
    // cudaHostAlloc) can wait for the device to go idle -- a deadlock when another rank on the same
    // device is spinning on this rank's next push
    const int64_t n = (int64_t)HG_MAX_BATCH * c->cfg.max_n;
    HG_TRY(ensure(c, (void **)&c->ylocal, &c->ylocal_elems, n * 4));
    HG_TRY(ensure(c, &c->act, &c->act_elems, n * 2));
    HG_TRY(ensure(c, (void **)&c->yscr, &c->yscr_elems, n * 4));
    HG_TRY(ensure(c, &c->h1, &c->h1_elems, n * 2));
    HG_TRY(ensure_mirror(c));
    if (c->cfg.pageable) HG_TRY(ensure_pinlane(c));
    HG_CK(c, cudaDeviceSynchronize());
    return HG_OK;
}

HG_API hg_status hg_debug_peer_words(hg_ctx *c, uint32_t *out) {
    if (!c || !out || !c->peer) return set_error(HG_EINVAL, "no peer group");
    cudaSetDevice(c->device);
    peer_debug_words(c->peer, out);
    return HG_OK;
}

HG_API hg_status hg_dist_unique_id(void *id128) {
    if (!id128) return set_error(HG_EINVAL, "NULL id");
    return dist_unique_id(id128);
}

HG_API hg_status hg_dist_init(hg_ctx *c, int nranks, int rank, const void *id128) {
    if (!c || !id128 || nranks < 1 || rank < 0 || rank >= nranks)
        return set_error(HG_EINVAL, "bad arguments");
    if (c->device < 0) return set_error(HG_ESTATE, "host-only context");
    if (c->dist) return set_error(HG_ESTATE, "already initialised");
    HG_CK(c, cudaSetDevice(c->device));
    hg_status st = HG_OK;
    c->dist = dist_create(nranks, rank, id128, &st);
    return st;
}

HG_API hg_status hg_numa_node(int device, int *node) {
    if (!node) return set_error(HG_EINVAL, "NULL node");
    *node = numa_node_of_device(device);
    return HG_OK;
}

HG_API hg_status hg_numa_cpus(int node, int *cpus, int max, int *n) {
    if (!n || (max > 0 && !cpus)) return set_error(HG_EINVAL, "NULL argument");
    const std::vector<int> v = numa_cpus(node);
    if (v.empty()) return set_error(HG_EINVAL, "NUMA node %d has no cpulist", node);
    for (int i = 0; i < max && i < (int)v.size(); ++i) cpus[i] = v[(size_t)i];
    *n = (int)v.size();
    return HG_OK;
}

HG_API hg_status hg_host_alloc(size_t bytes, int node, int lock, void **ptr) {
    if (!ptr || bytes == 0) return set_error(HG_EINVAL, "bad arguments");
    *ptr = host_alloc_node(bytes, node, lock != 0);
    if (!*ptr) return set_error(HG_ENOMEM, "host_alloc of %zu bytes on node %d failed", bytes, node);
    return HG_OK;
}

HG_API hg_status hg_host_free(void *ptr, size_t bytes, int lock) {
    host_free_node(ptr, bytes, lock != 0);
    return HG_OK;
}

HG_API hg_status hg_numa_node_of_ptr(const void *ptr, int *node) {
    if (!ptr || !node) return set_error(HG_EINVAL, "NULL argument");
    *node = numa_node_of_page(ptr);
    return HG_OK;
}

HG_API hg_status hg_stats(hg_ctx *c, hg_stats_t *out) {
    if (!c || !out) return set_error(HG_EINVAL, "NULL argument");
    if (c->device >= 0 && c->call_timed) {
        HG_CK(c, cudaSetDevice(c->device));
        HG_CK(c, cudaEventSynchronize(c->ev_done));
        HG_TRY(check_device_error(c));
        float ms = 0;
        HG_CK(c, cudaEventElapsedTime(&ms, c->ev_call0, c->ev_call1));
        c->st.wall_s = ms * 1e-3;
        if (c->cfg.collect_stats) {
            HG_TRY(sync_naive(c));
            HG_CK(c, cudaStreamSynchronize(c->copy));
            // busy time inside the calls' window [ev_call0, ev_call1]: the copy stream also runs
            // ahead into chunks of later calls (prefetch), which belong to those calls
            const double wall = c->st.wall_s;
            auto clipped = [&](const std::pair<size_t, size_t> &pr) {
                float a = 0, b = 0;
                if (cudaEventElapsedTime(&a, c->ev_call0, c->tev[pr.first]) != cudaSuccess ||
                    cudaEventElapsedTime(&b, c->ev_call0, c->tev[pr.second]) != cudaSuccess)
                    return 0.0;
                const double t0 = std::min(std::max(a * 1e-3, 0.0), wall);
                const double t1 = std::min(std::max(b * 1e-3, 0.0), wall);
                return t1 > t0 ? t1 - t0 : 0.0;
            };
            // Link time of these calls = the bytes they streamed at the link's measured copy rate.
            // (Busy time inside the window is not it: with a ring larger than a call's streamed
            // bytes the copy stream keeps prefetching later calls' chunks the whole time.)
            double dur = 0, bytes = 0, gpu = 0;
            for (size_t k = 0; k < c->copy_ev.size(); ++k) {
                const double d = clipped(c->copy_ev[k]);
                float full = 0;
                if (d > 0 && cudaEventElapsedTime(&full, c->tev[c->copy_ev[k].first], c->tev[c->copy_ev[k].second]) ==
                                 cudaSuccess && full > 0) {
                    dur += d;
                    bytes += (double)c->copy_bytes[k] * d / (full * 1e-3);
                }
            }
            for (auto &pr : c->gemv_ev) gpu += clipped(pr);
            cudaGetLastError();
            c->st.link_busy_s = (bytes > 0 && dur > 0) ? (double)c->st.bytes_str / (bytes / dur) : 0.0;
            if (c->naive && c->naive->bytes > 0)  // naive strategy: the transfer thread's staged-copy rate
                c->st.link_busy_s = (double)c->st.bytes_str * (c->naive->busy_ns * 1e-9) / (double)c->naive->bytes;
            if (c->cfg.stream_mode == 1) c->st.link_busy_s = gpu;  // zero-copy: the GEMVs are the transfer
            c->st.gpu_busy_s = gpu;
        }
    }
    if (c->pin && c->cfg.strategy == HG_STRATEGY_HYBRID) {  // (pinned-blocking counts its pins as it does them)
        double busy = 0;
        int64_t pinned = 0;
        pinlane_stats(c->pin, &busy, &pinned, false);
        // like the link: the lane runs ahead into later calls' chunks, so the calls' pin time is
        // their streamed bytes at the lane's measured rate
        c->st.bytes_pinned = pinned;
        c->st.pin_busy_s = pinned > 0 ? (double)c->st.bytes_str * busy / (double)pinned : 0.0;
        if (pinlane_error(c->pin)) {
            c->error = true;
            return set_error(HG_ETIMEOUT, "the pin lane waited longer than %.1f s for a staging slot", c->cfg.timeout_s);
        }
    }
    *out = c->st;
    return HG_OK;
}

HG_API hg_status hg_reset_stats(hg_ctx *c) {
    if (!c) return set_error(HG_EINVAL, "NULL ctx");
    if (c->device >= 0 && c->have_last) {  // pending timing events belong to the old window
        HG_CK(c, cudaSetDevice(c->device));
        if (cudaEventSynchronize(c->ev_done) != cudaSuccess) dbg_trace_report(c);
        HG_CK(c, cudaEventSynchronize(c->ev_done));
        HG_TRY(sync_naive(c));
        HG_CK(c, cudaStreamSynchronize(c->copy));
    }
    if (c->pin) {
        double b;
        int64_t n;
        pinlane_stats(c->pin, &b, &n, true);
    }
    if (c->naive) {  // the lane's counters restart with the stats window
        c->naive->busy_ns = 0;
        c->naive->bytes = 0;
    }
    c->tev_used = 0;
    c->copy_ev.clear();
    c->copy_bytes.clear();
    c->gemv_ev.clear();
    c->stats_open = false;
    c->call_timed = false;
    std::memset(&c->st, 0, sizeof c->st);
    return HG_OK;
}

// ---------------------------------------------------------------- alpha benchmark
HG_API hg_status hg_alpha_bench(hg_ctx *c, const hg_opt_layer *layers, int n_layers, void *h, int batch,
                                double alpha_seed, const hg_abench_cfg *cfg_in, hg_abench_result *out,
                                void *stream) {
    if (!c || !layers || n_layers < 1 || !h || !out) return set_error(HG_EINVAL, "NULL argument");
    if (!(alpha_seed >= 0.0 && alpha_seed <= 1.0)) return set_error(HG_EINVAL, "alpha_seed outside [0,1]");
    hg_abench_cfg cfg = {0.06, 0.02, 2, 1, 1, 0};
    if (cfg_in) cfg = *cfg_in;
    if (!(cfg.gamma > 0) || !(cfg.lambda > 0) || cfg.reps < 1 || cfg.degree < 1)
        return set_error(HG_EINVAL, "bad alpha-bench config");
    const int max_rounds = cfg.max_rounds > 1 ? cfg.max_rounds : 1;
    std::vector<hg_opt_layer> work(layers, layers + n_layers);
    hg_rates unit = {1, 1, 1, 1, 1, 1, 1};
    double seed = alpha_seed;
    for (int round = 1;; ++round) {
        // window [seed - gamma, seed + gamma] cap [0, 1] in steps of lambda (reading R9)
        const double lo = std::max(0.0, seed - cfg.gamma), hi = std::min(1.0, seed + cfg.gamma);
        std::vector<double> pts;
        const int npts = (int)std::floor((hi - lo) / cfg.lambda + 1e-9) + 1;
        for (int i = 0; i < npts && (int)pts.size() < HG_ABENCH_MAX; ++i) pts.push_back(lo + i * cfg.lambda);
        if (hi - pts.back() > 1e-12 && (int)pts.size() < HG_ABENCH_MAX) pts.push_back(hi);
        if ((int)pts.size() < cfg.degree + 1) return set_error(HG_EINVAL, "window has too few alphas");
        const int saved_stats = c->cfg.collect_stats;
        c->cfg.collect_stats = 1;
        std::memset(out, 0, sizeof *out);
        out->alpha_seed = seed;
        hg_status st = HG_OK;
        for (size_t i = 0; i < pts.size() && st == HG_OK; ++i) {
            for (auto &L : work)
                for (int j = 0; j < 4 && st == HG_OK; ++j) {
                    const hg_plan_t &p = L.lin[j].plan;
                    st = hg_plan(&unit, p.N, p.K, batch, p.n_res, HG_ALPHA_FIXED, pts[i], p.granule,
                                 c->cfg.chunk_bytes, &L.lin[j].plan);
                }
            if (st != HG_OK) break;
            st = hg_stack(c, work.data(), n_layers, h, batch, stream);  // warm the pipeline at this alpha
            if (st == HG_OK) st = hg_reset_stats(c);
            for (int r = 0; r < cfg.reps && st == HG_OK; ++r) st = hg_stack(c, work.data(), n_layers, h, batch, stream);
            hg_stats_t s;
            if (st == HG_OK) st = hg_stats(c, &s);
            if (st == HG_OK) {
                out->alpha[i] = pts[i];
                out->t_cpu[i] = s.cpu_busy_s / cfg.reps;
                out->t_com[i] = s.link_busy_s / cfg.reps;
                out->t_step[i] = s.wall_s / cfg.reps;
                out->t_pin[i] = s.pin_busy_s / cfg.reps;
            }
        }
        c->cfg.collect_stats = saved_stats;
        if (st != HG_OK) return st;  // keep the failing call's message (hg_reset_stats would overwrite it)
        HG_TRY(hg_reset_stats(c));
        out->n = (int)pts.size();
        // F_COM = max(F_PIN, F_TRANS): the pin lane counts when it did any work
        bool pinned_any = false;
        for (int i = 0; i < out->n; ++i) pinned_any |= out->t_pin[i] > 0;
        HG_TRY(hg_alpha_solve(out->alpha, out->t_cpu, out->t_com, pinned_any ? out->t_pin : nullptr, out->n,
                              cfg.degree, pts.front(), pts.back(), seed, &out->alpha_bar, &out->clamped));
        out->rounds = round;
        // no balance point inside the window: re-centre it on the clamped edge
        if (!out->clamped || round >= max_rounds || !(out->alpha_bar > 0.0 && out->alpha_bar < 1.0)) break;
        seed = out->alpha_bar;
    }
    out->alpha_seed = alpha_seed;
    return HG_OK;
}

// T-bar_CPU for the scheduler's gain: the CPU lane's rate on this module's weight.
HG_API hg_status hg_module_tcpu(hg_ctx *c, const void *W_host, int64_t N, int64_t K, int batch, double alpha,
                                double *t_cpu, double *rate_out) {
    if (!c || !W_host || !t_cpu) return set_error(HG_EINVAL, "NULL argument");
    if (N <= 0 || K <= 0 || K % 8 || batch < 1 || batch > HG_MAX_BATCH || !(alpha >= 0.0 && alpha <= 1.0))
        return set_error(HG_EINVAL, "hg_module_tcpu: bad shape or alpha");
    std::vector<uint16_t> x((size_t)batch * K, 0x3f80);
    std::vector<float> y((size_t)batch * N);
    std::vector<double> ts;
    for (int it = 0; it < 3; ++it) {
        const auto t0 = clk::now();
        HG_TRY(hg_host_gemv(c, x.data(), batch, N, K, W_host, nullptr, y.data()));
        ts.push_back(secs(t0, clk::now()));
    }
    std::sort(ts.begin(), ts.end());
    const double rate = (double)(2 * N * K) / ts[1];
    *t_cpu = (1.0 - alpha) * (double)(2 * N * K) / rate;
    if (rate_out) *rate_out = rate;
    return HG_OK;
}

// ---------------------------------------------------------------- measurement
HG_API hg_status hg_measure(hg_ctx *c, const void *W_host, int64_t N, int64_t K, int batch,
                            int flags, hg_rates *out) {
    if (!c || !W_host || !out) return set_error(HG_EINVAL, "NULL argument");
    if (c->error) return set_error(HG_ESTATE, "context is in an error state");
    if (c->device < 0) return set_error(HG_ESTATE, "host-only context");
    if (N <= 0 || K <= 0 || K % 8 || batch < 1 || batch > HG_MAX_BATCH || K > c->cfg.max_k ||
        N > c->cfg.max_n)
        return set_error(HG_EINVAL, "hg_measure: bad shape");
    HG_CK(c, cudaSetDevice(c->device));
    gemv_set_tc_min_batch(c->cfg.gemv_tc_min_batch);
    HG_TRY(check_ptr(c, W_host, false, "W_host"));
    // the ring is reused below: release every prefetched chunk, then wait for the device
    HG_TRY(pump(c));
    HG_TRY(drop_inflight(c));
    c->future.clear();
    c->fpos = 0;
    // this context's streams only (ranks sharing the device may be mid-exchange)
    HG_TRY(sync_naive(c));
    if (c->have_last) HG_CK(c, cudaEventSynchronize(c->ev_done));
    HG_CK(c, cudaStreamSynchronize(c->copy));
    if (c->d2h) HG_CK(c, cudaStreamSynchronize(c->d2h));
    HG_TRY(check_device_error(c));
    std::fill(c->slot_used.begin(), c->slot_used.end(), 0);

    const int64_t wbytes = 2 * N * K;
    const int64_t ring_bytes = (int64_t)c->nslots * c->slot_bytes;
    cudaEvent_t e0, e1;
    HG_CK(c, cudaEventCreate(&e0));
    HG_CK(c, cudaEventCreate(&e1));
    float ms = 0;
    // pageable weight (hg_config.pageable): the link is probed from the pin lane's staging ring and
    // V_PIN is the lane's own rate (Eq. (9)); pinned weight: V_PIN = +inf (reading R7)
    // (naive strategy, Fig. 5a: no pin lane; the link is probed straight from the pageable rows)
    const bool pageable = c->cfg.pageable && is_pageable(W_host) && c->cfg.strategy != HG_STRATEGY_NAIVE;
    const uint8_t *src = (const uint8_t *)W_host;
    int64_t lbytes = wbytes;
    double v_pin = INFINITY;
    if (c->cfg.pageable && is_pageable(W_host) && c->cfg.strategy == HG_STRATEGY_NAIVE)
        lbytes = std::min<int64_t>(wbytes, (int64_t)c->nslots * c->slot_bytes);
    if (pageable) {
        HG_TRY(ensure_pinlane(c));
        lbytes = std::min<int64_t>(wbytes, (int64_t)c->nstage * c->slot_bytes);
        std::vector<double> tp;
        for (int it = 0; it < 3; ++it) tp.push_back(pinlane_copy_timed(c->pin, c->staging, W_host, lbytes));
        std::sort(tp.begin(), tp.end());
        v_pin = (double)lbytes / tp[1];
        src = c->staging;
    }

    // link: chunk-sized copies (v_link) and one large copy (b_link)
    const int64_t C = chunk_rows_for(K, c->cfg.granule, c->cfg.chunk_bytes);
    const int64_t chunk = std::min<int64_t>(C * K * 2, lbytes);
    int64_t total = 0;
    // warm-up: first DMA over these pages and ring addresses is not representative
    HG_CK(c, cudaMemcpyAsync(c->ring, src, std::min<int64_t>(lbytes, ring_bytes), cudaMemcpyHostToDevice,
                             c->copy));
    HG_CK(c, cudaEventRecord(e0, c->copy));
    for (int64_t off = 0; off + chunk <= lbytes && total < (512ll << 20); off += chunk) {
        HG_CK(c, cudaMemcpyAsync(c->ring + (total % (ring_bytes - chunk + 1)) / 256 * 256, src + off,
                                 chunk, cudaMemcpyHostToDevice, c->copy));
        total += chunk;
    }
    HG_CK(c, cudaEventRecord(e1, c->copy));
    HG_CK(c, cudaEventSynchronize(e1));
    HG_CK(c, cudaEventElapsedTime(&ms, e0, e1));
    out->v_link = (double)total / (ms * 1e-3);
    const int64_t big = std::min<int64_t>(std::min<int64_t>(lbytes, ring_bytes), 512ll << 20);
    HG_CK(c, cudaEventRecord(e0, c->copy));
    HG_CK(c, cudaMemcpyAsync(c->ring, src, big, cudaMemcpyHostToDevice, c->copy));
    HG_CK(c, cudaEventRecord(e1, c->copy));
    HG_CK(c, cudaEventSynchronize(e1));
    HG_CK(c, cudaEventElapsedTime(&ms, e0, e1));
    out->b_link = (double)big / (ms * 1e-3);

    // GPU: GEMV over the rows now in the ring (>= L2 size when the weight allows)
    const int64_t rows = std::min<int64_t>(N, big / (2 * K));
    void *px = nullptr, *py = nullptr;
    HG_CK(c, cudaMalloc(&px, (size_t)batch * K * 2));
    HG_CK(c, cudaMalloc(&py, (size_t)batch * rows * 4));
    HG_CK(c, cudaMemset(px, 0, (size_t)batch * K * 2));  // x = 0 (values irrelevant to timing)
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
        HG_CK(c, cudaEventRecord(e0, c->copy));
        HG_TRY(kerr(c, launch_gemv(px, batch, K, c->ring, rows, nullptr, (float *)py, rows, c->ws,
                                   c->counters, c->gbar, c->err, c->copy), "gemv probe"));
        HG_CK(c, cudaEventRecord(e1, c->copy));
        HG_CK(c, cudaEventSynchronize(e1));
        HG_CK(c, cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
    }
    out->v_gpu = (double)rows * K * 2 / (best * 1e-3);
    HG_CK(c, cudaStreamSynchronize(c->copy));
    cudaFree(px);
    cudaFree(py);
    best = 1e30f;
    for (int it = 0; it < 5; ++it) {
        HG_CK(c, cudaEventRecord(e0, c->copy));
        HG_TRY(kerr(c, launch_read_bw(c->ring, ring_bytes, c->sink, c->copy), "read probe"));
        HG_CK(c, cudaEventRecord(e1, c->copy));
        HG_CK(c, cudaEventSynchronize(e1));
        HG_CK(c, cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
    }
    out->b_hbm = (double)ring_bytes / (best * 1e-3);

    // CPU lane: the pool's GEMV over the whole weight and the pool's read bandwidth, optionally
    // while the link streams (flags bit 0: both lanes read the same host DRAM).  Medians of many
    // short runs: single runs on a shared host are noisy.
    std::vector<uint16_t> xh((size_t)batch * K, 0x3f80);
    std::vector<float> yh((size_t)batch * N);
    // A weight that is not much larger than the host's last-level cache would be measured from
    // cache: every timed CPU probe is preceded by a read of a 256 MiB scratch buffer.
    const int64_t sbytes = 256ll << 20;
    std::vector<uint8_t> scratch((size_t)sbytes, 1);
    // 512 chunks of <= 32 MiB ~ 16 GiB ~ 300 ms of link time: three 80 ms windows fit inside it, and
    // whole-chunk counting at the window edges is within +-0.4% of the ~18 GB a window moves
    const int NB = (flags & 1) ? 512 : 0;
    std::vector<cudaEvent_t> evb((size_t)NB, nullptr);
    for (int i = 0; i < NB; ++i) HG_CK(c, cudaEventCreateWithFlags(&evb[i], cudaEventDisableTiming));
    for (int64_t off = 0, n = 0; n < NB; ++n, off = (off + chunk) % (lbytes - chunk + 1)) {
        HG_CK(c, cudaMemcpyAsync(c->ring, src + off / 256 * 256, chunk, cudaMemcpyHostToDevice, c->copy));
        HG_CK(c, cudaEventRecord(evb[n], c->copy));
    }
    auto completed = [&]() {
        int n = 0;
        while (n < NB && cudaEventQuery(evb[n]) == cudaSuccess) ++n;
        cudaGetLastError();
        return n;
    };
    struct RJ { const uint8_t *p; int64_t bytes, block; std::atomic<int64_t> next; std::atomic<uint64_t> sum; };
    RJ rj;
    rj.block = 1 << 20;
    auto read_region = [&](const uint8_t *p, int64_t bytes) {
        rj.p = p;
        rj.bytes = bytes;
        rj.next.store(0);
        rj.sum.store(0);
        pool_run(c->pool, [](void *a, int) {
            RJ *r = (RJ *)a;
            const int64_t nb = (r->bytes + r->block - 1) / r->block;
            uint64_t s = 0;
            for (;;) {
                int64_t b = r->next.fetch_add(1);
                if (b >= nb) break;
                int64_t len = std::min(r->block, r->bytes - b * r->block);
                if (!strcmp(hg_host_isa(), "avx512bf16")) s ^= host_read_avx512(r->p + b * r->block, len);
                else for (int64_t i = 0; i < len; i += 64) s += r->p[b * r->block + i];
            }
            r->sum.fetch_xor(s);
        }, &rj);
    };
    auto flush_llc = [&]() { read_region(scratch.data(), sbytes); };
    auto read_pass = [&]() { read_region((const uint8_t *)W_host, wbytes); };
    auto median = [](std::vector<double> v) {
        std::sort(v.begin(), v.end());
        return v[v.size() / 2];
    };
    out->b_host = 0;
    if (NB > 0) {  // joint host-DRAM rate: CPU reads + DMA reads in the same window (a peak: max of 3)
        read_pass();  // warm
        for (int w = 0; w < 3; ++w) {
            const int n0 = completed();
            const auto t0 = clk::now();
            int64_t cpu_bytes = 0;
            while (secs(t0, clk::now()) < 0.08) {  // weight + scratch: a footprint far above the LLC
                read_pass();
                flush_llc();
                cpu_bytes += wbytes + sbytes;
            }
            const int n1 = completed();
            const double dt = secs(t0, clk::now());
            if (n1 < NB && n1 > n0)
                out->b_host = std::max(out->b_host, ((double)cpu_bytes + (double)(n1 - n0) * chunk) / dt);
        }
    }
    // the solo CPU probes below must not share host DRAM with the joint probe's remaining DMA
    HG_CK(c, cudaStreamSynchronize(c->copy));
    std::vector<double> tg, tr;
    for (int it = 0; it < 9; ++it) {
        flush_llc();
        auto t0 = clk::now();
        HG_TRY(hg_host_gemv(c, xh.data(), batch, N, K, W_host, nullptr, yh.data()));
        tg.push_back(secs(t0, clk::now()));
    }
    out->v_cpu = (double)wbytes / median(tg);
    for (int it = 0; it < 9; ++it) {
        flush_llc();
        auto t0 = clk::now();
        read_pass();
        tr.push_back(secs(t0, clk::now()));
    }
    out->b_cpu = (double)wbytes / median(tr);
    // both lanes together move at least what either moves alone; a lower joint probe is noise
    if (out->b_host > 0) out->b_host = std::max(out->b_host, std::max(out->b_cpu, out->b_link));
    HG_CK(c, cudaStreamSynchronize(c->copy));
    for (auto e : evb) cudaEventDestroy(e);
    out->v_pin = v_pin;
    HG_CK(c, cudaStreamSynchronize(c->copy));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return HG_OK;
}

}  // extern "C"
