// hg_internal.h -- declarations shared by the library's translation units.
// Not part of the ABI (include/hg.h is).
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "hg.h"

namespace hg {

// ---------------------------------------------------------------- errors
// Thread-local last-error message; returns `st` so call sites can `return set_error(...)`.
hg_status set_error(hg_status st, const char *fmt, ...) __attribute__((format(printf, 2, 3)));

// ---------------------------------------------------------------- plan.cpp
hg_status partition_rows(int64_t N, int64_t n_res, double alpha, int64_t G, int64_t *n_str,
                         int64_t *n_cpu);
int64_t chunk_rows_for(int64_t K, int64_t G, int64_t chunk_bytes);

// ---------------------------------------------------------------- gemv_sm100.cu
// Deterministic split-K geometry: depends on K only, so every output element is
// reduced in the same order whichever launch (resident / chunk) computes it.
struct GemvGeom {
    int64_t ks;      // k-slice length (elements, multiple of 256 unless == K)
    int s;           // number of k-slices
    int rows_per_cta;
};
GemvGeom gemv_geom(int64_t K, int batch);
// Workspace floats and counters needed for one launch over n rows.
int64_t gemv_ws_floats(int64_t n, int64_t K, int batch);
int64_t gemv_counters(int64_t n, int64_t K, int batch);
// Launch: y[b*ldy + j] = sum_k x[b,k] W[j,k] (+bias[j]), j < n.  Returns a CUDA error code (int).
// ws/counters: split-K workspace (tcgen05) or part sums (SIMT, P > 1); gbar: 2 zeroed words
// for the SIMT grid barrier; err: device error word (timeouts).
int launch_gemv(const void *x, int batch, int64_t K, const void *W, int64_t n, const float *bias,
                float *y, int64_t ldy, float *ws, int *counters, uint32_t *gbar, uint32_t *err,
                void *stream);
bool gemv_use_tc(int batch, int64_t K);

// One persistent SIMT launch over the GPU lanes of a linear: resident rows [0, n_res) of W_res,
// then streamed chunk c (rows [n_res + c*chunk_rows, ...)) in ring slot (seq0 + c) % nslots.
// With `arrived` set the kernel waits for arrived[slot] >= seq+1 (copy stream's
// cuStreamWriteValue32) before reading a chunk and, once every CTA has drained it, writes
// consumed[slot] = seq+1 (the copy stream's cuStreamWaitValue32 before reusing the slot).
// With arrived == NULL the chunks are taken as present (no tags).  Rows of y are global.
struct StreamLaunch {
    const void *x;
    int batch;
    int64_t K;
    const void *W_res;
    int64_t n_res;
    const void *W_dir = nullptr;  // zero-copy streamed rows [n_res, n_res + n_dir) (mapped pinned host)
    int64_t n_dir = 0;
    const uint8_t *ring;
    int64_t slot_bytes, nslots;
    int64_t seq0, n_chunks, chunk_rows, n_str;
    const uint32_t *arrived;
    uint32_t *consumed, *slot_cnt;
    const float *bias;
    float *y;
    int64_t ldy;
    float *ws;
    uint32_t *gbar;
    uint32_t *err;
    double timeout_s;
    volatile uint32_t *trace = nullptr;  // debug trace words (mapped host) or NULL
    uint32_t trace_id = 0;
};
// SIMT GEMV per-row-group part counters (P > 1) after the 4 words of gbar
constexpr int kGroupCounters = 1024;
int launch_gemv_stream(const StreamLaunch &L, void *stream);
unsigned long long *gemv_stamps_enable(bool on);
unsigned long long *gemv_stamps_dev();  // NULL unless hg_debug_gemv_stamps enabled them

// ---------------------------------------------------------------- glue_sm100.cu
int launch_join(float *y, int64_t ldy, int64_t col0, int64_t ncols, int batch, const float *ycpu,
                int64_t ldsrc, const float *bias, void *stream);
int launch_layernorm(const void *h, int64_t H, int batch, const float *g, const float *b, void *out,
                     void *stream);
int launch_slice_to_bf16(const float *y, int64_t ldy, int64_t col0, int64_t ncols, int batch,
                         void *out, void *stream);
int launch_residual_ln(const void *h, const float *y, int64_t H, int batch, void *h1,
                       const float *g, const float *b, void *a2, void *stream);
int launch_relu_bf16(const float *y, int64_t n, int batch, void *out, void *stream);
int launch_residual(const void *h1, const float *y, int64_t H, int batch, void *out, void *stream);
int launch_gather_permute(const float *gbuf, int P, int batch, int64_t n_local, float *y,
                          void *stream);
int launch_read_bw(const void *p, int64_t bytes, float *sink, void *stream);

// ---------------------------------------------------------------- host_gemv*.cpp
// One block of rows [r0, r1) of the CPU lane: y[b*ldy + (r - r0) + yoff] ...
typedef void (*host_rows_fn)(const uint16_t *x, int batch, int64_t K, const uint16_t *W,
                             int64_t r0, int64_t r1, const float *bias, float *y, int64_t ldy);
void host_rows_avx512bf16(const uint16_t *x, int batch, int64_t K, const uint16_t *W, int64_t r0,
                          int64_t r1, const float *bias, float *y, int64_t ldy);
void host_rows_avx2(const uint16_t *x, int batch, int64_t K, const uint16_t *W, int64_t r0,
                    int64_t r1, const float *bias, float *y, int64_t ldy);
void host_rows_scalar(const uint16_t *x, int batch, int64_t K, const uint16_t *W, int64_t r0,
                      int64_t r1, const float *bias, float *y, int64_t ldy);
host_rows_fn host_rows_select(const char **name);
// AMX-BF16 tiles (batch >= 4 by default); host_amx_enable() asks the OS for tile state once.
void host_rows_amx(const uint16_t *x, int batch, int64_t K, const uint16_t *W, int64_t r0, int64_t r1,
                   const float *bias, float *y, int64_t ldy);
bool host_amx_enable();
void host_gemv_new_job();  // call before posting a CPU-lane job (AMX repacks its x)
// Host read-bandwidth kernel (probe): returns a checksum so the loads are not elided.
uint64_t host_read_avx512(const void *p, int64_t bytes);

// ---------------------------------------------------------------- host_glue.cpp
// Bit-exact host mirrors of the glue_sm100.cu kernels (bf16 = uint16 bit patterns).  Built with
// AVX2+FMA: hglue_supported() must be true before any of them is called.
bool hglue_supported();
void hglue_layernorm(const uint16_t *h, int64_t H, int batch, const float *g, const float *b, uint16_t *out);
void hglue_residual_ln(const uint16_t *h, const float *y, int64_t ldy, int64_t H, int batch, uint16_t *h1,
                       const float *g, const float *b, uint16_t *a2);
void hglue_residual(const uint16_t *h1, const float *y, int64_t ldy, int64_t H, int batch, uint16_t *out);
void hglue_slice_bf16(const float *y, int64_t ldy, int64_t col0, int64_t ncols, int batch, uint16_t *out);
void hglue_relu_bf16(const float *y, int64_t ldy, int64_t n, int batch, uint16_t *out);

// ---------------------------------------------------------------- pinlane.cpp
struct PinLane;
PinLane *pinlane_create(int threads, uint8_t *staging, int64_t slot_bytes, int nslots, volatile uint32_t *pinned,
                        volatile uint32_t *freed, double timeout_s);
void pinlane_destroy(PinLane *p);
// Copy [src, src+bytes) into staging slot `slot`, then publish pinned[slot] = tag (asynchronous, FIFO).
void pinlane_submit(PinLane *p, const void *src, int64_t bytes, int slot, uint32_t tag);
bool pinlane_error(const PinLane *p);
void pinlane_stats(PinLane *p, double *busy_s, int64_t *bytes, bool reset);
double pinlane_copy_timed(PinLane *p, void *dst, const void *src, int64_t bytes);

// ---------------------------------------------------------------- threadpool.cpp
class ThreadPool;
ThreadPool *pool_create(int nthreads, int first_core);
// workers pinned to cpus[i % cpus.size()] (worker 0 is the caller's thread and is not pinned)
ThreadPool *pool_create_cpus(int nthreads, const std::vector<int> &cpus);

// Device-side bounded waits use timeout_s x this (HG_DEV_TIMEOUT_SCALE, default 1; debugging: < 1
// lets the kernels give up -- and print what they waited for -- before the host's own waits do).
inline double dev_timeout_scale() {
    static const double s = getenv("HG_DEV_TIMEOUT_SCALE") ? atof(getenv("HG_DEV_TIMEOUT_SCALE")) : 1.0;
    return s > 0 ? s : 1.0;
}

// peer.cu: the a8 exchange over peer memory (device pushes + flags; shared host segment)
constexpr int kMaxPeers = 8;
constexpr int kDevSlots = 4;
struct PeerGroup;
hg_status peer_export(PeerGroup **pg, int device, int nranks, int rank, int64_t box_floats, int64_t host_floats,
                      void *blob_out);
hg_status peer_open(PeerGroup *g, const void *blobs);
void peer_destroy(PeerGroup *g);
int peer_nranks(const PeerGroup *g);
void peer_debug_words(PeerGroup *g, uint32_t *out);
int peer_rank(const PeerGroup *g);
int peer_exchange(PeerGroup *g, const float *ylocal, int B, int64_t n_local, float *y, int64_t ldy, uint32_t *err,
                  double timeout_s, void *stream);
int peer_reduce(PeerGroup *g, const float *partial, int B, int64_t N, const float *bias, float *y, int64_t ldy,
                uint32_t *err, double timeout_s, void *stream);
float *peer_host_y(PeerGroup *g, int64_t k);
float *peer_host_y_dev(PeerGroup *g, int64_t k);
int peer_host_slots();
void peer_host_publish(PeerGroup *g, int64_t k);
hg_status peer_host_wait_ready(PeerGroup *g, int64_t k, double timeout_s);
void peer_host_consumed(PeerGroup *g, int64_t k);
hg_status peer_host_wait_free(PeerGroup *g, int64_t k, double timeout_s);

// numa.cpp: host placement of a rank
std::vector<int> parse_cpulist(const char *s);
int numa_node_of_device(int device);
std::vector<int> numa_cpus(int node);
void *host_alloc_node(size_t bytes, int node, bool lock);
void host_free_node(void *p, size_t bytes, bool locked);
int numa_node_of_page(const void *p);
void pool_destroy(ThreadPool *p);
int pool_size(const ThreadPool *p);
// Run fn(arg, worker_index) on every worker (the caller is worker 0); returns when all finished.
void pool_run(ThreadPool *p, void (*fn)(void *, int), void *arg);
// Asynchronous form: post() starts workers 1..n-1; join() runs worker 0 on the caller and waits.
void pool_post(ThreadPool *p, void (*fn)(void *, int), void *arg);
void pool_join(ThreadPool *p);

}  // namespace hg

namespace hg {
// ---------------------------------------------------------------- dist.cpp (NCCL, dlopen'ed)
struct Dist;
hg_status dist_unique_id(void *id128);
Dist *dist_create(int nranks, int rank, const void *id128, hg_status *st);
void dist_destroy(Dist *d);
int dist_nranks(const Dist *d);
int dist_rank(const Dist *d);
hg_status dist_allgather(Dist *d, const float *send, float *recv, size_t count_per_rank,
                         void *stream);
// gemv kernel attributes (dynamic smem) for the current device
int gemv_prepare();
void gemv_set_tc_min_batch(int b);
// gemv_tc_sm100.cu: tcgen05 path (batch 5..8)
GemvGeom gemv_tc_geom(int64_t K);
int gemv_tc_prepare();
int launch_gemv_tc(const void *x, int batch, int64_t K, const void *W, int64_t n, const float *bias,
                   float *y, int64_t ldy, float *ws, int *counters, void *stream);
// persistent per-linear tcgen05 GEMV (resident block + every streamed chunk, arrival tags)
bool gemv_tc_stream_ok(int64_t n_res, int64_t n_chunks);
int64_t gemv_tc_stream_tiles(int64_t n_res, int64_t n_str, int64_t chunk_rows, int64_t n_chunks);
int launch_gemv_tc_stream(const StreamLaunch &L, int *counters, void *stream);
}  // namespace hg
