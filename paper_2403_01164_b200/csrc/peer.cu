// peer.cu -- the a8 exchange over peer memory (BJ:5 -- not in the paper, which
// uses one A10).
//
// Rank p owns W rows [pN/P, (p+1)N/P) of every linear.  After a linear, every rank needs the full
// y [B, N] -- on the device for the GPU glue, and on the host for the CPU lane's mirrored glue
// (reading R24).  Instead of an NCCL all-gather plus a permute kernel, each rank
//   * device: pushes its [B, N/P] rows straight into every rank's "box" at their global columns
//     (stores through peer pointers: NVLink P2P on a multi-GPU box; plain stores when ranks share
//     a device), then raises its flag in every box; a rank's wait kernel spins until all P flags of
//     the exchange are up and copies the box into the layer's y -- a two-kernel collective with no
//     permute and no host involvement;
//   * host: writes its CPU rows (and, by a D2H, its GPU rows) into one host segment shared by all
//     ranks (POSIX shm), at their global columns, and publishes a ready word; every rank's CPU lane
//     waits for all P ready words and runs the glue on the full y -- no device round trip on the
//     CPU lane's critical path at any P.
// Ranks may be processes (peer pointers from CUDA IPC handles, the host segment mapped by name) or
// threads of one process (pointers used directly) -- the latter runs P > 1 on a single GPU (tests).
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>

#include "hg_internal.h"

namespace hg {

namespace {

#define PEER_TRY(expr)                \
    do {                              \
        hg_status s_ = (expr);        \
        if (s_ != HG_OK) return s_;   \
    } while (0)

constexpr uint32_t kMagic = 0x48475052u;  // "HGPR"
constexpr int kHostSlots = 8;             // host ring depth (linears in flight on the host)

// What a rank tells its peers (HG_PEER_BLOB bytes).
struct Blob {
    uint32_t magic;
    int32_t nranks, rank, device;
    int64_t pid;
    int64_t box_floats;       // per device slot
    int64_t host_floats;      // per host slot
    uint64_t dev_base;        // raw device pointer of this rank's allocation (same-process peers)
    cudaIpcMemHandle_t ipc;   // the same allocation for other processes
    char shm[64];             // rank 0: the host segment's name
};
static_assert(sizeof(Blob) <= 512, "blob");

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

struct PushArgs {
    const float *src;        // this rank's [B][n_local]
    int64_t n_local;
    int64_t dst0, dst_ld;    // element (b, j) lands at box slot + dst0 + b * dst_ld + j
    int B, P, p, slot;
    uint32_t tag;            // exchange sequence + 1
    int64_t box_floats;
    float *box[kMaxPeers];   // every rank's box (slot 0)
    uint32_t *flag[kMaxPeers];        // every rank's flags [kDevSlots][P]
    const uint32_t *done[kMaxPeers];  // every rank's consumed word
    uint32_t *count;         // this rank's CTA counter (zero between launches)
    uint32_t *err;
    unsigned long long timeout_ns;
};

// Push [B][n_local] into every rank's box (all-gather: at columns [p n_local, (p+1) n_local) of
// [B][N_full]; all-reduce: as partial p of [P][B][N]), then raise this rank's flag in every box.  The box slot is reused every kDevSlots exchanges: first wait until every
// rank has copied out the exchange that used it before.
__global__ void peer_push_kernel(const __grid_constant__ PushArgs a) {
    if (threadIdx.x < a.P && a.tag > (uint32_t)kDevSlots) {
        const uint32_t need = a.tag - (uint32_t)kDevSlots;
        const unsigned long long t0 = gtime();
        while ((int32_t)(ld_acquire_sys(a.done[threadIdx.x]) - need) < 0) {
            __nanosleep(128);
            if (gtime() - t0 > a.timeout_ns) {
                *(volatile uint32_t *)a.err = 2u;
                if (blockIdx.x == 0)
                    printf("hg peer push: rank %d tag %u: rank %d consumed %u, need %u\n", a.p, a.tag, threadIdx.x,
                           ld_acquire_sys(a.done[threadIdx.x]), need);
                break;
            }
        }
    }
    __syncthreads();
    const int64_t total = (int64_t)a.B * a.n_local;
    const int64_t off = (int64_t)a.slot * a.box_floats + a.dst0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / a.n_local, j = i - b * a.n_local;
        const float v = a.src[i];
        for (int r = 0; r < a.P; ++r) a.box[r][off + b * a.dst_ld + j] = v;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t old = atomicAdd(a.count, 1u);
        if (old == gridDim.x - 1) {  // every CTA's stores are visible system-wide: raise the flags
            *a.count = 0;
            __threadfence_system();
            for (int r = 0; r < a.P; ++r) st_release_sys(a.flag[r] + a.slot * a.P + a.p, a.tag);
        }
    }
}

struct WaitArgs {
    const float *box;        // this rank's box, slot 0
    const uint32_t *flag;    // this rank's flags
    uint32_t *done;          // this rank's consumed word
    float *y;
    const float *bias;       // all-reduce: added once after the sum (NULL = none)
    int64_t ldy, N_full, box_floats;
    int B, P, slot;
    int reduce;              // 0: copy [B][N_full]; 1: y = sum over ranks of [P][B][N_full], rank order
    uint32_t tag;
    uint32_t *count;
    uint32_t *err;
    unsigned long long timeout_ns;
};

// Wait until every rank's part of this exchange is in this rank's box, copy them into y (all-gather)
// or sum them into y in rank order and add the bias (all-reduce: every rank adds the same values in
// the same order, so every rank holds the same bits), and mark the box slot consumed.
__global__ void peer_wait_kernel(const __grid_constant__ WaitArgs a) {
    if (threadIdx.x < a.P) {
        const unsigned long long t0 = gtime();
        while ((int32_t)(ld_acquire_sys(a.flag + a.slot * a.P + threadIdx.x) - a.tag) < 0) {
            __nanosleep(64);
            if (gtime() - t0 > a.timeout_ns) {
                *(volatile uint32_t *)a.err = 2u;
                if (blockIdx.x == 0)
                    printf("hg peer wait: slot %d tag %u: flag of rank %d is %u\n", a.slot, a.tag, threadIdx.x,
                           ld_acquire_sys(a.flag + a.slot * a.P + threadIdx.x));
                break;
            }
        }
    }
    __syncthreads();
    const float *src = a.box + (int64_t)a.slot * a.box_floats;
    const int64_t total = (int64_t)a.B * a.N_full;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / a.N_full, j = i - b * a.N_full;
        float v = __ldcv(src + i);
        if (a.reduce) {
            for (int q = 1; q < a.P; ++q) v = __fadd_rn(v, __ldcv(src + (int64_t)q * total + i));
            if (a.bias) v = __fadd_rn(v, a.bias[j]);
        }
        a.y[b * a.ldy + j] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t old = atomicAdd(a.count, 1u);
        if (old == gridDim.x - 1) {
            *a.count = 0;
            __threadfence_system();
            st_release_sys(a.done, a.tag);
        }
    }
}

// Same-process peers: rank contexts of one group find each other's host segment here.
struct SegEntry {
    std::string name;
    void *base;
    size_t bytes;
    int refs;
};
std::mutex g_seg_mu;
std::vector<SegEntry> g_segs;

}  // namespace

struct PeerGroup {
    int P = 1, p = 0, device = 0;
    // device side
    void *alloc = nullptr;           // this rank's: [kDevSlots][box_floats] floats, flags, done, counters
    int64_t box_floats = 0;
    float *box[kMaxPeers] = {};
    uint32_t *flag[kMaxPeers] = {};
    uint32_t *done[kMaxPeers] = {};
    void *ipc_open[kMaxPeers] = {};  // opened IPC mappings (other processes' allocations)
    uint32_t *count = nullptr;       // [2]: push, wait CTA counters
    uint64_t seq = 0;
    // host side
    std::string shm;
    uint8_t *seg = nullptr;
    size_t seg_bytes = 0;
    bool seg_registered = false, seg_owner = false;
    int64_t host_floats = 0;
    float *hy = nullptr, *hy_dev = nullptr;  // [kHostSlots][host_floats]
    uint32_t *ready = nullptr;               // [kHostSlots][P]
    uint32_t *hdone = nullptr;               // [P] (64-byte stride)
};

namespace {
size_t dev_bytes(int64_t box_floats) {
    return (size_t)kDevSlots * box_floats * 4 + (size_t)(kDevSlots * kMaxPeers + 64) * 4;
}
void dev_layout(PeerGroup *g, int r, uint8_t *base) {
    g->box[r] = (float *)base;
    g->flag[r] = (uint32_t *)(base + (size_t)kDevSlots * g->box_floats * 4);
    g->done[r] = g->flag[r] + kDevSlots * kMaxPeers;
}
size_t host_header() { return 4096 + 64 * kMaxPeers; }
void host_layout(PeerGroup *g) {
    g->ready = (uint32_t *)g->seg;
    g->hdone = (uint32_t *)(g->seg + 4096);
    g->hy = (float *)(g->seg + host_header());
}
}  // namespace

hg_status peer_export(PeerGroup **pg, int device, int nranks, int rank, int64_t box_floats, int64_t host_floats,
                      void *blob_out) {
    if (nranks < 1 || nranks > kMaxPeers || rank < 0 || rank >= nranks)
        return set_error(HG_EINVAL, "peer group: %d ranks (max %d), rank %d", nranks, kMaxPeers, rank);
    PeerGroup *g = *pg;
    if (!g) {
        g = new PeerGroup;
        g->P = nranks;
        g->p = rank;
        g->device = device;
        g->box_floats = box_floats;
        g->host_floats = host_floats;
        if (cudaMalloc(&g->alloc, dev_bytes(box_floats)) != cudaSuccess ||
            cudaMemset(g->alloc, 0, dev_bytes(box_floats)) != cudaSuccess ||
            cudaDeviceSynchronize() != cudaSuccess) {
            cudaGetLastError();
            if (g->alloc) cudaFree(g->alloc);
            delete g;
            return set_error(HG_ENOMEM, "peer group: device box of %zu bytes", dev_bytes(box_floats));
        }
        dev_layout(g, rank, (uint8_t *)g->alloc);
        g->count = g->done[rank] + 16;
        if (rank == 0) {  // the shared host segment
            static std::atomic<int> counter{0};
            char name[64];
            snprintf(name, sizeof name, "/hg_peer_%d_%d", (int)getpid(), counter++);
            g->shm = name;
            g->seg_bytes = host_header() + (size_t)kHostSlots * host_floats * 4;
            const int fd = shm_open(name, O_CREAT | O_EXCL | O_RDWR, 0600);
            if (fd < 0 || ftruncate(fd, (off_t)g->seg_bytes) != 0) {
                if (fd >= 0) close(fd);
                cudaFree(g->alloc);
                delete g;
                return set_error(HG_ENOMEM, "peer group: shm_open/ftruncate of %s failed", name);
            }
            close(fd);
            g->seg_owner = true;
        }
        *pg = g;
    }
    Blob b;
    std::memset(&b, 0, sizeof b);
    b.magic = kMagic;
    b.nranks = nranks;
    b.rank = rank;
    b.device = device;
    b.pid = (int64_t)getpid();
    b.box_floats = g->box_floats;
    b.host_floats = g->host_floats;
    b.dev_base = (uint64_t)(uintptr_t)g->alloc;
    if (cudaIpcGetMemHandle(&b.ipc, g->alloc) != cudaSuccess) cudaGetLastError();  // same-process use only
    if (rank == 0) snprintf(b.shm, sizeof b.shm, "%s", g->shm.c_str());
    std::memset(blob_out, 0, 512);
    std::memcpy(blob_out, &b, sizeof b);
    return HG_OK;
}

hg_status peer_open(PeerGroup *g, const void *blobs) {
    const Blob *bs = (const Blob *)blobs;
    for (int r = 0; r < g->P; ++r) {
        const Blob &b = *(const Blob *)((const uint8_t *)bs + (size_t)512 * r);
        if (b.magic != kMagic || b.nranks != g->P || b.rank != r || b.box_floats != g->box_floats ||
            b.host_floats != g->host_floats)
            return set_error(HG_EINVAL, "peer group: blob %d does not match (ranks, sizes)", r);
        if (r == g->p) continue;
        uint8_t *base = nullptr;
        if (b.pid == (int64_t)getpid()) {
            base = (uint8_t *)(uintptr_t)b.dev_base;
            if (b.device != g->device) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                    return set_error(HG_ECUDA, "peer access %d -> %d: %s", g->device, b.device, cudaGetErrorString(e));
                cudaGetLastError();
            }
        } else {
            void *p = nullptr;
            const cudaError_t e = cudaIpcOpenMemHandle(&p, b.ipc, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) return set_error(HG_ECUDA, "cudaIpcOpenMemHandle(rank %d): %s", r, cudaGetErrorString(e));
            g->ipc_open[r] = p;
            base = (uint8_t *)p;
        }
        dev_layout(g, r, base);
    }
    // host segment: rank 0 named it; same-process ranks share one mapping
    const Blob &b0 = *(const Blob *)bs;
    g->shm = b0.shm;
    g->seg_bytes = host_header() + (size_t)kHostSlots * g->host_floats * 4;
    {
        std::lock_guard<std::mutex> lk(g_seg_mu);
        for (auto &e : g_segs)
            if (e.name == g->shm) {
                g->seg = (uint8_t *)e.base;
                ++e.refs;
            }
        if (!g->seg) {
            const int fd = shm_open(g->shm.c_str(), O_RDWR, 0600);
            if (fd < 0) return set_error(HG_EINVAL, "peer group: shm_open(%s) failed", g->shm.c_str());
            void *m = mmap(nullptr, g->seg_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
            close(fd);
            if (m == MAP_FAILED) return set_error(HG_ENOMEM, "peer group: mmap of %s failed", g->shm.c_str());
            if (cudaHostRegister(m, g->seg_bytes, cudaHostRegisterMapped | cudaHostRegisterPortable) != cudaSuccess) {
                cudaGetLastError();
                munmap(m, g->seg_bytes);
                return set_error(HG_ECUDA, "peer group: cudaHostRegister of the host segment failed");
            }
            g->seg = (uint8_t *)m;
            g_segs.push_back({g->shm, m, g->seg_bytes, 1});
        }
    }
    host_layout(g);
    if (cudaHostGetDevicePointer((void **)&g->hy_dev, g->hy, 0) != cudaSuccess) {
        cudaGetLastError();
        return set_error(HG_ECUDA, "peer group: host segment has no device mapping");
    }
    return HG_OK;
}

void peer_destroy(PeerGroup *g) {
    if (!g) return;
    for (int r = 0; r < kMaxPeers; ++r)
        if (g->ipc_open[r]) cudaIpcCloseMemHandle(g->ipc_open[r]);
    if (g->seg) {
        std::lock_guard<std::mutex> lk(g_seg_mu);
        for (size_t i = 0; i < g_segs.size(); ++i)
            if (g_segs[i].base == g->seg && --g_segs[i].refs == 0) {
                cudaHostUnregister(g_segs[i].base);
                munmap(g_segs[i].base, g_segs[i].bytes);
                g_segs.erase(g_segs.begin() + (long)i);
                break;
            }
    }
    if (g->seg_owner) shm_unlink(g->shm.c_str());
    if (g->alloc) cudaFree(g->alloc);
    cudaGetLastError();
    delete g;
}

int peer_nranks(const PeerGroup *g) { return g ? g->P : 1; }

// Debug: this rank's flag words [kDevSlots][P], its done word, its seq, and the addresses it uses for
// every rank's flags (as 32-bit halves) -> out[0 .. kDevSlots*kMaxPeers + 2 + 2*kMaxPeers).
void peer_debug_words(PeerGroup *g, uint32_t *out) {
    cudaMemcpy(out, g->flag[g->p], kDevSlots * kMaxPeers * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(out + kDevSlots * kMaxPeers, g->done[g->p], 4, cudaMemcpyDeviceToHost);
    out[kDevSlots * kMaxPeers + 1] = (uint32_t)g->seq;
    for (int r = 0; r < kMaxPeers; ++r) {
        const uint64_t a = (uint64_t)(uintptr_t)g->flag[r];
        out[kDevSlots * kMaxPeers + 2 + 2 * r] = (uint32_t)a;
        out[kDevSlots * kMaxPeers + 3 + 2 * r] = (uint32_t)(a >> 32);
    }
}
int peer_rank(const PeerGroup *g) { return g ? g->p : 0; }

namespace {
// One device exchange: push this rank's [B][n_local] into every box at (dst0, dst_ld), then wait for
// all P parts and copy (reduce = 0) or sum (reduce = 1) the box's [B][N_out] view into y.
int exchange(PeerGroup *g, const float *src, int B, int64_t n_local, int64_t dst0, int64_t dst_ld, int64_t N_out,
             int reduce, const float *bias, float *y, int64_t ldy, uint32_t *err, double timeout_s, void *stream) {
    const uint64_t q = g->seq++;
    static const bool dbg = getenv("HG_PEER_DEBUG") != nullptr;
    if (dbg) fprintf(stderr, "hg peer: rank %d exchange %llu (%s) n_local %lld B %d stream %p\n", g->p,
                     (unsigned long long)q, reduce ? "reduce" : "gather", (long long)n_local, B, stream);
    const int slot = (int)(q % kDevSlots);
    const uint32_t tag = (uint32_t)(q + 1);
    const unsigned long long tns = (unsigned long long)(timeout_s * 1e9 * dev_timeout_scale());
    PushArgs pa{};
    pa.src = src;
    pa.n_local = n_local;
    pa.dst0 = dst0;
    pa.dst_ld = dst_ld;
    pa.B = B;
    pa.P = g->P;
    pa.p = g->p;
    pa.slot = slot;
    pa.tag = tag;
    pa.box_floats = g->box_floats;
    for (int r = 0; r < g->P; ++r) {
        pa.box[r] = g->box[r];
        pa.flag[r] = g->flag[r];
        pa.done[r] = g->done[r];
    }
    pa.count = g->count;
    pa.err = err;
    pa.timeout_ns = tns;
    const int64_t total = (int64_t)B * n_local;
    int grid = (int)std::min<int64_t>(64, (total + 255) / 256);
    if (grid < 1) grid = 1;
    peer_push_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(pa);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return (int)e;
    WaitArgs wa{};
    wa.box = g->box[g->p];
    wa.flag = g->flag[g->p];
    wa.done = g->done[g->p];
    wa.y = y;
    wa.bias = bias;
    wa.ldy = ldy;
    wa.N_full = N_out;
    wa.box_floats = g->box_floats;
    wa.B = B;
    wa.P = g->P;
    wa.slot = slot;
    wa.reduce = reduce;
    wa.tag = tag;
    wa.count = g->count + 1;
    wa.err = err;
    wa.timeout_ns = tns;
    int wgrid = (int)std::min<int64_t>(32, ((int64_t)B * N_out + 255) / 256);
    if (wgrid < 1) wgrid = 1;
    peer_wait_kernel<<<wgrid, 256, 0, (cudaStream_t)stream>>>(wa);
    return (int)cudaGetLastError();
}
}  // namespace

// All-gather of one linear's row shards: ylocal [B][n_local] (this rank's rows) -> y [B][ldy] full, in
// global column order, on `stream`.
int peer_exchange(PeerGroup *g, const float *ylocal, int B, int64_t n_local, float *y, int64_t ldy, uint32_t *err,
                  double timeout_s, void *stream) {
    const int64_t N_full = n_local * g->P;
    if ((int64_t)B * N_full > g->box_floats) return (int)cudaErrorInvalidValue;
    return exchange(g, ylocal, B, n_local, (int64_t)g->p * n_local, N_full, N_full, 0, nullptr, y, ldy, err,
                    timeout_s, stream);
}

// All-reduce of a row-parallel linear's partial sums (Megatron pairing, reading R32): partial [B][N]
// -> y [B][ldy] = sum over ranks in rank order (+ bias once), identical bits on every rank.
int peer_reduce(PeerGroup *g, const float *partial, int B, int64_t N, const float *bias, float *y, int64_t ldy,
                uint32_t *err, double timeout_s, void *stream) {
    if ((int64_t)g->P * B * N > g->box_floats) return (int)cudaErrorInvalidValue;
    return exchange(g, partial, B, N, (int64_t)g->p * B * N, N, N, 1, bias, y, ldy, err, timeout_s, stream);
}

// ---- host side: the shared [kHostSlots][B][N_full] segment
float *peer_host_y(PeerGroup *g, int64_t k) { return g->hy + (k % kHostSlots) * g->host_floats; }
float *peer_host_y_dev(PeerGroup *g, int64_t k) { return g->hy_dev + (k % kHostSlots) * g->host_floats; }
int peer_host_slots() { return kHostSlots; }

namespace {
hg_status spin_until(const uint32_t *w, uint32_t need, double timeout_s, const char *what, int r, int64_t k) {
    const auto t0 = std::chrono::steady_clock::now();
    for (int spin = 0; (int32_t)(__atomic_load_n(w, __ATOMIC_ACQUIRE) - need) < 0; ++spin) {
        if (spin < 2048) continue;
        std::this_thread::yield();
        if ((spin & 1023) == 0 &&
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s)
            return set_error(HG_ETIMEOUT, "peer group: %s of rank %d for host linear %lld not reached within %.1f s "
                             "(word %u, need %u)", what, r, (long long)k, timeout_s, __atomic_load_n(w, __ATOMIC_ACQUIRE),
                             need);
    }
    return HG_OK;
}
}  // namespace

// This rank's rows of linear k are in the host segment (CPU rows written, GPU rows' D2H landed).
void peer_host_publish(PeerGroup *g, int64_t k) {
    __atomic_store_n(g->ready + (k % kHostSlots) * g->P + g->p, (uint32_t)(k + 1), __ATOMIC_RELEASE);
}
// Every rank's rows of linear k are in the host segment.
hg_status peer_host_wait_ready(PeerGroup *g, int64_t k, double timeout_s) {
    for (int r = 0; r < g->P; ++r)
        PEER_TRY(spin_until(g->ready + (k % kHostSlots) * g->P + r, (uint32_t)(k + 1), timeout_s, "host rows ready", r, k));
    return HG_OK;
}
// This rank has read linear k's full y (its host slot may be refilled once every rank has).
void peer_host_consumed(PeerGroup *g, int64_t k) {
    __atomic_store_n(g->hdone + 16 * g->p, (uint32_t)(k + 1), __ATOMIC_RELEASE);
}
// Host slot of linear k is free: every rank consumed linear k - kHostSlots.
hg_status peer_host_wait_free(PeerGroup *g, int64_t k, double timeout_s) {
    if (k < kHostSlots) return HG_OK;
    for (int r = 0; r < g->P; ++r)
        PEER_TRY(spin_until(g->hdone + 16 * r, (uint32_t)(k - kHostSlots + 1), timeout_s, "host slot free", r, k));
    return HG_OK;
}
// A new call sequence (linear indices restart at 0): the host words restart too.  Every rank must
// have finished the previous call (the caller's barrier) before any rank resets.
void peer_host_reset(PeerGroup *g) {
    for (int s = 0; s < kHostSlots; ++s) __atomic_store_n(g->ready + s * g->P + g->p, 0u, __ATOMIC_RELEASE);
    __atomic_store_n(g->hdone + 16 * g->p, 0u, __ATOMIC_RELEASE);
}

}  // namespace hg
