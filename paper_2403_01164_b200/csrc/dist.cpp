// dist.cpp -- column-sharded tensor parallelism across the GPUs of one box
// (BJ:5 -- not in the paper, which uses one A10).
//
// Rank p owns W rows [pN/P, (p+1)N/P) of every linear and runs the full
// heterogeneous split on them with its own host link and its share of host
// cores; the P output shards are then all-gathered over NVLink/NVSwitch with
// NCCL.  NCCL is dlopen'ed (the torch-bundled libnccl.so.2 when torch is
// loaded, else HG_NCCL_LIB), so the library links and loads without it.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>

#include "hg_internal.h"

namespace hg {

namespace {
typedef int nccl_result;       // ncclResult_t
typedef void *nccl_comm;       // ncclComm_t
struct nccl_id { char internal[128]; };
constexpr int kNcclFloat32 = 7;  // ncclFloat32 in nccl.h

struct Nccl {
    void *h = nullptr;
    nccl_result (*GetUniqueId)(nccl_id *) = nullptr;
    nccl_result (*CommInitRank)(nccl_comm *, int, nccl_id, int) = nullptr;
    nccl_result (*AllGather)(const void *, void *, size_t, int, nccl_comm, cudaStream_t) = nullptr;
    nccl_result (*CommDestroy)(nccl_comm) = nullptr;
    nccl_result (*CommAbort)(nccl_comm) = nullptr;
    const char *(*GetErrorString)(nccl_result) = nullptr;
};

Nccl *nccl() {
    static Nccl n;
    static bool tried = false;
    if (tried) return n.h ? &n : nullptr;
    tried = true;
    const char *env = getenv("HG_NCCL_LIB");
    const char *cands[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char *c : cands) {
        if (!c) continue;
        n.h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
        if (n.h) break;
    }
    if (!n.h) return nullptr;
    n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(n.h, "ncclGetUniqueId");
    n.CommInitRank = (decltype(n.CommInitRank))dlsym(n.h, "ncclCommInitRank");
    n.AllGather = (decltype(n.AllGather))dlsym(n.h, "ncclAllGather");
    n.CommDestroy = (decltype(n.CommDestroy))dlsym(n.h, "ncclCommDestroy");
    n.CommAbort = (decltype(n.CommAbort))dlsym(n.h, "ncclCommAbort");
    n.GetErrorString = (decltype(n.GetErrorString))dlsym(n.h, "ncclGetErrorString");
    if (!n.GetUniqueId || !n.CommInitRank || !n.AllGather || !n.CommDestroy) {
        n.h = nullptr;
        return nullptr;
    }
    return &n;
}
}  // namespace

struct Dist {
    nccl_comm comm = nullptr;
    int nranks = 1, rank = 0;
};

hg_status dist_unique_id(void *id128) {
    Nccl *n = nccl();
    if (!n) return set_error(HG_ENCCL, "NCCL library not found (set HG_NCCL_LIB)");
    nccl_id id;
    nccl_result r = n->GetUniqueId(&id);
    if (r != 0) return set_error(HG_ENCCL, "ncclGetUniqueId: %d", r);
    std::memcpy(id128, &id, sizeof id);
    return HG_OK;
}

Dist *dist_create(int nranks, int rank, const void *id128, hg_status *st) {
    Nccl *n = nccl();
    if (!n) {
        *st = set_error(HG_ENCCL, "NCCL library not found (set HG_NCCL_LIB)");
        return nullptr;
    }
    nccl_id id;
    std::memcpy(&id, id128, sizeof id);
    Dist *d = new Dist;
    d->nranks = nranks;
    d->rank = rank;
    nccl_result r = n->CommInitRank(&d->comm, nranks, id, rank);
    if (r != 0) {
        *st = set_error(HG_ENCCL, "ncclCommInitRank(%d,%d): %s", nranks, rank,
                        n->GetErrorString ? n->GetErrorString(r) : "?");
        delete d;
        return nullptr;
    }
    *st = HG_OK;
    return d;
}

void dist_destroy(Dist *d) {
    if (!d) return;
    Nccl *n = nccl();
    if (n && d->comm) n->CommDestroy(d->comm);
    delete d;
}

int dist_nranks(const Dist *d) { return d ? d->nranks : 1; }
int dist_rank(const Dist *d) { return d ? d->rank : 0; }

hg_status dist_allgather(Dist *d, const float *send, float *recv, size_t count_per_rank,
                         void *stream) {
    Nccl *n = nccl();
    if (!n || !d) return set_error(HG_ESTATE, "all-gather without hg_dist_init");
    nccl_result r = n->AllGather(send, recv, count_per_rank, kNcclFloat32, d->comm,
                                 (cudaStream_t)stream);
    if (r != 0)
        return set_error(HG_ENCCL, "ncclAllGather: %s", n->GetErrorString ? n->GetErrorString(r) : "?");
    return HG_OK;
}

}  // namespace hg
