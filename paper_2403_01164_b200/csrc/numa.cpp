// numa.cpp -- host placement for one rank per GPU ("threads and pinned weights NUMA-local
// to each GPU").
//
// A rank's CPU lane reads its offloaded rows from host DRAM and its copy engine DMAs the streamed rows
// over the GPU's own PCIe root port; both are cheapest from the memory node the GPU hangs off.  The node
// is the PCI device's `numa_node` in sysfs; its cores are the node's `cpulist`.  Weights are placed by
// binding the pages to the node BEFORE they are first touched (page-locking them afterwards keeps them
// there: locked pages are not migrated), so no libnuma is needed: mmap + mbind(2) + cudaHostRegister.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cctype>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "hg_internal.h"

namespace hg {

namespace {
constexpr int kMpolBind = 2;  // MPOL_BIND (linux/mempolicy.h)

std::string read_file(const std::string &path) {
    FILE *f = fopen(path.c_str(), "r");
    if (!f) return std::string();
    char buf[4096];
    const size_t n = fread(buf, 1, sizeof buf - 1, f);
    fclose(f);
    buf[n] = 0;
    return std::string(buf);
}
}  // namespace

// "0-3,8,10-11" -> {0,1,2,3,8,10,11}; empty on a malformed list
std::vector<int> parse_cpulist(const char *s) {
    std::vector<int> out;
    const char *p = s;
    while (*p) {
        while (*p == ',' || isspace((unsigned char)*p)) ++p;
        if (!*p) break;
        if (!isdigit((unsigned char)*p)) return {};
        const long a = strtol(p, (char **)&p, 10);
        long b = a;
        if (*p == '-') {
            ++p;
            if (!isdigit((unsigned char)*p)) return {};
            b = strtol(p, (char **)&p, 10);
        }
        if (b < a || b - a > 65536) return {};
        for (long c = a; c <= b; ++c) out.push_back((int)c);
    }
    return out;
}

int numa_node_of_device(int device) {
    char bus[64] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    for (char *q = bus; *q; ++q) *q = (char)tolower((unsigned char)*q);
    const std::string v = read_file(std::string("/sys/bus/pci/devices/") + bus + "/numa_node");
    if (v.empty()) return -1;
    const int node = atoi(v.c_str());
    return node >= 0 ? node : -1;
}

std::vector<int> numa_cpus(int node) {
    if (node < 0) return {};
    const std::string v = read_file("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist");
    return parse_cpulist(v.c_str());
}

// Anonymous memory whose pages are bound to `node` (node < 0: no binding), optionally page-locked and
// mapped for the device.  Returns nullptr on failure.
void *host_alloc_node(size_t bytes, int node, bool lock) {
    if (bytes == 0) return nullptr;
    void *p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return nullptr;
    if (node >= 0 && node < 1024) {
        unsigned long mask[1024 / (8 * sizeof(unsigned long))] = {0};
        mask[node / (8 * sizeof(unsigned long))] |= 1ul << (node % (8 * sizeof(unsigned long)));
        // best effort: a kernel without NUMA support leaves the default policy
        syscall(SYS_mbind, p, bytes, kMpolBind, mask, (unsigned long)1024, 0u);
    }
    if (lock) {
        if (cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable) != cudaSuccess) {
            cudaGetLastError();
            munmap(p, bytes);
            return nullptr;
        }
    } else {
        std::memset(p, 0, bytes);  // first touch under the binding
    }
    return p;
}

void host_free_node(void *p, size_t bytes, bool locked) {
    if (!p) return;
    if (locked) {
        cudaHostUnregister(p);
        cudaGetLastError();
    }
    munmap(p, bytes);
}

// The node a page of p currently lives on (-1 unknown): move_pages(2) in query mode.
int numa_node_of_page(const void *p) {
    void *pages[1] = {const_cast<void *>(p)};
    int status[1] = {-1};
    if (syscall(SYS_move_pages, 0, 1ul, pages, nullptr, status, 0) != 0) return -1;
    return status[0] >= 0 ? status[0] : -1;
}

}  // namespace hg
