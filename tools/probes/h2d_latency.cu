// Small-transfer latency while another stream streams 32 MiB H2D chunks (the link lane):
//   y (86 KB fp32, host->device): cudaMemcpyAsync (normal / high-priority stream) or a kernel
//   reading the mapped pinned buffer; x (14 KB, device->host): cudaMemcpyAsync or a kernel writing
//   mapped pinned memory + a flag the host polls.  The big queue is kept `depth` chunks deep by
//   a feeder that tops it up.  Development probe, not part of the library.
#include <cuda_runtime.h>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>

__global__ void zc_read(const float *__restrict__ h, float *__restrict__ d, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) d[i] = h[i];
}
__global__ void zc_write(const uint4 *__restrict__ d, uint4 *h, int n, volatile unsigned *flag, unsigned v) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) h[i] = d[i];
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) *flag = v;
}

int main() {
    const size_t big = 2ull << 30;
    const int n = 21504;
    void *hb, *db;
    float *hs, *ds;
    cudaHostAlloc(&hb, big, cudaHostAllocDefault);
    cudaMalloc(&db, big);
    cudaHostAlloc((void **)&hs, n * 4, cudaHostAllocMapped);
    cudaMalloc((void **)&ds, n * 4);
    unsigned *flag;
    cudaHostAlloc((void **)&flag, 64, cudaHostAllocMapped);
    *flag = 0;
    int lo, hi;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStream_t sb, ss, sh;
    cudaStreamCreateWithPriority(&sb, cudaStreamNonBlocking, lo);
    cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking);
    cudaStreamCreateWithPriority(&sh, cudaStreamNonBlocking, hi);
    cudaEvent_t evs[512];
    for (auto &e : evs) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    unsigned tagv = 0;
    for (size_t chunk : {32ull << 20, 8ull << 20})
        for (int depth : {64, 2}) {
            const char *names[] = {"y memcpy", "y memcpy hi-prio", "y zero-copy read", "x memcpy d2h",
                                   "x zero-copy write"};
            for (int mode = 0; mode < 5; ++mode) {
                std::vector<double> lat;
                int issued = 0, done = 0;
                auto feed = [&]() {  // keep `depth` chunks queued on sb
                    while (done < issued && cudaEventQuery(evs[done % 512]) == cudaSuccess) ++done;
                    while (issued - done < depth) {
                        const size_t off = (issued * chunk) % (big - chunk);
                        cudaMemcpyAsync((char *)db + off, (char *)hb + off, chunk, cudaMemcpyHostToDevice, sb);
                        cudaEventRecord(evs[issued % 512], sb);
                        ++issued;
                    }
                };
                feed();
                std::this_thread::sleep_for(std::chrono::milliseconds(2));
                for (int it = 0; it < 200; ++it) {
                    feed();
                    auto t0 = std::chrono::steady_clock::now();
                    if (mode == 0) cudaMemcpyAsync(ds, hs, n * 4, cudaMemcpyHostToDevice, ss);
                    if (mode == 1) cudaMemcpyAsync(ds, hs, n * 4, cudaMemcpyHostToDevice, sh);
                    if (mode == 2) zc_read<<<42, 512, 0, ss>>>(hs, ds, n);
                    if (mode == 3) cudaMemcpyAsync(hs, ds, 14336, cudaMemcpyDeviceToHost, ss);
                    if (mode == 4) {
                        ++tagv;
                        zc_write<<<1, 512, 0, ss>>>((const uint4 *)ds, (uint4 *)hs, 14336 / 16, flag, tagv);
                        while (*(volatile unsigned *)flag != tagv) {}
                    }
                    if (mode != 4) cudaStreamSynchronize(mode == 1 ? sh : ss);
                    lat.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
                    feed();
                }
                cudaDeviceSynchronize();
                std::sort(lat.begin(), lat.end());
                printf("chunk %2zu MiB depth %2d  %-18s median %8.1f us  p90 %8.1f us  max %8.1f us\n", chunk >> 20,
                       depth, names[mode], lat[lat.size() / 2], lat[lat.size() * 9 / 10], lat.back());
                fflush(stdout);
            }
        }
    return 0;
}
