// Per-launch cost of kernels shaped like the persistent GEMV (148 CTAs x 288 threads):
// empty / 129 KB dynamic smem / + mbarrier + one 14 KB TMA bulk copy per CTA.  Mean over 2000
// back-to-back launches (CUDA events), and alternating with a small-smem kernel (carveout switch).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void k_empty(int *p) { if (threadIdx.x == 999999) p[0] = 1; }
__global__ void k_smem(int *p) {
    extern __shared__ uint8_t sm[];
    if (threadIdx.x == 0) sm[0] = 1;
    __syncthreads();
    if (sm[1] == 77 && threadIdx.x == 999999) p[0] = 1;
}
__global__ void k_tma(const uint8_t *src, int bytes, int *p) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t *bar = (uint64_t *)sm;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm + 128);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "l"(src + (size_t)blockIdx.x * bytes), "r"(bytes), "r"(b) : "memory");
    }
    uint32_t ok = 0;
    do {
        asm volatile("{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\n selp.u32 %0,1,0,q;\n}"
                     : "=r"(ok) : "r"(b) : "memory");
    } while (!ok);
    if (sm[128 + threadIdx.x] == 77 && threadIdx.x == 999999) p[0] = 1;
}

template <typename F>
float time_it(F f, int n, cudaStream_t s) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 20; ++i) f();
    cudaEventRecord(a, s);
    for (int i = 0; i < n; ++i) f();
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e3f / n;
}

int main() {
    int *p;
    cudaMalloc(&p, 4);
    uint8_t *src;
    cudaMalloc(&src, 148 * 16384 * 4);
    cudaStream_t s;
    cudaStreamCreate(&s);
    const int big = 129 * 1024;
    cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    const int n = 2000;
    printf("empty 0 KB smem        : %6.2f us/launch\n", time_it([&] { k_empty<<<148, 288, 0, s>>>(p); }, n, s));
    printf("empty 129 KB smem      : %6.2f us/launch\n", time_it([&] { k_smem<<<148, 288, big, s>>>(p); }, n, s));
    printf("tma 14 KB, 129 KB smem : %6.2f us/launch\n",
           time_it([&] { k_tma<<<148, 288, big, s>>>(src, 14336, p); }, n, s));
    printf("tma 14 KB, 16 KB smem  : %6.2f us/launch\n",
           time_it([&] { k_tma<<<148, 288, 16 * 1024, s>>>(src, 14336, p); }, n, s));
    printf("alternate empty0/129KB : %6.2f us/pair\n", time_it([&] {
               k_empty<<<148, 288, 0, s>>>(p);
               k_smem<<<148, 288, big, s>>>(p);
           }, n, s));
    printf("alternate tiny(1 CTA)/129KB : %6.2f us/pair\n", time_it([&] {
               k_empty<<<1, 256, 0, s>>>(p);
               k_smem<<<148, 288, big, s>>>(p);
           }, n, s));
    cudaFuncSetAttribute(k_smem, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_empty, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    printf("alternate (carveout 100 both): %6.2f us/pair\n", time_it([&] {
               k_empty<<<1, 256, 0, s>>>(p);
               k_smem<<<148, 288, big, s>>>(p);
           }, n, s));
    return 0;
}
