// Dev probe (not part of the product): does a kernel that allocates tensor memory (tcgen05.alloc)
// still run two CTAs per SM?  The occupancy API answers 1 for every such kernel; the SM itself
// co-schedules them (CTA pairs overlap on all SMs), which is why fcw_launch.cu sizes the
// persistent grid of the TMEM-twiddle kernels from the register / SMEM / column budgets.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
template <int USE_TMEM, int COLS>
__global__ void __launch_bounds__(256, 2) k(unsigned long long* rec, int smem_pad) {
    extern __shared__ float4 dyn[];
    __shared__ uint32_t slot;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (USE_TMEM) {
        if ((threadIdx.x >> 5) == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&slot)), "n"(COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    float a = threadIdx.x;
    for (int i = 0; i < 400000; ++i) a = a * 1.0001f + 0.5f;
    if (a == 12345.f) dyn[0].x = a;
    unsigned long long t2;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (threadIdx.x == 0) { rec[blockIdx.x * 4] = smid; rec[blockIdx.x * 4 + 1] = t0; rec[blockIdx.x * 4 + 2] = t1; rec[blockIdx.x * 4 + 3] = t2; }
    if (USE_TMEM) {
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        if ((threadIdx.x >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "n"(COLS));
    }
}
template <class K> void run(const char* name, K kern, int smem) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int grid = 2 * sms;
    unsigned long long* d; cudaMalloc(&d, grid * 32);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
    kern<<<grid, 256, smem>>>(d, 0);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(grid * 4);
    cudaMemcpy(h.data(), d, grid * 32, cudaMemcpyDeviceToHost);
    // count SMs where two CTAs overlapped in their compute interval
    int overlap = 0; unsigned long long tmin = ~0ull, tmax = 0;
    for (int a = 0; a < grid; ++a) { tmin = std::min(tmin, h[a*4+1]); tmax = std::max(tmax, h[a*4+3]);
        for (int b = a + 1; b < grid; ++b) if (h[a*4] == h[b*4]) {
            unsigned long long s = std::max(h[a*4+2], h[b*4+2]), e = std::min(h[a*4+3], h[b*4+3]);
            if (e > s && (e - s) * 2 > (h[a*4+3] - h[a*4+2])) ++overlap; } }
    printf("%-34s occ API %d, CTA pairs overlapping on one SM: %d of %d SMs, total %.3f ms, err %s\n", name, occ, overlap, sms, (tmax - tmin) * 1e-6, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    run("no TMEM, 110 KB smem", k<0, 128>, 110 * 1024);
    run("TMEM 128 cols, 110 KB smem", k<1, 128>, 110 * 1024);
    run("TMEM 128 cols, 32 KB smem", k<1, 128>, 32 * 1024);
    run("TMEM 256 cols, 110 KB smem", k<1, 256>, 110 * 1024);
    run("TMEM 32 cols, 110 KB smem", k<1, 32>, 110 * 1024);
    return 0;
}
