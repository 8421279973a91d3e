// Dev microbenchmark (not part of the product): the half-warp FFT_256
// (fcw_fft.cuh fft256_half) with its pass-2 twiddles read from
//   (a) the per-lane SMEM table tw16 (the product path: 15 LDS.64 per lane),
//   (b) TMEM, one tcgen05.ld.32x32b.x32 per transform,
//   (c) TMEM, two tcgen05.ld.32x32b.x16 per transform.
// The twiddles are lane constants (W_256^(m t), t = lane & 15), so every
// thread parks its 15 values in its own TMEM lane once per kernel.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2008_00672_b200/csrc
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "fcw_fft.cuh"

using namespace fcw;

#define R16(a, o) a(o + 0), a(o + 1), a(o + 2), a(o + 3), a(o + 4), a(o + 5), a(o + 6), a(o + 7), a(o + 8), a(o + 9), \
                  a(o + 10), a(o + 11), a(o + 12), a(o + 13), a(o + 14), a(o + 15)

__device__ __forceinline__ void tmem_alloc(uint32_t* slot, int warp) {
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
            (unsigned)__cvta_generic_to_shared(slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
}
__device__ __forceinline__ void tmem_free(uint32_t base, int warp) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(base));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&d)[16]) {
#define IN(i) "r"(d[i])
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%16], {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15};" ::R16(IN, 0),
        "r"(taddr)
        : "memory");
#undef IN
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&d)[16]) {
#define OUT(i) "=r"(d[i])
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : R16(OUT, 0)
        : "r"(taddr));
#undef OUT
}
// wait for the loads and tie the destination registers to the wait, so no
// consumer is scheduled ahead of it
__device__ __forceinline__ void tmem_wait16(uint32_t (&d)[16]) {
#define IO(i) "+r"(d[i])
    asm volatile("tcgen05.wait::ld.sync.aligned;" : R16(IO, 0)::"memory");
#undef IO
}

template <int MODE, int SIGN>
__device__ __forceinline__ void fft256_x(float2 (&v)[16], float2* buf, int t, const float2* tw16, uint32_t taddr) {
    if constexpr (MODE == 0) {
        fft256_half<SIGN>(v, buf, nullptr, t, 0, tw16);
    } else {
        fft_reg<16, SIGN>(v);
        uint32_t wa[16], wb[16];
        if constexpr (MODE == 1) {  // both chunks in flight across the exchange
            tmem_ld16(taddr, wa);
            tmem_ld16(taddr + 16, wb);
        }
        __syncwarp();
        float2* wp = buf + 17 * t;
#pragma unroll
        for (int k = 0; k < 16; ++k) wp[k] = v[k];
        __syncwarp();
        if constexpr (MODE == 2) tmem_ld16(taddr, wa);
        const float2* rp = buf + t;
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m] = rp[17 * m];
        if constexpr (MODE == 1) {
            tmem_wait16(wa);
            tmem_wait16(wb);
        } else {
            tmem_wait16(wa);
            tmem_ld16(taddr + 16, wb);
        }
#pragma unroll
        for (int m = 1; m < 8; ++m) {
            float2 w = make_float2(__uint_as_float(wa[2 * m]), __uint_as_float(wa[2 * m + 1]));
            if constexpr (SIGN > 0) w.y = -w.y;
            v[m] = cmul(v[m], w);
        }
        if constexpr (MODE == 2) tmem_wait16(wb);
#pragma unroll
        for (int m = 8; m < 16; ++m) {
            float2 w = make_float2(__uint_as_float(wb[2 * (m - 8)]), __uint_as_float(wb[2 * (m - 8) + 1]));
            if constexpr (SIGN > 0) w.y = -w.y;
            v[m] = cmul(v[m], w);
        }
        fft_reg<16, SIGN>(v);
    }
}

template <int MODE>
__global__ void __launch_bounds__(256, 2) half_kernel(const float2* tw_g, float2* out, int reps) {
    __shared__ float2 tw16[256];
    __shared__ float2 scr[8][2][272];
    __shared__ uint32_t tmem_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, h = lane >> 4, t = lane & 15;
    for (int i = threadIdx.x; i < 256; i += 256) tw16[i] = tw_g[((i >> 4) * (i & 15)) & 255];
    uint32_t taddr = 0;
    if constexpr (MODE != 0) {
        tmem_alloc(&tmem_base, warp);
        taddr = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
        uint32_t d[16];
        for (int c = 0; c < 2; ++c) {
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const float2 w = tw_g[((m + 8 * c) * t) & 255];
                d[2 * m] = __float_as_uint(w.x);
                d[2 * m + 1] = __float_as_uint(w.y);
            }
            tmem_st16(taddr + 16 * c, d);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    __syncthreads();
    float2 v[16];
    for (int k = 0; k < 16; ++k) v[k] = make_float2(lane * 0.001f + k, h - k * 0.5f);
    float2* buf = scr[warp][h];
    for (int r = 0; r < reps; ++r) {
        fft256_x<MODE, -1>(v, buf, t, tw16, taddr);
        fft256_x<MODE, +1>(v, buf, t, tw16, taddr);
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = cscale(v[k], 1.f / 256.f);
    }
    float2 acc = make_float2(0, 0);
    for (int k = 0; k < 16; ++k) acc = cadd(acc, cscale(v[k], (float)(k + 1)));
    out[blockIdx.x * 256 + threadIdx.x] = acc;
    if constexpr (MODE != 0) tmem_free(tmem_base, warp);
}

template <class F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    std::vector<float2> t256(256);
    for (int k = 0; k < 256; ++k) t256[k] = make_float2((float)cos(-2 * M_PI * k / 256), (float)sin(-2 * M_PI * k / 256));
    float2 *d_tw, *d_out;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 2, reps = 400;
    cudaMalloc(&d_tw, 256 * 8);
    cudaMalloc(&d_out, 3 * grid * 256 * 8);
    cudaMemcpy(d_tw, t256.data(), 256 * 8, cudaMemcpyHostToDevice);
    std::vector<float2> o(3 * grid * 256);
    const char* names[3] = {"SMEM tw16 (15 LDS.64)", "TMEM 2 x x16 early", "TMEM 2 x x16 late"};
    float ms[3];
    ms[0] = timeit([&] { half_kernel<0><<<grid, 256>>>(d_tw, d_out, reps); });
    ms[1] = timeit([&] { half_kernel<1><<<grid, 256>>>(d_tw, d_out + grid * 256, reps); });
    ms[2] = timeit([&] { half_kernel<2><<<grid, 256>>>(d_tw, d_out + 2 * grid * 256, reps); });
    cudaMemcpy(o.data(), d_out, o.size() * 8, cudaMemcpyDeviceToHost);
    double clk = 1.965e9;
    for (int i = 0; i < 3; ++i) {
        double ffts = (double)grid * 16 * reps * 2;
        double diff = 0, ref = 0;
        for (int k = 0; k < grid * 256; ++k) {
            diff += std::hypot(o[i * grid * 256 + k].x - o[k].x, o[i * grid * 256 + k].y - o[k].y);
            ref += std::hypot(o[k].x, o[k].y);
        }
        printf("%-26s %.3f ms  %.1f SM-cycles per FFT_256  rel diff vs (a) %.2e\n", names[i], ms[i],
               ms[i] * 1e-3 * clk * sms / ffts, diff / ref);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
