// Dev microbenchmark (not part of the product): throughput of the warp-team
// short FFT and the CTA-team long FFT building blocks in isolation.
#include <cstdio>
#include <vector>

#include "fcw_fft.cuh"

using namespace fcw;

template <int L, int NF>
__global__ void __launch_bounds__(256, 2) warp_fft_kernel(const float2* tw_g, float2* out, int reps) {
    constexpr int PPT = L / 32;
    __shared__ float2 stw[L];
    __shared__ float2 scr[8][2][L + L / 16 + 2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < L; i += 256) stw[i] = tw_g[i];
    __syncthreads();
    float2 v[NF][PPT];
    for (int f = 0; f < NF; ++f)
        for (int k = 0; k < PPT; ++k) v[f][k] = make_float2(lane * 0.001f + k, f - k * 0.5f);
    float2* const b[2] = {scr[warp][0], scr[warp][1]};
    for (int r = 0; r < reps; ++r) {
        team_fft<L, 32, PPT, -1, NF, false>(v, b, stw, 1, lane, true);
        team_fft<L, 32, PPT, +1, NF, false>(v, b, stw, 1, lane, true);
    }
    float2 acc = make_float2(0, 0);
    for (int f = 0; f < NF; ++f)
        for (int k = 0; k < PPT; ++k) acc = cadd(acc, v[f][k]);
    out[blockIdx.x * 256 + threadIdx.x] = acc;
}

// Half-warp teams: each 16-lane half of a warp transforms its own FFT_L with
// L/16 points per lane (radix-16 x 16 for L = 256: one exchange).
template <int L>
__global__ void __launch_bounds__(256, 2) half_fft_kernel(const float2* tw_g, float2* out, int reps) {
    constexpr int PPT = L / 16;
    __shared__ float2 stw[L];
    __shared__ float2 scr[8][2][L + L / 16 + 2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, h = lane >> 4, t = lane & 15;
    for (int i = threadIdx.x; i < L; i += 256) stw[i] = tw_g[i];
    __syncthreads();
    float2 v[1][PPT];
    for (int k = 0; k < PPT; ++k) v[0][k] = make_float2(lane * 0.001f + k, h - k * 0.5f);
    float2* const b[1] = {scr[warp][h]};
    for (int r = 0; r < reps; ++r) {
        team_fft<L, 16, PPT, -1, 1, false>(v, b, stw, 1, t, true);
        team_fft<L, 16, PPT, +1, 1, false>(v, b, stw, 1, t, true);
    }
    float2 acc = make_float2(0, 0);
    for (int k = 0; k < PPT; ++k) acc = cadd(acc, v[0][k]);
    out[blockIdx.x * 256 + threadIdx.x] = acc;
}

template <int N>
__global__ void __launch_bounds__(256, 2) cta_fft_kernel(const float2* tw_g, float2* out, int reps) {
    constexpr int T = N / 16;
    extern __shared__ float2 sm[];
    float2* b0 = sm;
    float2* b1 = sm + N + N / 16 + 2;
    const int tid = threadIdx.x;
    float2 v[2][16];
    for (int k = 0; k < 16; ++k) {
        v[0][k] = make_float2(tid * 0.001f + k, -k * 0.5f);
        v[1][k] = make_float2(k * 0.25f, tid * 0.002f);
    }
    float2* const b[2] = {b0, b1};
    for (int r = 0; r < reps; ++r) {
        team_fft<N, T, 16, -1, 2, true>(v, b, tw_g, 1, tid, tid < T);
        team_fft<N, T, 16, +1, 2, true>(v, b, tw_g, 1, tid, tid < T);
    }
    float2 acc = make_float2(0, 0);
    for (int f = 0; f < 2; ++f)
        for (int k = 0; k < 16; ++k) acc = cadd(acc, v[f][k]);
    out[blockIdx.x * 256 + threadIdx.x] = acc;
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
    const int N = 4096;
    std::vector<float2> tw(N);
    for (int k = 0; k < N; ++k) tw[k] = make_float2(cos(-2 * M_PI * k / N), sin(-2 * M_PI * k / N));
    float2 *d_tw, *d_tw256, *d_out;
    cudaMalloc(&d_tw, N * 8);
    cudaMalloc(&d_tw256, 256 * 8);
    cudaMalloc(&d_out, 148 * 8 * 256 * 8);
    cudaMemcpy(d_tw, tw.data(), N * 8, cudaMemcpyHostToDevice);
    std::vector<float2> t256(256);
    for (int k = 0; k < 256; ++k) t256[k] = tw[k * 16];
    cudaMemcpy(d_tw256, t256.data(), 256 * 8, cudaMemcpyHostToDevice);
    const int grid = 148 * 2, reps = 200;
    {
        float ms = timeit([&] { warp_fft_kernel<256, 1><<<grid, 256>>>(d_tw256, d_out, reps); });
        double ffts = (double)grid * 8 * reps * 2;
        printf("warp FFT_256 NF=1: %.3f ms, %.2f ns/FFT (GPU), %.0f cycles/FFT/SM @1.965GHz\n", ms, ms * 1e6 / ffts,
               ms * 1e-3 * 1.965e9 * 148 / ffts);
    }
    {
        float ms = timeit([&] { warp_fft_kernel<256, 2><<<grid, 256>>>(d_tw256, d_out, reps); });
        double ffts = (double)grid * 8 * reps * 2 * 2;
        printf("warp FFT_256 NF=2: %.3f ms, %.2f ns/FFT (GPU), %.0f cycles/FFT/SM\n", ms, ms * 1e6 / ffts,
               ms * 1e-3 * 1.965e9 * 148 / ffts);
    }
    {
        float ms = timeit([&] { half_fft_kernel<256><<<grid, 256>>>(d_tw256, d_out, reps); });
        double ffts = (double)grid * 8 * reps * 2 * 2;
        printf("half-warp FFT_256 (16x16, 16 pts/lane): %.3f ms, %.2f ns/FFT (GPU), %.0f cycles/FFT/SM\n", ms,
               ms * 1e6 / ffts, ms * 1e-3 * 1.965e9 * 148 / ffts);
    }
    {
        size_t smem = 2 * (N + N / 16 + 2) * 8;
        cudaFuncSetAttribute(cta_fft_kernel<4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        float ms = timeit([&] { cta_fft_kernel<4096><<<grid, 256, smem>>>(d_tw, d_out, reps / 4); });
        double ffts = (double)grid * (reps / 4) * 2 * 2;
        printf("CTA FFT_4096 x2 lockstep: %.3f ms, %.2f ns/FFT (GPU), %.0f cycles/FFT/SM\n", ms, ms * 1e6 / ffts,
               ms * 1e-3 * 1.965e9 * 148 / ffts);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
