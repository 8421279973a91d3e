// Dev microbenchmark (not part of the product): does a packed FP32 instruction
// (FFMA2, two cycles on the FMA pipe) block the warp scheduler's issue port for
// both cycles, or can integer / shared-memory instructions issue in its shadow?
// Each kernel runs REPS iterations of a body with NF independent FFMA2 (or 2 NF
// scalar FFMA) plus NI independent integer ops (LOP3/IADD3) plus NL LDS per
// thread; cycles per iteration per SM sub-partition tell how the slots add up.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int REPS = 4096;

template <int PACKED, int NI, int NL>
__global__ void __launch_bounds__(256, 2) k(float2* out, int* iout, float s, int q) {
    __shared__ float sm[1024];
    for (int i = threadIdx.x; i < 1024; i += 256) sm[i] = i * s;
    __syncthreads();
    float2 a[8];
    int b[8];
    float l[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = make_float2(threadIdx.x * 1e-3f + i, s * i);
        b[i] = threadIdx.x + i * q;
    }
    const float2 m = make_float2(s, 1.0f - s), c = make_float2(1e-3f, s);
    const float* p = sm + (threadIdx.x & 31);
    for (int r = 0; r < REPS; ++r) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (PACKED) {
                a[i] = __ffma2_rn(a[i], m, c);
            } else {
                a[i].x = fmaf(a[i].x, m.x, c.x);
                a[i].y = fmaf(a[i].y, m.y, c.y);
            }
            if (i < NI) b[i] = (b[i] ^ q) + (b[i] >> 3);  // 2 integer instructions (LOP3/SHF + IADD3)
            if (i < NL) l[i & 3] += p[((r + i) & 31) * 32];
        }
    }
    float2 acc = make_float2(l[0] + l[1], l[2] + l[3]);
    int ib = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        acc.x += a[i].x;
        acc.y += a[i].y;
        ib += b[i];
    }
    out[blockIdx.x * 256 + threadIdx.x] = acc;
    iout[blockIdx.x * 256 + threadIdx.x] = ib;
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
    int sms = 148, khz = 1965000;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    float2* o;
    int* io;
    cudaMalloc(&o, sms * 2 * 256 * 8);
    cudaMalloc(&io, sms * 2 * 256 * 4);
    const int grid = sms * 2;  // 16 warps per SM = 4 per sub-partition
    auto rep = [&](const char* name, float ms, int nf_slots, int ni, int nl) {
        // per sub-partition: 4 warps x REPS iterations
        const double cyc = ms * 1e-3 * khz * 1e3 / (4.0 * REPS);
        printf("%-44s %.3f ms  %.2f cycles / (warp-iteration)  [8 FFMA2-equivalents + %d int + %d LDS]\n", name, ms, cyc,
               2 * ni, nl);
    };
    rep("8 FFMA2", timeit([&] { k<1, 0, 0><<<grid, 256>>>(o, io, 0.5f, 3); }), 16, 0, 0);
    rep("16 FFMA (scalar)", timeit([&] { k<0, 0, 0><<<grid, 256>>>(o, io, 0.5f, 3); }), 16, 0, 0);
    rep("8 FFMA2 + 8 int", timeit([&] { k<1, 4, 0><<<grid, 256>>>(o, io, 0.5f, 3); }), 16, 4, 0);
    rep("16 FFMA + 8 int", timeit([&] { k<0, 4, 0><<<grid, 256>>>(o, io, 0.5f, 3); }), 16, 4, 0);
    rep("8 FFMA2 + 16 int", timeit([&] { k<1, 8, 0><<<grid, 256>>>(o, io, 0.5f, 3); }), 16, 8, 0);
    rep("16 FFMA + 16 int", timeit([&] { k<0, 8, 0><<<grid, 256>>>(o, io, 0.5f, 3); }), 16, 8, 0);
    rep("8 FFMA2 + 4 LDS", timeit([&] { k<1, 0, 4><<<grid, 256>>>(o, io, 0.5f, 3); }), 16, 0, 4);
    rep("16 FFMA + 4 LDS", timeit([&] { k<0, 0, 4><<<grid, 256>>>(o, io, 0.5f, 3); }), 16, 0, 4);
    rep("8 FFMA2 + 8 int + 4 LDS", timeit([&] { k<1, 4, 4><<<grid, 256>>>(o, io, 0.5f, 3); }), 16, 4, 4);
    rep("16 FFMA + 8 int + 4 LDS", timeit([&] { k<0, 4, 4><<<grid, 256>>>(o, io, 0.5f, 3); }), 16, 4, 4);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
