// Dev microbenchmark: issue rate of the sm_100a packed-FP32 instructions
// (FADD2 / FMUL2 / FFMA2, PTX add/mul/fma.rn.f32x2) against their scalar forms,
// and of a complex multiply as FMUL2 + FFMA2 (operand-broadcast / swap
// modifiers) against the 4-instruction scalar form, in warp-instr/clk/SM and
// complex-op/clk/SM.
#include <cstdio>

__device__ __forceinline__ unsigned long long pk(float2 a) { return *reinterpret_cast<unsigned long long*>(&a); }
__device__ __forceinline__ float2 upk(unsigned long long a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    unsigned long long d;
    asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk(a)), "l"(pk(b)));
    return upk(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    unsigned long long d;
    asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk(a)), "l"(pk(b)));
    return upk(d);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c)));
    return upk(d);
}
__device__ __forceinline__ float2 cmul_p(float2 a, float2 b) {  // FMUL2 + FFMA2
    const float2 t = mul2(make_float2(a.y, a.y), make_float2(-b.y, b.x));
    return fma2(make_float2(a.x, a.x), b, t);
}
__device__ __forceinline__ float2 cmul_s(float2 a, float2 b) {  // 2 FMUL + 2 FFMA
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}

template <int KIND>
__global__ void __launch_bounds__(256) kern(float2* out, int reps, float s) {
    float2 a[8];
    for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    float2 b = make_float2(s * 0.9999f, s * 1e-4f), c = make_float2(s * 1e-3f, -s * 1e-3f);
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (KIND == 0) a[i] = add2(a[i], b);                                  // FADD2
            if (KIND == 1) a[i] = fma2(a[i], b, c);                               // FFMA2
            if (KIND == 2) a[i] = make_float2(a[i].x + b.x, a[i].y + b.y);        // 2 FADD
            if (KIND == 3) a[i] = cmul_p(a[i], b);                                // FMUL2 + FFMA2
            if (KIND == 4) a[i] = cmul_s(a[i], b);                                // 4 scalar
            if (KIND == 5) a[i] = add2(a[i], a[(i + 1) & 7]);                     // FADD2 distinct regs
        }
    }
    float2 acc = make_float2(0.f, 0.f);
    for (int i = 0; i < 8; ++i) acc = make_float2(acc.x + a[i].x, acc.y + a[i].y);
    out[blockIdx.x * 256 + threadIdx.x] = acc;
}

template <int K>
void run(const char* name, float2* d, int sms, int instr_per_op) {
    const int grid = sms * 8, reps = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<K><<<grid, 256>>>(d, 16, 1.f);
    cudaEventRecord(e0);
    kern<K><<<grid, 256>>>(d, reps, 1.f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double ops = (double)grid * 8 * reps * 8;  // warp-level complex ops
    const double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
    printf("%-34s %.3f ms  %.2f warp-op/clk/SM  %.2f warp-instr/clk/SM\n", name, ms, per_clk_sm,
           per_clk_sm * instr_per_op);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float2* d;
    cudaMalloc(&d, sms * 8 * 256 * sizeof(float2));
    run<0>("cadd as FADD2", d, sms, 1);
    run<2>("cadd as 2 FADD", d, sms, 2);
    run<5>("cadd as FADD2 (distinct regs)", d, sms, 1);
    run<1>("FFMA2", d, sms, 1);
    run<3>("cmul as FMUL2 + FFMA2", d, sms, 2);
    run<4>("cmul as 2 FMUL + 2 FFMA", d, sms, 4);
    return 0;
}
