// Dev microbenchmark: FP32 issue ceiling on this GPU (FFMA 3-reg, FFMA with
// an immediate, FADD, FMUL), as warp-instructions per clock per SM.
#include <cstdio>

template <int KIND>
__global__ void __launch_bounds__(256) fp_kernel(float* out, int reps, float s) {
    float a[16];
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
    float b = s * 1.0001f, c = s * 0.9999f;
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (KIND == 0) a[i] = fmaf(a[i], b, c);          // 3-reg FFMA
            if (KIND == 1) a[i] = fmaf(a[i], 1.0001f, 0.5f); // FFMA with immediates
            if (KIND == 2) a[i] = a[i] + b;                   // FADD
            if (KIND == 3) a[i] = a[i] * b;                   // FMUL
            if (KIND == 4) a[i] = fmaf(a[i], a[(i + 1) & 15], b);  // 3 distinct regs
        }
    }
    float acc = 0;
    for (int i = 0; i < 16; ++i) acc += a[i];
    out[blockIdx.x * 256 + threadIdx.x] = acc;
}

template <int K>
double run(const char* name, float* d, int sms) {
    const int grid = sms * 8, reps = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fp_kernel<K><<<grid, 256>>>(d, 16, 1.f);
    cudaEventRecord(e0);
    fp_kernel<K><<<grid, 256>>>(d, reps, 1.f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double warp_instr = (double)grid * 8 * reps * 16;
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-28s %.3f ms  %.2f Twarp-instr/s  = %.2f warp-instr/clk/SM at %.0f MHz (%.1f TFLOP/s-equiv x32 lanes)\n", name, ms,
           warp_instr / (ms * 1e-3) / 1e12, warp_instr / (ms * 1e-3) / (clk * 1e3) / sms, clk / 1e3,
           warp_instr * 32 * (K == 0 || K == 1 || K == 4 ? 2 : 1) / (ms * 1e-3) / 1e12);
    return warp_instr * 32 * (K == 0 || K == 1 || K == 4 ? 2 : 1) / (ms * 1e-3) / 1e12;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* d;
    cudaMalloc(&d, sms * 8 * 256 * 4);
    const double f0 = run<0>("FFMA a*b+c (3 reg)", d, sms);
    run<1>("FFMA a*imm+imm", d, sms);
    run<2>("FADD", d, sms);
    run<3>("FMUL", d, sms);
    const double f4 = run<4>("FFMA 3 distinct regs", d, sms);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    // the JSON line bench.py reads (profiles/fp32_peak.json): FFMA TFLOP/s (2 flop per lane)
    printf("{\"ffma_tflops\": %.2f, \"ffma_3distinct_tflops\": %.2f, \"sms\": %d, \"clock_mhz\": %.0f, "
           "\"how\": \"tools/ubench_fp32.cu: 8 CTAs x 256 thr per SM, 16 independent FFMA chains\"}\n",
           f0, f4, sms, clk / 1e3);
    return 0;
}
