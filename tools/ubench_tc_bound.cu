// Tensor cores for the FFT passes: a measured lower bound.
//
// A radix-16 pass of the long / short transforms does, per 16-point column, a
// DFT16 on the CUDA cores (fft_reg<16>, FFMA2/FADD2) between the twiddle
// multiply and the SMEM exchange.  On tcgen05 the same pass is a GEMM
// D[128 x 32] = X^T[128 x 32] F^T[32 x 32] (re/im real-ified), which needs
// split precision to meet north_star's 1e-5 (fp16 x3: hi*hi + hi*lo + lo*hi,
// or tf32 x3).  The MMA itself is asynchronous and nearly free at these
// sizes, but the CUDA cores still have to
//   (1) split every fp32 value into hi/lo operands,
//   (2) store both operands into the SMEM operand tiles, and
//   (3) read the fp32 accumulator back from TMEM (tcgen05.ld) —
// work the FP32 path does not do.  This benchmark times (1)-(3) alone
// (no MMA, no mbarrier wait: a LOWER bound on the tensor-core pass) against
// the FP32 DFT16 it would replace, per column, at the kernels' occupancy
// (2 CTAs x 256 threads per SM, 16 complex values per thread).  If the bound
// is not below the FP32 cost, tensor cores cannot speed up these passes.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2008_00672_b200/csrc -I include -o /tmp/ubtc tools/ubench_tc_bound.cu
#include <cuda_fp16.h>

#include <cstdint>

#include <cstdio>

#include "fcw_fft.cuh"

using namespace fcw;

constexpr int kReps = 2048;

// operand-tile store that the compiler cannot drop (the MMA would read it)
__device__ __forceinline__ void sts128(void* p, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// FP32 path: one DFT16 per column (the kernels' fft_reg<16>).
__global__ void __launch_bounds__(256, 2) fp32_dft16(float2* out, float s) {
    float2 v[16];
    for (int k = 0; k < 16; ++k) v[k] = make_float2(threadIdx.x * 1e-3f + k, s * k);
    for (int r = 0; r < kReps; ++r) {
        fft_reg<16, -1>(v);
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k].x += s;  // new data every iteration (same in every variant)
    }
    float2 a = make_float2(0.f, 0.f);
    for (int k = 0; k < 16; ++k) a = cadd(a, v[k]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}

// tcgen05 fp16x3 path, CUDA-core side: split into fp16 hi/lo, store both
// operand rows (K-major, 64 B each) to SMEM, read 32 fp32 accumulator
// columns back from TMEM.
__global__ void __launch_bounds__(256, 2) tc_side_fp16(float2* out, float s) {
    __shared__ __align__(128) uint4 tile[256 * 8];  // hi 64 B + lo 64 B per row, core-matrix interleaved
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // warp w of a CTA may access TMEM lanes 32 (w mod 4) .. +32
    const uint32_t taddr = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
    float2 v[16];
    for (int k = 0; k < 16; ++k) v[k] = make_float2(threadIdx.x * 1e-3f + k, s * k);
    // 16-byte chunk q of row t at tile[q * 256 + t]: consecutive rows 16 B
    // apart as in the UMMA no-swizzle K-major core matrices (conflict-free)
    uint4* row = tile + threadIdx.x;
    for (int r = 0; r < kReps; ++r) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const __half2 h = __float22half2_rn(v[k]);
            const float2 back = __half22float2(h);
            const __half2 l = __float22half2_rn(make_float2(v[k].x - back.x, v[k].y - back.y));
            hi[k] = *reinterpret_cast<const uint32_t*>(&h);
            lo[k] = *reinterpret_cast<const uint32_t*>(&l);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            sts128(row + q * 256, make_uint4(hi[4 * q], hi[4 * q + 1], hi[4 * q + 2], hi[4 * q + 3]));
            sts128(row + (4 + q) * 256, make_uint4(lo[4 * q], lo[4 * q + 1], lo[4 * q + 2], lo[4 * q + 3]));
        }
        // accumulator readback: 32 fp32 columns of this thread's TMEM lane
        uint32_t d[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
              "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]),
              "=r"(d[15]), "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]),
              "=r"(d[22]), "=r"(d[23]), "=r"(d[24]), "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]),
              "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int k = 0; k < 16; ++k)
            v[k] = make_float2(__uint_as_float(d[2 * k]), __uint_as_float(d[2 * k + 1]));  // D -> next pass
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k].x += s;
    }
    float2 a = make_float2(0.f, 0.f);
    for (int k = 0; k < 16; ++k) a = cadd(a, v[k]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = a;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem_base));
}

// tcgen05 tf32x3 path, CUDA-core side: hi = x with the low 13 mantissa bits
// cleared, lo = x - hi (both fp32 operands, 128 B per row each), readback.
__global__ void __launch_bounds__(256, 2) tc_side_tf32(float2* out, float s) {
    extern __shared__ uint4 tile_d[];  // per thread: hi 128 B + lo 128 B
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t taddr = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
    float2 v[16];
    for (int k = 0; k < 16; ++k) v[k] = make_float2(threadIdx.x * 1e-3f + k, s * k);
    uint4* row = tile_d + threadIdx.x;
    for (int r = 0; r < kReps; ++r) {
        float2 hi[16], lo[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            hi[k] = make_float2(__uint_as_float(__float_as_uint(v[k].x) & 0xFFFFE000u),
                                __uint_as_float(__float_as_uint(v[k].y) & 0xFFFFE000u));
            lo[k] = csub(v[k], hi[k]);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            sts128(row + q * 256, *reinterpret_cast<const uint4*>(&hi[2 * q]));
            sts128(row + (8 + q) * 256, *reinterpret_cast<const uint4*>(&lo[2 * q]));
        }
        uint32_t d[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
              "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]),
              "=r"(d[15]), "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]),
              "=r"(d[22]), "=r"(d[23]), "=r"(d[24]), "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]),
              "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int k = 0; k < 16; ++k)
            v[k] = make_float2(__uint_as_float(d[2 * k]), __uint_as_float(d[2 * k + 1]));  // D -> next pass
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k].x += s;
    }
    float2 a = make_float2(0.f, 0.f);
    for (int k = 0; k < 16; ++k) a = cadd(a, v[k]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = a;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem_base));
}

template <class K>
double run(const char* name, K kern, float2* d, int sms, size_t smem) {
    const int grid = 2 * sms;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 256, smem>>>(d, 1.f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<grid, 256, smem>>>(d, 1.f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double cols = (double)grid * 256 * kReps;  // 16-point columns processed
    const double cyc = ms * 1e-3 * clk * 1e3 * sms / cols;
    printf("%-44s %8.3f ms  %6.2f SM-cycles per 16-point column  (%s)\n", name, ms, cyc,
           cudaGetErrorString(cudaGetLastError()));
    return cyc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float2* d = nullptr;
    cudaMalloc(&d, sizeof(float2) * 2 * sms * 256);
    const double a = run("FP32 DFT16 (fft_reg<16>, FFMA2/FADD2)", fp32_dft16, d, sms, 0);
    const double b = run("tcgen05 fp16x3 CUDA-core side (lower bound)", tc_side_fp16, d, sms, 0);
    const double c = run("tcgen05 tf32x3 CUDA-core side (lower bound)", tc_side_tf32, d, sms, 256 * 256);
    // the bound leaves out the MMA issue, commit / mbarrier round trip and the
    // B operand: a tensor-core pass can save at most this share of the DFT16 cost
    printf("{\"fp32_dft16_cycles\": %.2f, \"tc_fp16x3_side_cycles\": %.2f, \"tc_tf32x3_side_cycles\": %.2f, "
           "\"max_saving_fp16x3\": %.3f, \"max_saving_tf32x3\": %.3f}\n", a, b, c, (a - b) / a, (a - c) / a);
    return 0;
}
