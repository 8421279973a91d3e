// Reference-granularity entry points of the symbol-synchronized path
// (include/fcwave/fc_sync.hpp:38-75): tx_symbol, combine_symbols,
// rx_block_freq, rx_symbol_simplified and rx_symbol_direct, each batched over
// S items (units) of one (subband, symbol) on the device.  These serve
// callers of the reference's per-symbol API; the hot path is the fused
// whole-frame K-TX / K-RX (fcw_device.cuh), which these kernels do not use.
//
// One CTA (256 threads) per item.  Transforms of any power-of-two length
// n <= 4096 run as a radix-2 Stockham autosort FFT through two SMEM buffers
// (natural order in and out), twiddles from the plan's N-entry table
// exp(-2 pi i k / N).  All arithmetic is complex fp32; the per-call constants
// (symbol / block phases, scales) are computed on the host in double.
#include "fcw_fft.cuh"
#include "fcw_internal.hpp"

namespace fcw {
namespace {

constexpr int kSymThreads = 256;

// Stockham radix-2 FFT of n points in a (natural order); returns the buffer
// holding the result (a or b).  SIGN = -1 forward, +1 inverse (unscaled).
// tw: exp(-2 pi i k / N), W_n^k = tw[k N / n].
template <int SIGN>
__device__ float2* smem_fft(float2* a, float2* b, int n, const float2* __restrict__ tw, int N) {
    for (int p = 1; p < n; p <<= 1) {
        for (int i = threadIdx.x; i < n / 2; i += blockDim.x) {
            const int k = i & (p - 1);
            const float2 u0 = a[i];
            float2 w = __ldg(&tw[(long long)k * N / (2 * p)]);
            if (SIGN > 0) w.y = -w.y;
            const float2 u1 = cmul(a[i + n / 2], w);
            const int j = (i << 1) - k;
            b[j] = cadd(u0, u1);
            b[j + p] = csub(u0, u1);
        }
        __syncthreads();
        float2* t = a;
        a = b;
        b = t;
    }
    return a;
}

// Subband window weight w[p0] from the plan's bin-class row (fcw_capi.cpp:
// entry b holds bits(w[b ^ L/2])).
__device__ __forceinline__ float win(const int2* __restrict__ cls, int cls_off, int L, int p0) {
    return __int_as_float(__ldg(&cls[cls_off + (p0 ^ (L / 2))]).y);
}

// tx_symbol (fc_sync.cpp:60-84): 3N/2 filtered samples of one CP-OFDM symbol
// of L + l_cp samples.  zero_pad_symbol (:34-43), block r windows (first
// block: first_block_analysis_window :52-58, second: analysis_window
// fc_core.cpp:57-61), synth_core (fc_core.cpp:76-90) per block, OLA at N/2.
struct TxSymArgs {
    const float2* sym;
    long long sym_stride;
    float2* out;
    long long out_stride;
    const float2* tw;
    const int2* cls;
    int cls_off, L, N, c, l_cp, L_L, L_S;
    float2 phase[2];  // block_phase(r) * theta_n
    float scale;      // sqrt(I)
};

__global__ void __launch_bounds__(kSymThreads) tx_symbol_kernel(const TxSymArgs A) {
    extern __shared__ float4 smem_raw[];
    float2* bufa = reinterpret_cast<float2*>(smem_raw);
    float2* bufb = bufa + A.N;
    float2* acc = bufb + A.N;  // 3N/2 output accumulator
    const float2* sym = A.sym + (long long)blockIdx.x * A.sym_stride;
    const int L = A.L, N = A.N, s_l = A.L_L - A.l_cp;
    for (int t = threadIdx.x; t < 3 * N / 2; t += blockDim.x) acc[t] = make_float2(0.f, 0.f);
    for (int r = 0; r < 2; ++r) {
        // x_w[i] = z[r L/2 + i] a_r[i], z[s_l + j] = sym[j] (j < L + l_cp)
        const int lo = r == 0 ? s_l : A.L_L, hi = r == 0 ? s_l + A.L_S + A.l_cp : A.L_L + A.L_S;
        for (int i = threadIdx.x; i < L; i += blockDim.x) {
            const int j = r * (L / 2) + i - s_l;
            bufa[i] = (i >= lo && i < hi && j >= 0 && j < L + A.l_cp) ? sym[j] : make_float2(0.f, 0.f);
        }
        __syncthreads();
        const float2* X = smem_fft<-1>(bufa, bufb, L, A.tw, N);
        // map into the N-bin spectrum (the other buffer): q = (c - ceil(L/2) + p0) mod N
        float2* spec = X == bufa ? bufb : bufa;
        for (int q = threadIdx.x; q < N; q += blockDim.x) spec[q] = make_float2(0.f, 0.f);
        __syncthreads();
        const int half = (L + 1) / 2;
        // the spectrum buffer must not alias X: for L < N it is the other buffer,
        // and X occupies at most L entries of its own
        for (int p0 = threadIdx.x; p0 < L; p0 += blockDim.x) {
            const int b = (p0 + L / 2) % L;
            const int q = (((A.c - half + p0) % N) + N) % N;
            spec[q] = cscale(cmul(X[b], A.phase[r]), win(A.cls, A.cls_off, L, p0));
        }
        __syncthreads();
        float2* other = spec == bufa ? bufb : bufa;
        const float2* y = smem_fft<+1>(spec, other, N, A.tw, N);
        const float s = A.scale / (float)N;  // fft::inverse's 1/N and sqrt(I)
        for (int t = threadIdx.x; t < N; t += blockDim.x) acc[r * (N / 2) + t] = cadd(acc[r * (N / 2) + t], cscale(y[t], s));
        __syncthreads();
    }
    float2* out = A.out + (long long)blockIdx.x * A.out_stride;
    for (int t = threadIdx.x; t < 3 * N / 2; t += blockDim.x) out[t] = acc[t];
}

// combine_symbols (fc_sync.cpp:96-112): symbol n's 3N/2 samples added at
// sigma_n, in symbol order, onto zeros.  One thread per output sample.
__global__ void combine_kernel(const float2* __restrict__ syms, long long sym_unit_stride, int B, int N,
                               const SymDev* __restrict__ sym, float2* __restrict__ wave, long long wave_stride,
                               long long Q) {
    const int s = blockIdx.y;
    const float2* su = syms + (long long)s * sym_unit_stride;
    float2* w = wave + (long long)s * wave_stride;
    const int len = 3 * N / 2;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < Q; t += (long long)gridDim.x * blockDim.x) {
        // last symbol with sigma <= t (binary search), then walk back while it still covers t
        int lo = 0, hi = B - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) / 2;
            if (__ldg(&sym[mid].sigma) <= t) lo = mid;
            else hi = mid - 1;
        }
        int first = lo;
        while (first > 0 && t - __ldg(&sym[first - 1].sigma) < len) --first;
        float2 v = make_float2(0.f, 0.f);
        for (int n = first; n <= lo; ++n) {
            const long long o = t - __ldg(&sym[n].sigma);
            if (o >= 0 && o < len) v = cadd(v, su[(long long)n * len + o]);
        }
        w[t] = v;
    }
}

// rx_block_freq (fc_sync.cpp:178-193): g[b] = conj(phase) w[p0] FFT_N(y)[q].
struct BlockFreqArgs {
    const float2* y;
    long long y_stride;
    float2* g;
    long long g_stride;
    const float2* tw;
    const int2* cls;
    int cls_off, L, N, c;
    float2 cph;  // conj(phase)
};

__global__ void __launch_bounds__(kSymThreads) rx_block_freq_kernel(const BlockFreqArgs A) {
    extern __shared__ float4 smem_raw[];
    float2* bufa = reinterpret_cast<float2*>(smem_raw);
    float2* bufb = bufa + A.N;
    const float2* y = A.y + (long long)blockIdx.x * A.y_stride;
    for (int t = threadIdx.x; t < A.N; t += blockDim.x) bufa[t] = y[t];
    __syncthreads();
    const float2* Y = smem_fft<-1>(bufa, bufb, A.N, A.tw, A.N);
    float2* g = A.g + (long long)blockIdx.x * A.g_stride;
    const int L = A.L, half = (L + 1) / 2;
    for (int p0 = threadIdx.x; p0 < L; p0 += blockDim.x) {
        const int b = (p0 + L / 2) % L;
        const int q = (((A.c - half + p0) % A.N) + A.N) % A.N;
        g[b] = cscale(cmul(Y[q], A.cph), win(A.cls, A.cls_off, L, p0));
    }
}

// W_L^(phi q) v (omega of rx_symbol_simplified, fc_sync.cpp:206-215)
__device__ __forceinline__ float2 omega(const float2* __restrict__ tw, int N, int L, int phi, int q, float2 v) {
    const long long e = (((long long)phi * q) % L + L) % L;
    return cmul(v, __ldg(&tw[e * (N / L)]));
}

// rx_symbol_simplified (fc_sync.cpp:195-243), Eq. (30) of the paper.
struct SimplArgs {
    const float2 *g0, *g1;
    long long g_stride;
    float2* out;
    long long out_stride;
    const float2* tw;
    int L, N, L_L, L_S;
    float scale;  // sqrt(I) (L / N) / sqrt(L)
};

__global__ void __launch_bounds__(kSymThreads) rx_simplified_kernel(const SimplArgs A) {
    extern __shared__ float4 smem_raw[];
    const int L = A.L, N = A.N;
    float2* bufa = reinterpret_cast<float2*>(smem_raw);
    float2* bufb = bufa + L;
    float2* tt = bufb + L;  // t = Omega_{L/2} g1
    const float2* g0 = A.g0 + (long long)blockIdx.x * A.g_stride;
    const float2* g1 = A.g1 + (long long)blockIdx.x * A.g_stride;
    for (int q = threadIdx.x; q < L; q += blockDim.x) {
        const float2 t = omega(A.tw, N, L, L / 2, q, g1[q]);
        tt[q] = t;
        bufa[q] = omega(A.tw, N, L, -L / 4, q, csub(g0[q], t));  // f = Omega_{-L/4}(g0 - t)
    }
    __syncthreads();
    float2* f = smem_fft<+1>(bufa, bufb, L, A.tw, N);  // fft::inverse (1/L below)
    float2* o = f == bufa ? bufb : bufa;
    // S-hat: the low-rate synthesis window [L_L, L_L + L_S) shifted by L/4
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        const int k = (i + L / 4) % L;
        f[i] = (k >= A.L_L && k < A.L_L + A.L_S) ? cscale(f[i], 1.f / (float)L) : make_float2(0.f, 0.f);
    }
    __syncthreads();
    f = smem_fft<-1>(f, o, L, A.tw, N);
    float2* out = A.out + (long long)blockIdx.x * A.out_stride;
    for (int q = threadIdx.x; q < L; q += blockDim.x) {
        const float2 v = cadd(omega(A.tw, N, L, L / 4, q, f[q]), tt[q]);
        out[q] = cscale(omega(A.tw, N, L, -L / 4, q, v), A.scale);
    }
}

// rx_symbol_direct (fc_sync.cpp:158-176): afb_block_ols (fc_core.cpp:144-153)
// of both blocks, central halves, ofdm_demodulate (ofdm.cpp:125-131).
struct DirectArgs {
    const float2 *y0, *y1;
    long long y_stride;
    float2* out;
    long long out_stride;
    const float2* tw;
    const int2* cls;
    int cls_off, L, N, c, L_L, L_S;
    float2 cph[2];  // conj(block_phase(r) theta_n)
    float scale;    // sqrt(I)
};

__global__ void __launch_bounds__(kSymThreads) rx_direct_kernel(const DirectArgs A) {
    extern __shared__ float4 smem_raw[];
    const int L = A.L, N = A.N, half = (L + 1) / 2;
    float2* bufa = reinterpret_cast<float2*>(smem_raw);
    float2* bufb = bufa + N;
    float2* x = bufb + N;  // x_ofdm, L entries
    for (int r = 0; r < 2; ++r) {
        const float2* y = (r == 0 ? A.y0 : A.y1) + (long long)blockIdx.x * A.y_stride;
        for (int t = threadIdx.x; t < N; t += blockDim.x) bufa[t] = y[t];
        __syncthreads();
        const float2* Y = smem_fft<-1>(bufa, bufb, N, A.tw, N);
        float2* Z = Y == bufa ? bufb : bufa;
        __syncthreads();
        for (int p0 = threadIdx.x; p0 < L; p0 += blockDim.x) {
            const int b = (p0 + L / 2) % L;
            const int q = (((A.c - half + p0) % N) + N) % N;
            Z[b] = cscale(cmul(Y[q], A.cph[r]), win(A.cls, A.cls_off, L, p0));
        }
        __syncthreads();
        float2* Zo = Z == bufa ? bufb : bufa;
        const float2* z = smem_fft<+1>(Z, Zo, L, A.tw, N);
        // (1/L of fft::inverse) (L/N) sqrt(I); synthesis window [L_L, L_L + L_S); central half
        const float s = A.scale / (float)N;
        for (int i = threadIdx.x; i < L / 2; i += blockDim.x) {
            const int k = L / 4 + i;
            x[r * (L / 2) + i] = (k >= A.L_L && k < A.L_L + A.L_S) ? cscale(z[k], s) : make_float2(0.f, 0.f);
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < L; i += blockDim.x) bufa[i] = x[i];
    __syncthreads();
    const float2* X = smem_fft<-1>(bufa, bufb, L, A.tw, N);
    float2* out = A.out + (long long)blockIdx.x * A.out_stride;
    const float s = rsqrtf((float)L);
    for (int q = threadIdx.x; q < L; q += blockDim.x) out[q] = cscale(X[q], s);
}

cudaError_t launch_sym(const void* k, void** args, int S, size_t smem, cudaStream_t st) {
    static std::mutex mu;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (smem > 48 * 1024) {
            const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
        }
    }
    return cudaLaunchKernel(k, dim3(S), dim3(kSymThreads), args, smem, st);
}

}  // namespace

cudaError_t sym_tx_symbol(const Plan& p, int m, const float2* sym, long long sym_stride, int l_cp, float2 ph0,
                          float2 ph1, float scale, float2* out, long long out_stride, int S, cudaStream_t st) {
    const auto& sb = p.subs[m];
    TxSymArgs a{sym, sym_stride, out, out_stride, p.d_tw, p.d_cls, p.h_sub[m].cls_off, sb.desc.L, p.N,
                sb.desc.c, l_cp, sb.p.L_L, sb.p.L_S, {ph0, ph1}, scale};
    void* args[] = {&a};
    return launch_sym(reinterpret_cast<const void*>(tx_symbol_kernel), args, S, sizeof(float2) * (3.5 * p.N), st);
}

cudaError_t sym_combine(const Plan& p, const float2* syms, long long sym_unit_stride, float2* wave,
                        long long wave_stride, int S, cudaStream_t st) {
    const int gx = (int)std::min<long long>((p.Q + 255) / 256, 4LL * device_sms());
    combine_kernel<<<dim3(gx, S), 256, 0, st>>>(syms, sym_unit_stride, p.B, p.N, p.d_sym, wave, wave_stride, p.Q);
    return cudaGetLastError();
}

cudaError_t sym_rx_block_freq(const Plan& p, int m, const float2* y, long long y_stride, float2 cph, float2* g,
                              long long g_stride, int S, cudaStream_t st) {
    const auto& sb = p.subs[m];
    BlockFreqArgs a{y, y_stride, g, g_stride, p.d_tw, p.d_cls, p.h_sub[m].cls_off, sb.desc.L, p.N, sb.desc.c, cph};
    void* args[] = {&a};
    return launch_sym(reinterpret_cast<const void*>(rx_block_freq_kernel), args, S, sizeof(float2) * 2 * p.N, st);
}

cudaError_t sym_rx_simplified(const Plan& p, int m, const float2* g0, const float2* g1, long long g_stride,
                              float scale, float2* out, long long out_stride, int S, cudaStream_t st) {
    const auto& sb = p.subs[m];
    const int L = sb.desc.L;
    SimplArgs a{g0, g1, g_stride, out, out_stride, p.d_tw, L, p.N, sb.p.L_L, sb.p.L_S, scale};
    void* args[] = {&a};
    return launch_sym(reinterpret_cast<const void*>(rx_simplified_kernel), args, S, sizeof(float2) * 3 * L, st);
}

cudaError_t sym_rx_direct(const Plan& p, int m, const float2* y0, const float2* y1, long long y_stride, float2 cph0,
                          float2 cph1, float scale, float2* out, long long out_stride, int S, cudaStream_t st) {
    const auto& sb = p.subs[m];
    DirectArgs a{y0, y1, y_stride, out, out_stride, p.d_tw, p.d_cls, p.h_sub[m].cls_off, sb.desc.L, p.N,
                 sb.desc.c, sb.p.L_L, sb.p.L_S, {cph0, cph1}, scale};
    void* args[] = {&a};
    return launch_sym(reinterpret_cast<const void*>(rx_direct_kernel), args, S,
                      sizeof(float2) * (2 * p.N + sb.desc.L), st);
}

}  // namespace fcw
