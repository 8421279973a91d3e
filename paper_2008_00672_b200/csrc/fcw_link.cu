// Link step around the FC hot path: device-side
// hard-decision QAM demap with bit-error and EVM sums against the seeded
// transmit grid, AWGN and power measurement.  They replace the per-drop CPU
// loop of run_scenario (proj/src/scenario.cpp:469-494) with
//   qam_demap            ofdm.cpp:67-78
//   ber / evm_db sums    metrics.cpp:105-127
//   awgn_with_variance   channel.cpp:136-141 (GaussianRng::next_complex :37-42)
//   measure_power        channel.cpp:148-155
//
// All three are HBM-streaming passes.  The reductions are deterministic: a
// fixed element-to-thread map, a fixed shared-memory tree per chunk and an
// in-order sum of the chunk partials (no floating-point atomics).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "fcw_fft.cuh"
#include "fcw_internal.hpp"

namespace fcw {

namespace {

constexpr int kLinkThreads = 256;
constexpr int kLinkPerThread = 32;
constexpr long long kLinkChunk = (long long)kLinkThreads * kLinkPerThread;
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// GaussianRng(derive_seed(seed, index)) initial state (channel.cpp:26,45-48)
__device__ __forceinline__ uint64_t stream_state(uint64_t seed, uint64_t index) {
    uint64_t st = mix64((seed ^ (kGamma * (index + 1))) + kGamma);
    return st ? st : 0x1234567890abcdefULL;
}

// Draw j (1-based) of a splitmix64 stream is mix(state + j * gamma): the
// generator is counter-based, so element i's draws are independent of order.
__device__ __forceinline__ uint64_t draw(uint64_t st, uint64_t j) { return mix64(st + j * kGamma); }

__device__ __forceinline__ double pam_scale(int levels) {
    return 1.0 / sqrt(2.0 * ((double)levels * levels - 1.0) / 3.0);
}

// ofdm.cpp:73-78 slice: lround, clamp, Gray encode (double, like the reference)
__device__ __forceinline__ unsigned slice(double v, double s, int levels) {
    // static_cast<int>(std::lround(...)): narrowed to int (modular) before the clamp
    int idx = (int)llround((v / s - 1.0 + levels) / 2.0);
    idx = idx < 0 ? 0 : (idx >= levels ? levels - 1 : idx);
    return (unsigned)idx ^ ((unsigned)idx >> 1);
}

struct Acc {
    double a, b;
    long long e;
};

// Fixed-order block reduction of (a, b, e); thread 0 returns the total.
__device__ Acc block_reduce(Acc v) {
    __shared__ double sa[kLinkThreads], sb[kLinkThreads];
    __shared__ long long se[kLinkThreads];
    const int t = threadIdx.x;
    sa[t] = v.a;
    sb[t] = v.b;
    se[t] = v.e;
    __syncthreads();
    for (int h = kLinkThreads / 2; h > 0; h >>= 1) {
        if (t < h) {
            sa[t] += sa[t + h];
            sb[t] += sb[t + h];
            se[t] += se[t + h];
        }
        __syncthreads();
    }
    return Acc{sa[0], sb[0], se[0]};
}

// grid S*chunks: block u*chunks + c covers packed elements
// [c*kLinkChunk, (c+1)*kLinkChunk) of unit u's [B][A] grid.
__global__ void __launch_bounds__(kLinkThreads) link_stats_kernel(const float2* __restrict__ grid,
                                                                  long long stride, long long per_unit,
                                                                  uint64_t seed, long long unit0, int bits,
                                                                  int chunks, Acc* __restrict__ part) {
    const int u = blockIdx.x / chunks, c = blockIdx.x - u * chunks;
    const uint64_t st = stream_state(seed, (uint64_t)(unit0 + u));
    const int k = bits / 2, levels = 1 << k;
    const unsigned mask = (1u << k) - 1u;
    const double s = pam_scale(levels);
    Acc acc{0.0, 0.0, 0};
    const float2* g = grid + (long long)u * stride;
#pragma unroll 1
    for (int r = 0; r < kLinkPerThread; ++r) {
        const long long i = c * kLinkChunk + (long long)r * kLinkThreads + threadIdx.x;
        if (i >= per_unit) break;
        // transmitted symbol: scenario.cpp:120-128 draws, one per bit, LSB first
        unsigned sym = 0;
        for (int b = 0; b < bits; ++b) sym |= (unsigned)(draw(st, (uint64_t)i * bits + b + 1) & 1u) << b;
        unsigned gi = sym & mask, gq = (sym >> k) & mask, li = 0, lq = 0;
        for (; gi; gi >>= 1) li ^= gi;
        for (; gq; gq >>= 1) lq ^= gq;
        const double xr = s * (2.0 * li + 1 - levels), xi = s * (2.0 * lq + 1 - levels);
        const float2 y = g[i];
        const double dr = (double)y.x - xr, di = (double)y.y - xi;
        acc.a += dr * dr + di * di;
        acc.b += xr * xr + xi * xi;
        const unsigned got = slice((double)y.x, s, levels) | (slice((double)y.y, s, levels) << k);
        acc.e += __popc(got ^ sym);
    }
    const Acc tot = block_reduce(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// One thread per unit sums its chunk partials in chunk order.
__global__ void reduce_parts_kernel(const Acc* __restrict__ part, int chunks, int S, Acc* __restrict__ out) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= S) return;
    Acc t{0.0, 0.0, 0};
    for (int c = 0; c < chunks; ++c) {
        const Acc p = part[(long long)u * chunks + c];
        t.a += p.a;
        t.b += p.b;
        t.e += p.e;
    }
    out[u] = t;
}

// channel.cpp:136-141: v += sqrt(sigma2) * next_complex(), sample t of unit u
// using draws 2t+1, 2t+2 of GaussianRng(derive_seed(seed, unit0 + u)).
__global__ void awgn_kernel(float2* __restrict__ wave, long long stride, long long len, int S, double sd,
                            uint64_t seed, long long unit0) {
    const long long total = (long long)S * len;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long u = idx / len, t = idx - u * len;
        const uint64_t st = stream_state(seed, (uint64_t)(unit0 + u));
        const double u1 = ((double)(draw(st, 2 * (uint64_t)t + 1) >> 11) + 1.0) * 0x1p-53;
        const double u2 = (double)(draw(st, 2 * (uint64_t)t + 2) >> 11) * 0x1p-53;
        const double r = sqrt(-log(u1));
        double sn, cs;
        sincos(2.0 * 3.14159265358979323846 * u2, &sn, &cs);
        float2* p = wave + u * stride + t;
        const float2 v = *p;
        *p = make_float2((float)((double)v.x + sd * (r * cs)), (float)((double)v.y + sd * (r * sn)));
    }
}

// grid S*chunks: sum of |v|^2 over [begin, end) of each unit (channel.cpp:148-155)
__global__ void __launch_bounds__(kLinkThreads) power_kernel(const float2* __restrict__ wave, long long stride,
                                                             long long begin, long long end, int chunks,
                                                             Acc* __restrict__ part) {
    const int u = blockIdx.x / chunks, c = blockIdx.x - u * chunks;
    const float2* w = wave + (long long)u * stride;
    Acc acc{0.0, 0.0, 0};
#pragma unroll 1
    for (int r = 0; r < kLinkPerThread; ++r) {
        const long long t = begin + c * kLinkChunk + (long long)r * kLinkThreads + threadIdx.x;
        if (t >= end) break;
        const float2 v = w[t];
        acc.a += (double)v.x * v.x + (double)v.y * v.y;
    }
    const Acc tot = block_reduce(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// Two-stage deterministic reduction into host results.
template <class Launch>
cudaError_t reduce_to_host(int S, int chunks, cudaStream_t st, Launch&& launch, Acc* host) {
    Acc* d = nullptr;
    const size_t nparts = (size_t)S * chunks;
    cudaError_t e = scratch_alloc(&d, (nparts + S) * sizeof(Acc), st);
    if (e != cudaSuccess) return e;
    launch(d);
    reduce_parts_kernel<<<(S + 127) / 128, 128, 0, st>>>(d, chunks, S, d + nparts);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(host, d + nparts, S * sizeof(Acc), cudaMemcpyDeviceToHost, st);
    const cudaError_t f = cudaFreeAsync(d, st);
    if (e == cudaSuccess) e = f;
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e;
}

// ----------------------------------------------------- TDL channel (f3)
// channel.cpp:113-124 apply_channel, per unit its own tap line:
// out[t] = sum_k g_k in[t - d_k] over taps with d_k <= t, in tap order.
constexpr int kMaxTaps = 64;
__global__ void __launch_bounds__(256) channel_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                                                      long long stride, long long len, const int* __restrict__ delays,
                                                      const float2* __restrict__ gains, int n_taps) {
    __shared__ int sd[kMaxTaps];
    __shared__ float2 sg[kMaxTaps];
    const long long u = blockIdx.y;
    for (int k = threadIdx.x; k < n_taps; k += blockDim.x) {
        sd[k] = delays[u * n_taps + k];
        sg[k] = gains[u * n_taps + k];
    }
    __syncthreads();
    const float2* x = in + u * stride;
    float2* y = out + u * stride;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < len; t += (long long)gridDim.x * blockDim.x) {
        float2 acc = make_float2(0.f, 0.f);
        for (int k = 0; k < n_taps; ++k) {
            const long long j = t - sd[k];
            if (j >= 0) {
                const float2 v = __ldg(&x[j]);
                acc.x = fmaf(sg[k].x, v.x, fmaf(-sg[k].y, v.y, acc.x));
                acc.y = fmaf(sg[k].x, v.y, fmaf(sg[k].y, v.x, acc.y));
            }
        }
        y[t] = acc;
    }
}

// ---------------------------------------------------------- Welch PSD (f4)
// metrics.cpp:128-155: Hann-windowed segments, |FFT_L|^2 summed per bin.
// Grid (chunks, S): a CTA sums |X|^2 of segments [c*spc, (c+1)*spc) of unit u
// in double, in segment order per thread; warps (L <= 256: one segment per
// warp) or the whole CTA (L >= 512: T = L/16 threads x 16 points) transform;
// per-CTA partials are summed in chunk order by psd_reduce_kernel.
constexpr int kPsdSegPerCta = 32;

template <int L>
__global__ void __launch_bounds__(256) psd_kernel(const float2* __restrict__ wave, long long stride,
                                                  const float* __restrict__ win, int hop, int n_seg,
                                                  const float2* __restrict__ tw, int ts, double* __restrict__ part) {
    extern __shared__ float2 psd_smem[];
    const long long u = blockIdx.y;
    const float2* w = wave + u * stride;
    const int s0 = blockIdx.x * kPsdSegPerCta, s1 = min(n_seg, s0 + kPsdSegPerCta);
    double* dst = part + ((long long)u * gridDim.x + blockIdx.x) * L;
    if constexpr (L <= 256) {
        constexpr int PPT = L / 32;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        float2* const bufs[1] = {psd_smem + warp * (L + L / 16 + 2)};
        double acc[PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) acc[k] = 0.0;
        for (int sg = s0 + warp; sg < s1; sg += 8) {
            const float2* x = w + (long long)sg * hop;
            float2 v[1][PPT];
#pragma unroll
            for (int k = 0; k < PPT; ++k) v[0][k] = cscale(x[lane + 32 * k], win[lane + 32 * k]);
            team_fft<L, 32, PPT, -1, 1, false>(v, bufs, tw, ts, lane, true);
#pragma unroll
            for (int k = 0; k < PPT; ++k) acc[k] += (double)v[0][k].x * v[0][k].x + (double)v[0][k].y * v[0][k].y;
            __syncwarp();
        }
        // fixed-order sum over the 8 warps
        __shared__ double red[256 * 8];
#pragma unroll
        for (int k = 0; k < PPT; ++k) red[warp * L + lane + 32 * k] = acc[k];
        __syncthreads();
        for (int b = threadIdx.x; b < L; b += 256) {
            double t = 0.0;
            for (int q = 0; q < 8; ++q) t += red[q * L + b];
            dst[b] = t;
        }
    } else {
        constexpr int T = L / 16;
        float2* const bufs[1] = {psd_smem};
        const int t = threadIdx.x;
        const bool act = t < T;
        double acc[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k] = 0.0;
        for (int sg = s0; sg < s1; ++sg) {
            const float2* x = w + (long long)sg * hop;
            float2 v[1][16];
            if (act) {
#pragma unroll
                for (int k = 0; k < 16; ++k) v[0][k] = cscale(x[t + T * k], win[t + T * k]);
            }
            team_fft<L, T, 16, -1, 1, true>(v, bufs, tw, ts, t, act);
            if (act) {
#pragma unroll
                for (int k = 0; k < 16; ++k) acc[k] += (double)v[0][k].x * v[0][k].x + (double)v[0][k].y * v[0][k].y;
            }
            __syncthreads();
        }
        if (act) {
#pragma unroll
            for (int k = 0; k < 16; ++k) dst[t + T * k] = acc[k];
        }
    }
}

__global__ void psd_reduce_kernel(const double* __restrict__ part, int chunks, int L, int S, double scale,
                                  double* __restrict__ out) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= (long long)S * L) return;
    const long long u = idx / L, b = idx - u * L;
    double t = 0.0;
    for (int c = 0; c < chunks; ++c) t += part[(u * chunks + c) * L + b];
    out[idx] = t * scale;
}

}  // namespace

cudaError_t link_stats(const Plan& p, const float2* grid, long long stride, int S, uint64_t seed, long long unit0,
                       int bits, double* evm_num, double* evm_den, long long* errors, cudaStream_t st) {
    const long long per_unit = (long long)p.B * p.row_active;
    const int chunks = (int)((per_unit + kLinkChunk - 1) / kLinkChunk);
    Acc* host = new Acc[S];
    const cudaError_t e = reduce_to_host(
        S, chunks, st,
        [&](Acc* part) {
            link_stats_kernel<<<S * chunks, kLinkThreads, 0, st>>>(grid, stride, per_unit, seed, unit0, bits,
                                                                    chunks, part);
        },
        host);
    if (e == cudaSuccess)
        for (int u = 0; u < S; ++u) {
            evm_num[u] = host[u].a;
            evm_den[u] = host[u].b;
            errors[u] = host[u].e;
        }
    delete[] host;
    return e;
}

cudaError_t awgn(float2* wave, long long stride, long long len, int S, double sigma2, uint64_t seed,
                 long long unit0, cudaStream_t st) {
    const long long total = (long long)S * len;
    int grid = (int)std::min<long long>((total + 255) / 256, (long long)device_sms() * 16);
    if (grid < 1) grid = 1;
    awgn_kernel<<<grid, 256, 0, st>>>(wave, stride, len, S, sqrt(sigma2), seed, unit0);
    return cudaGetLastError();
}

cudaError_t wave_power(const float2* wave, long long stride, int S, long long begin, long long end, double* power,
                       cudaStream_t st) {
    const int chunks = (int)((end - begin + kLinkChunk - 1) / kLinkChunk);
    Acc* host = new Acc[S];
    const cudaError_t e = reduce_to_host(
        S, chunks, st,
        [&](Acc* part) { power_kernel<<<S * chunks, kLinkThreads, 0, st>>>(wave, stride, begin, end, chunks, part); },
        host);
    if (e == cudaSuccess)
        for (int u = 0; u < S; ++u) power[u] = host[u].a / (double)(end - begin);
    delete[] host;
    return e;
}

cudaError_t psd(const float2* wave, long long stride, long long len, int S, int L, double overlap, double* out_host,
                cudaStream_t st) {
    long hop = std::lround(L * (1.0 - overlap));
    if (hop < 1) hop = 1;
    const int n_seg = (int)((len - L) / hop + 1);
    const int chunks = (n_seg + kPsdSegPerCta - 1) / kPsdSegPerCta;
    std::vector<float> win(L);
    std::vector<float2> tw(L);
    double wpow = 0.0;
    for (int i = 0; i < L; ++i) {
        const double v = 0.5 - 0.5 * std::cos(2.0 * 3.14159265358979323846 * i / L);
        win[i] = (float)v;
        wpow += v * v;
        const double a = -2.0 * 3.14159265358979323846 * i / L;
        tw[i] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
    char* scratch = nullptr;
    const size_t part_b = sizeof(double) * (size_t)S * chunks * L, out_b = sizeof(double) * (size_t)S * L;
    const size_t tab_b = (sizeof(float) + sizeof(float2)) * L;
    cudaError_t e = scratch_alloc(&scratch, part_b + out_b + tab_b, st);
    if (e != cudaSuccess) return e;
    double* part = reinterpret_cast<double*>(scratch);
    double* dout = reinterpret_cast<double*>(scratch + part_b);
    float2* d_tw = reinterpret_cast<float2*>(scratch + part_b + out_b);
    float* d_win = reinterpret_cast<float*>(scratch + part_b + out_b + sizeof(float2) * L);
    e = cudaMemcpyAsync(d_win, win.data(), sizeof(float) * L, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_tw, tw.data(), sizeof(float2) * L, cudaMemcpyHostToDevice, st);
    const dim3 grid(chunks, S);
#define FCW_PSD_CASE(LL)                                                                                       \
    case LL: {                                                                                                 \
        const size_t smem = (LL <= 256 ? 8 : 1) * (size_t)(LL + LL / 16 + 2) * sizeof(float2);                 \
        if (smem > 48 * 1024) cudaFuncSetAttribute(psd_kernel<LL>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                                   (int)smem);                                                 \
        psd_kernel<LL><<<grid, 256, smem, st>>>(wave, stride, d_win, (int)hop, n_seg, d_tw, 1, part);          \
        break;                                                                                                 \
    }
    if (e == cudaSuccess) {
        switch (L) {
            FCW_PSD_CASE(64)
            FCW_PSD_CASE(128)
            FCW_PSD_CASE(256)
            FCW_PSD_CASE(512)
            FCW_PSD_CASE(1024)
            FCW_PSD_CASE(2048)
            FCW_PSD_CASE(4096)
            default: e = cudaErrorInvalidValue;
        }
#undef FCW_PSD_CASE
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
        const long long n = (long long)S * L;
        psd_reduce_kernel<<<(int)((n + 255) / 256), 256, 0, st>>>(part, chunks, L, S, 1.0 / ((double)n_seg * wpow),
                                                                 dout);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(out_host, dout, out_b, cudaMemcpyDeviceToHost, st);
    const cudaError_t f = cudaFreeAsync(scratch, st);
    if (e == cudaSuccess) e = f;
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e;
}

cudaError_t apply_channel(const float2* in, float2* out, long long stride, long long len, int S, const int* delays,
                          const float2* gains, int n_taps, cudaStream_t st) {
    // gains first: the float2 block must stay 8-byte aligned whatever S * n_taps is
    const size_t gbytes = sizeof(float2) * (size_t)S * n_taps;
    void* blk = nullptr;
    cudaError_t e = scratch_alloc(&blk, gbytes + sizeof(int) * (size_t)S * n_taps, st);
    if (e != cudaSuccess) return e;
    float2* g = static_cast<float2*>(blk);
    int* d = reinterpret_cast<int*>(static_cast<char*>(blk) + gbytes);
    e = cudaMemcpyAsync(d, delays, sizeof(int) * (size_t)S * n_taps, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(g, gains, sizeof(float2) * (size_t)S * n_taps, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        const int gx = (int)std::min<long long>((len + 255) / 256, 1184);
        channel_kernel<<<dim3(gx, S), 256, 0, st>>>(in, out, stride, len, d, g, n_taps);
        e = cudaGetLastError();
    }
    const cudaError_t f = cudaFreeAsync(blk, st);
    if (e == cudaSuccess) e = f;
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // host tap arrays may be released on return
    return e;
}

}  // namespace fcw
