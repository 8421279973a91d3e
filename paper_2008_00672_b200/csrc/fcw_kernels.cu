// sm_100a kernels of the symbol-synchronized FC-F-OFDM hot path.
//
//  K-TX  tx_kernel<N>: fused TX synthesis (replaces tx_discontinuous,
//        proj/src/fc_sync.cpp:114-143 and everything under it:
//        ofdm_modulate ofdm.cpp:97, cp_insert :108, zero_pad_symbol
//        fc_sync.cpp:34, tx_symbol :60, sfb_block_ola/synth_core
//        fc_core.cpp:115,76, combine_symbols fc_sync.cpp:96, subband sum :139).
//  K-RX  rx_kernel<N>: fused RX analysis for all subbands (replaces
//        rx_discontinuous fc_sync.cpp:245 with rx_segment :145, rx_block_freq
//        :178, rx_symbol_simplified :195 / rx_symbol_direct :158 +
//        afb_block_ols fc_core.cpp:144 + ofdm_demodulate ofdm.cpp:125).
//  K-GEN gen_qam_kernel: seeded QAM grid (channel.cpp:19-48,
//        scenario.cpp:110-128, ofdm.cpp:55-65).
//
// Work decomposition: one CTA (256 threads) owns a run of `chunk` consecutive
// OFDM symbols of one unit (antenna stream x frame) and walks them in order.
// Per symbol it builds the two N-bin block spectra of ALL subbands in SMEM
// (one shared N-point transform per block — the reference runs one per
// subband), transforms both blocks in lockstep, and overlap-adds in
// registers.  The tail of block 1 that overlaps the next symbol is carried in
// SMEM; the CTA recomputes the symbol just before its run to obtain the
// incoming carry, so every waveform sample is written exactly once by exactly
// one CTA (no atomics, no zero-fill pass, deterministic).
#include "fcw_fft.cuh"
#include "fcw_internal.hpp"

namespace fcw {

namespace {

constexpr int kPPT = 16;  // long-transform points per thread and block

FCW_DI float2 tw_conj(const float2* __restrict__ tw, int e) {
    const float2 w = __ldg(&tw[e]);
    return make_float2(w.x, -w.y);
}

// theta_n exponent: ((c mod N) * (S_n mod N)) mod N   (fc_sync.cpp:45-50)
template <int N>
FCW_DI int theta_exp(int cmodN, int smodN) {
    return (int)(((unsigned)cmodN * (unsigned)smodN) & (unsigned)(N - 1));
}

FCW_DI float2 zero2() { return make_float2(0.f, 0.f); }

// ---------------------------------------------------------------- K-TX parts

// Gather one grid column into the DFT-bin vector b -> value (0 off the active set).
FCW_DI float2 grid_bin(const KParams& P, const SubDev& sd, const float2* __restrict__ row, int b) {
    if (P.grid_full) return row[sd.full_off + b];
    const int a = __ldg(&P.inv[sd.full_off + b]);
    return a >= 0 ? row[sd.act_off + a] : zero2();
}

// Short-side TX of one subband-symbol by one thread (L <= 32).
template <int N, int L>
FCW_DI void tx_short_thread(const KParams& P, const SymDev& sy, const float2* __restrict__ row,
                            float2* spec0, float2* spec1, int gstart, int gcount) {
    for (int i = threadIdx.x; i < gcount; i += kThreads) {
        const int m = __ldg(&P.grp_sub[gstart + i]);
        const SubDev sd = P.sub[m];
        float2 x[L];
        const float2 ph = cscale(tw_conj(P.tw, theta_exp<N>(sd.cmodN, sy.smodN)), sd.tx_scale);
#pragma unroll
        for (int b = 0; b < L; ++b) x[b] = cmul(grid_bin(P, sd, row, b), ph);
        fft_reg<L, +1>(x);  // ofdm_modulate (scale folded into ph)
        const int lcp = sy.cp >> sd.logI;  // cp_truncate (fc_sync.cpp:26-32)
        float2 u0[L], u1[L];
#pragma unroll
        for (int k = 0; k < L; ++k) {
            // block 0: CP + first half through the reduced-overlap window a0;
            // block 1: second half through a1 (fc_sync.cpp:34-84)
            const bool in0 = (k >= L / 4 - lcp) && (k < 3 * L / 4);
            u0[k] = in0 ? x[(k - L / 4) & (L - 1)] : zero2();
            u1[k] = (k >= L / 4 && k < 3 * L / 4) ? x[(k + L / 4) & (L - 1)] : zero2();
        }
        fft_reg<L, -1>(u0);
        fft_reg<L, -1>(u1);
#pragma unroll
        for (int p0 = 0; p0 < L; ++p0) {
            const int b = (p0 + L / 2) & (L - 1);
            const int d = __ldg(&P.dest[sd.full_off + p0]);
            if (d >= 0) {
                const float w = __ldg(&P.win[sd.full_off + p0]);
                spec0[d] = cscale(u0[b], w);
                spec1[d] = cscale(u1[b], w * sd.bp1);
            }
        }
    }
}

// Short-side TX of one subband-symbol by one warp (L >= 64).
template <int N, int L>
FCW_DI void tx_short_warp(const KParams& P, const SymDev& sy, const float2* __restrict__ row,
                          float2* spec0, float2* spec1, float2* scr, int gstart, int gcount) {
    constexpr int PPT = L / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float2* s0 = scr;
    float2* s1 = scr + P.scratch_stride / 2;
    for (int i = warp; i < gcount; i += kWarps) {
        const int m = __ldg(&P.grp_sub[gstart + i]);
        const SubDev sd = P.sub[m];
        const float2 ph = cscale(tw_conj(P.tw, theta_exp<N>(sd.cmodN, sy.smodN)), sd.tx_scale);
        float2 v[1][PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) v[0][k] = cmul(grid_bin(P, sd, row, lane + 32 * k), ph);
        {
            float2* const b1[1] = {s0};
            team_fft<L, 32, PPT, +1, 1, false>(v, b1, P.tw, N / L, lane, true);
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < PPT; ++k) s0[lane + 32 * k] = v[0][k];
        __syncwarp();
        const int lcp = sy.cp >> sd.logI;
        float2 u[2][PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
            const int e = lane + 32 * k;
            const bool in0 = (e >= L / 4 - lcp) && (e < 3 * L / 4);
            const bool in1 = (e >= L / 4) && (e < 3 * L / 4);
            u[0][k] = in0 ? s0[(e - L / 4) & (L - 1)] : zero2();
            u[1][k] = in1 ? s0[(e + L / 4) & (L - 1)] : zero2();
        }
        {
            float2* const b2[2] = {s0, s1};
            team_fft<L, 32, PPT, -1, 2, false>(u, b2, P.tw, N / L, lane, true);
        }
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
            const int b = lane + 32 * k;
            const int p0 = (b + L / 2) & (L - 1);
            const int d = __ldg(&P.dest[sd.full_off + p0]);
            if (d >= 0) {
                const float w = __ldg(&P.win[sd.full_off + p0]);
                spec0[d] = cscale(u[0][k], w);
                spec1[d] = cscale(u[1][k], w * sd.bp1);
            }
        }
        __syncwarp();
    }
}

template <int N>
FCW_DI void tx_short_all(const KParams& P, const SymDev& sy, const float2* __restrict__ row,
                         float2* spec0, float2* spec1, float2* scr) {
    for (int g = 0; g < P.n_groups; ++g) {
        const int gs = P.grp_start[g], gc = P.grp_count[g];
        switch (P.grp_L[g]) {
#define FCW_TX_T(LL) \
    case LL:         \
        if constexpr (LL <= N) tx_short_thread<N, LL>(P, sy, row, spec0, spec1, gs, gc); break;
#define FCW_TX_W(LL) \
    case LL:         \
        if constexpr (LL <= N) tx_short_warp<N, LL>(P, sy, row, spec0, spec1, scr, gs, gc); break;
            FCW_TX_T(4) FCW_TX_T(8) FCW_TX_T(16) FCW_TX_T(32)
            FCW_TX_W(64) FCW_TX_W(128) FCW_TX_W(256) FCW_TX_W(512) FCW_TX_W(1024)
#undef FCW_TX_T
#undef FCW_TX_W
            default: break;
        }
    }
}

// ---------------------------------------------------------------- K-RX parts

template <int N, int L>
FCW_DI void rx_short_thread(const KParams& P, const SymDev& sy, const float2* spec0, const float2* spec1,
                            float2* __restrict__ orow, int gstart, int gcount) {
    for (int i = threadIdx.x; i < gcount; i += kThreads) {
        const int m = __ldg(&P.grp_sub[gstart + i]);
        const SubDev sd = P.sub[m];
        float2 g0[L], g1[L];
#pragma unroll
        for (int p0 = 0; p0 < L; ++p0) {
            // rx_block_freq (fc_sync.cpp:178-193) without the per-block phase,
            // which is applied once at the output (linearity)
            const int b = (p0 + L / 2) & (L - 1);
            const int q = (sd.c - L / 2 + p0) & (N - 1);
            const float w = __ldg(&P.win[sd.full_off + p0]);
            g0[b] = cscale(spec0[q], w);
            g1[b] = cscale(spec1[q], w * sd.bp1);
        }
        float2 x[L];
        if (P.fused) {
            // Eq. (30): t = Omega_{L/2} g1, f = Omega_{-L/4}(g0 - t), IDFT, S-hat,
            // DFT, Omega_{L/4}, + t, Omega_{-L/4}  (fc_sync.cpp:195-243)
            float2 t[L], f[L];
#pragma unroll
            for (int b = 0; b < L; ++b) {
                t[b] = (b & 1) ? make_float2(-g1[b].x, -g1[b].y) : g1[b];
                f[b] = csub(g0[b], t[b]);
            }
#pragma unroll
            for (int b = 0; b < L; ++b) {
                switch (b & 3) {
                    case 1: f[b] = mul_jpow<1>(f[b]); break;
                    case 2: f[b] = mul_jpow<2>(f[b]); break;
                    case 3: f[b] = mul_jpow<3>(f[b]); break;
                    default: break;
                }
            }
            fft_reg<L, +1>(f);
#pragma unroll
            for (int k = L / 2; k < L; ++k) f[k] = zero2();
            fft_reg<L, -1>(f);
            const float a = sd.rx_s0 / (float)L, s = sd.rx_s0;
#pragma unroll
            for (int b = 0; b < L; ++b) {
                float2 tj = t[b];
                switch (b & 3) {
                    case 1: tj = mul_jpow<1>(tj); break;
                    case 2: tj = mul_jpow<2>(tj); break;
                    case 3: tj = mul_jpow<3>(tj); break;
                    default: break;
                }
                x[b] = make_float2(fmaf(f[b].x, a, tj.x * s), fmaf(f[b].y, a, tj.y * s));
            }
        } else {
            // direct path: two OLS analysis blocks, central halves, OFDM DFT
            fft_reg<L, +1>(g0);
            fft_reg<L, +1>(g1);
#pragma unroll
            for (int k = 0; k < L / 2; ++k) {
                x[k] = g0[L / 4 + k];
                x[L / 2 + k] = g1[L / 4 + k];
            }
            fft_reg<L, -1>(x);
            const float a = sd.rx_s0 / (float)L;
#pragma unroll
            for (int b = 0; b < L; ++b) x[b] = cscale(x[b], a);
        }
        const float2 ph = __ldg(&P.tw[theta_exp<N>(sd.cmodN, sy.smodN)]);  // conj(theta_n)
#pragma unroll
        for (int b = 0; b < L; ++b) {
            const float2 val = cmul(x[b], ph);
            if (P.grid_full) {
                orow[sd.full_off + b] = val;
            } else {
                const int a = __ldg(&P.inv[sd.full_off + b]);
                if (a >= 0) orow[sd.act_off + a] = val;
            }
        }
    }
}

template <int N, int L>
FCW_DI void rx_short_warp(const KParams& P, const SymDev& sy, const float2* spec0, const float2* spec1,
                          float2* __restrict__ orow, float2* scr, int gstart, int gcount) {
    constexpr int PPT = L / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float2* s0 = scr;
    float2* s1 = scr + P.scratch_stride / 2;
    for (int i = warp; i < gcount; i += kWarps) {
        const int m = __ldg(&P.grp_sub[gstart + i]);
        const SubDev sd = P.sub[m];
        float2 g[2][PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
            const int b = lane + 32 * k;
            const int p0 = (b + L / 2) & (L - 1);
            const int q = (sd.c - L / 2 + p0) & (N - 1);
            const float w = __ldg(&P.win[sd.full_off + p0]);
            g[0][k] = cscale(spec0[q], w);
            g[1][k] = cscale(spec1[q], w * sd.bp1);
        }
        float2 x[1][PPT];
        if (P.fused) {
            const bool odd = lane & 1;
            float2 t[PPT];
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                t[k] = odd ? make_float2(-g[1][k].x, -g[1][k].y) : g[1][k];
                x[0][k] = mul_jpow_rt(csub(g[0][k], t[k]), lane);
            }
            float2* const b1[1] = {s0};
            team_fft<L, 32, PPT, +1, 1, false>(x, b1, P.tw, N / L, lane, true);
#pragma unroll
            for (int k = PPT / 2; k < PPT; ++k) x[0][k] = zero2();
            team_fft<L, 32, PPT, -1, 1, false>(x, b1, P.tw, N / L, lane, true);
            const float a = sd.rx_s0 / (float)L, s = sd.rx_s0;
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                const float2 tj = mul_jpow_rt(t[k], lane);
                x[0][k] = make_float2(fmaf(x[0][k].x, a, tj.x * s), fmaf(x[0][k].y, a, tj.y * s));
            }
        } else {
            float2* const b2[2] = {s0, s1};
            team_fft<L, 32, PPT, +1, 2, false>(g, b2, P.tw, N / L, lane, true);
            __syncwarp();
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                s0[lane + 32 * k] = g[0][k];
                s1[lane + 32 * k] = g[1][k];
            }
            __syncwarp();
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                const int e = lane + 32 * k;
                x[0][k] = (k < PPT / 2) ? s0[L / 4 + e] : s1[L / 4 + e - L / 2];
            }
            float2* const b1[1] = {s0};
            team_fft<L, 32, PPT, -1, 1, false>(x, b1, P.tw, N / L, lane, true);
            const float a = sd.rx_s0 / (float)L;
#pragma unroll
            for (int k = 0; k < PPT; ++k) x[0][k] = cscale(x[0][k], a);
        }
        const float2 ph = __ldg(&P.tw[theta_exp<N>(sd.cmodN, sy.smodN)]);
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
            const int b = lane + 32 * k;
            const float2 val = cmul(x[0][k], ph);
            if (P.grid_full) {
                orow[sd.full_off + b] = val;
            } else {
                const int a = __ldg(&P.inv[sd.full_off + b]);
                if (a >= 0) orow[sd.act_off + a] = val;
            }
        }
        __syncwarp();
    }
}

template <int N>
FCW_DI void rx_short_all(const KParams& P, const SymDev& sy, const float2* spec0, const float2* spec1,
                         float2* orow, float2* scr) {
    for (int g = 0; g < P.n_groups; ++g) {
        const int gs = P.grp_start[g], gc = P.grp_count[g];
        switch (P.grp_L[g]) {
#define FCW_RX_T(LL) \
    case LL:         \
        if constexpr (LL <= N) rx_short_thread<N, LL>(P, sy, spec0, spec1, orow, gs, gc); break;
#define FCW_RX_W(LL) \
    case LL:         \
        if constexpr (LL <= N) rx_short_warp<N, LL>(P, sy, spec0, spec1, orow, scr, gs, gc); break;
            FCW_RX_T(4) FCW_RX_T(8) FCW_RX_T(16) FCW_RX_T(32)
            FCW_RX_W(64) FCW_RX_W(128) FCW_RX_W(256) FCW_RX_W(512) FCW_RX_W(1024)
#undef FCW_RX_T
#undef FCW_RX_W
            default: break;
        }
    }
}

}  // namespace

// ------------------------------------------------------------------ kernels

template <int N>
__global__ void __launch_bounds__(kThreads) tx_kernel(const KParams P) {
    extern __shared__ float4 smem_raw[];
    float2* sm = reinterpret_cast<float2*>(smem_raw);
    float2* spec0 = sm;
    float2* spec1 = sm + P.spec_stride;
    float2* carry = spec1 + P.spec_stride;
    float2* scr = carry + N / 2 + (threadIdx.x >> 5) * P.scratch_stride;
    constexpr int T = N / kPPT;
    const int tid = threadIdx.x;
    const bool act = tid < T;
    const int unit = blockIdx.x / P.nchunks;
    const int n0 = (blockIdx.x % P.nchunks) * P.chunk;
    const int n1 = min(P.B, n0 + P.chunk);
    const float2* in_u = P.in + (long long)unit * P.in_stride;
    float2* out_u = P.out + (long long)unit * P.out_stride;

    for (int n = n0 > 0 ? n0 - 1 : 0; n < n1; ++n) {
        const SymDev sy = P.sym[n];
        __syncthreads();  // previous symbol's transform no longer reads spec
        tx_short_all<N>(P, sy, in_u + (long long)n * P.row_len, spec0, spec1, scr);
        __syncthreads();
        // secondary contributions of shared transition bins, in rank order
        for (int l = 0; l < P.n_lvl; ++l) {
            for (int k = P.lvl_start[l] + tid; k < P.lvl_start[l + 1]; k += kThreads) {
                const int q = __ldg(&P.fix_tgt[k]);
                spec0[q] = cadd(spec0[q], spec0[N + k]);
                spec1[q] = cadd(spec1[q], spec1[N + k]);
            }
            __syncthreads();
        }
        for (int k = tid; k < P.n_zero; k += kThreads) {
            const int q = __ldg(&P.zero_list[k]);
            spec0[q] = zero2();
            spec1[q] = zero2();
        }
        __syncthreads();

        float2 cr[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int u = tid + T * m;
            cr[m] = (act && u < sy.carry_len) ? carry[u] : zero2();
        }
        float2 v[2][kPPT];
        if (act) {
#pragma unroll
            for (int m = 0; m < kPPT; ++m) {
                v[0][m] = spec0[tid + T * m];
                v[1][m] = spec1[tid + T * m];
            }
        }
        {
            float2* const bufs[2] = {spec0, spec1};
            team_fft<N, T, kPPT, +1, 2, true>(v, bufs, P.tw, 1, tid, act);
        }
        // symbol-wise overlap-add: block 0 at 0, block 1 at N/2, carry from n-1
        if (act) {
            const bool emit = n >= n0;
            float2* dst = out_u + sy.sigma;
#pragma unroll
            for (int mm = 0; mm < 24; ++mm) {
                const int u = tid + T * mm;
                float2 val = zero2();
                if (mm < 16) val = v[0][mm];
                if (mm >= 8) val = cadd(val, v[1][mm - 8]);
                if (mm < 8) val = cadd(val, cr[mm]);
                if (u < sy.own_len) {
                    if (emit) dst[u] = val;
                } else {
                    carry[u - sy.own_len] = val;
                }
            }
        }
    }
}

template <int N>
__global__ void __launch_bounds__(kThreads) rx_kernel(const KParams P) {
    extern __shared__ float4 smem_raw[];
    float2* sm = reinterpret_cast<float2*>(smem_raw);
    float2* spec0 = sm;
    float2* spec1 = sm + P.spec_stride;
    float2* scr = spec1 + P.spec_stride + (threadIdx.x >> 5) * P.scratch_stride;
    constexpr int T = N / kPPT;
    const int tid = threadIdx.x;
    const bool act = tid < T;
    const int unit = blockIdx.x / P.nchunks;
    const int n0 = (blockIdx.x % P.nchunks) * P.chunk;
    const int n1 = min(P.B, n0 + P.chunk);
    const float2* in_u = P.in + (long long)unit * P.in_stride;
    float2* out_u = P.out + (long long)unit * P.out_stride;

    for (int n = n0; n < n1; ++n) {
        const SymDev sy = P.sym[n];
        __syncthreads();  // previous symbol's subband stage no longer reads spec
        float2 v[2][kPPT];
        if (act) {
            // rx_segment (fc_sync.cpp:145-156): y0 = w[start, +N), y1 = w[start + N/2, +N)
            const float2* src = in_u + P.rx_base + sy.sigma + tid;
#pragma unroll
            for (int mm = 0; mm < 24; ++mm) {
                const float2 val = __ldg(&src[T * mm]);
                if (mm < 16) v[0][mm] = val;
                if (mm >= 8) v[1][mm - 8] = val;
            }
        }
        {
            float2* const bufs[2] = {spec0, spec1};
            team_fft<N, T, kPPT, -1, 2, true>(v, bufs, P.tw, 1, tid, act);
        }
        __syncthreads();
        if (act) {
#pragma unroll
            for (int m = 0; m < kPPT; ++m) {
                spec0[tid + T * m] = v[0][m];
                spec1[tid + T * m] = v[1][m];
            }
        }
        __syncthreads();
        rx_short_all<N>(P, sy, spec0, spec1, out_u + (long long)n * P.row_len, scr);
    }
}

// K-GEN: one thread per QAM symbol; splitmix64 is counter-based, so draw j of
// unit u is mix(seed_u + (j+1) * gamma) and every bit is independent.
__global__ void gen_qam_kernel(uint64_t seed, long long unit0, int S, long long per_unit, int bits,
                               float2* __restrict__ out) {
    const long long total = (long long)S * per_unit;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long u = idx / per_unit, i = idx - u * per_unit;
        uint64_t s = seed ^ (0x9e3779b97f4a7c15ULL * (uint64_t)(unit0 + u + 1));  // derive_seed
        s += 0x9e3779b97f4a7c15ULL;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        uint64_t st = z ^ (z >> 31);
        if (st == 0) st = 0x1234567890abcdefULL;  // GaussianRng ctor (channel.cpp:26)
        unsigned sym = 0;
        const uint64_t base = st + (uint64_t)(i * bits) * 0x9e3779b97f4a7c15ULL;
        for (int b = 0; b < bits; ++b) {
            uint64_t x = base + (uint64_t)(b + 1) * 0x9e3779b97f4a7c15ULL;
            x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
            x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
            x ^= x >> 31;
            sym |= (unsigned)(x & 1u) << b;
        }
        const int k = bits / 2, levels = 1 << k;
        const unsigned mask = (1u << k) - 1u;
        unsigned gi = sym & mask, gq = (sym >> k) & mask, li = 0, lq = 0;
        for (; gi; gi >>= 1) li ^= gi;
        for (; gq; gq >>= 1) lq ^= gq;
        const double sc = 1.0 / sqrt(2.0 * ((double)levels * levels - 1.0) / 3.0);
        out[idx] = make_float2((float)(sc * (2.0 * li + 1 - levels)), (float)(sc * (2.0 * lq + 1 - levels)));
    }
}

// ----------------------------------------------------------------- launchers

namespace {

size_t common_smem(const Plan& p, int with_carry) {
    const int spec_stride = p.N + (p.n_ext > p.N / 16 ? p.n_ext : p.N / 16) + 2;
    const int scr = p.Lmax >= 64 ? 2 * (p.Lmax + p.Lmax / 16 + 2) : 0;
    size_t f2 = 2 * (size_t)((spec_stride + 1) & ~1) + (with_carry ? p.N / 2 : 0) + (size_t)kWarps * scr;
    return f2 * sizeof(float2);
}

template <class K>
cudaError_t launch_one(K kernel, size_t smem, int grid, const KParams& kp, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kernel<<<grid, kThreads, smem, st>>>(kp);
    return cudaGetLastError();
}

}  // namespace

void fill_common(const Plan& p, KParams& kp) {
    kp.N = p.N;
    kp.B = p.B;
    kp.M = p.M;
    kp.spec_stride = (p.N + (p.n_ext > p.N / 16 ? p.n_ext : p.N / 16) + 2 + 1) & ~1;
    kp.scratch_stride = p.Lmax >= 64 ? 2 * (p.Lmax + p.Lmax / 16 + 2) : 0;
    kp.n_ext = p.n_ext;
    kp.n_zero = (int)p.h_zero.size();
    kp.n_lvl = p.n_lvl;
    for (int i = 0; i <= kMaxLevels; ++i) kp.lvl_start[i] = i < (int)p.lvl_start.size() ? p.lvl_start[i] : p.n_ext;
    kp.n_groups = p.n_groups;
    for (int g = 0; g < kMaxGroups; ++g) {
        kp.grp_L[g] = p.grp_L[g];
        kp.grp_start[g] = p.grp_start[g];
        kp.grp_count[g] = p.grp_count[g];
    }
    kp.Q = p.Q;
    kp.sub = p.d_sub;
    kp.sym = p.d_sym;
    kp.win = p.d_win;
    kp.inv = p.d_inv;
    kp.dest = p.d_dest;
    kp.grp_sub = p.d_grp_sub;
    kp.fix_tgt = p.d_fix;
    kp.zero_list = p.d_zero;
    kp.tw = p.d_tw;
}

size_t tx_smem_bytes(const Plan& p) { return common_smem(p, 1); }
size_t rx_smem_bytes(const Plan& p) { return common_smem(p, 0); }

cudaError_t launch_tx(const Plan& p, KParams& kp, int S, cudaStream_t st) {
    const size_t smem = tx_smem_bytes(p);
    const int grid = S * kp.nchunks;
    switch (p.N) {
#define FCW_L(NN) \
    case NN: return launch_one(tx_kernel<NN>, smem, grid, kp, st);
        FCW_L(16) FCW_L(32) FCW_L(64) FCW_L(128) FCW_L(256) FCW_L(512) FCW_L(1024) FCW_L(2048) FCW_L(4096)
#undef FCW_L
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_rx(const Plan& p, KParams& kp, int S, cudaStream_t st) {
    const size_t smem = rx_smem_bytes(p);
    const int grid = S * kp.nchunks;
    switch (p.N) {
#define FCW_L(NN) \
    case NN: return launch_one(rx_kernel<NN>, smem, grid, kp, st);
        FCW_L(16) FCW_L(32) FCW_L(64) FCW_L(128) FCW_L(256) FCW_L(512) FCW_L(1024) FCW_L(2048) FCW_L(4096)
#undef FCW_L
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_gen_qam(const Plan& p, uint64_t seed, long long unit0, int S, int bits, float2* out,
                           cudaStream_t st) {
    const long long per_unit = (long long)p.B * p.row_active;
    const long long total = per_unit * S;
    int grid = (int)((total + 255) / 256);
    if (grid > 148 * 64) grid = 148 * 64;
    if (grid < 1) grid = 1;
    gen_qam_kernel<<<grid, 256, 0, st>>>(seed, unit0, S, per_unit, bits, out);
    return cudaGetLastError();
}

}  // namespace fcw
