// Continuous (non-symbol-synchronized) FC filterbank, SURVEY.md §8 row f2:
// tx_continuous / rx_continuous (proj/src/fc_core.cpp:155-223).
//
// The continuous filterbank hops blocks by N_S = N/2 on the high-rate side
// and L_S = L/2 on the low-rate side, so block pairs (2n, 2n+1) sit exactly
// where the symbol-synchronized path puts the two blocks of an OFDM symbol
// with no cyclic prefix: block 2n at n N and block 2n+1 at n N + N/2, each
// windowed on [L_L, L_L + L_S) (first_block_analysis_window with l_cp = 0 is
// the plain analysis window), with block_phase(2n) = 1 and block_phase(2n+1)
// = block_phase(1) at overlap 1/2.  So:
//   TX:  the L samples a block pair carries, x = stream[2n L_S - L_T, + L),
//        enter the fused TX kernel as the "OFDM symbol" whose IDFT is x:
//        column X = DFT_L(x) / sqrt(L) of a cp = 0 plan (cont_pre_kernel),
//        then fcw_tx with the full-grid layout.
//   RX:  fcw_rx (direct path, cp = 0, full grid) computes per pair
//        DFT_L([sqrt(I) z_2n[L_L..], sqrt(I) z_2n+1[L_L..]]) / sqrt(L); its
//        inverse (cont_post_kernel) is exactly the rx_continuous output
//        out[R L_S + u] = sqrt(I) z_R[L_L + u] for R = 2n, 2n+1.
// The waveform is zero-extended by N_L in front for RX, as rx_continuous
// does (fc_core.cpp:207-208).
// The column passes cancel against the kernels' own short IDFT (TX) / OFDM
// DFT (RX), so by default the kernels run with time-domain I/O instead
// (KParams.td, fcw::tx_time_domain / rx_time_domain): no column passes, no
// grid round trip, no RX staging copy (RX reads the waveform with zeros
// outside it).  FCW_CONT_COLUMNS=1 keeps the column passes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "fcw_fft.cuh"
#include "fcw_internal.hpp"

struct fcw_cont_plan {
    int N = 0, M = 0, Lmax = 0;
    double overlap = 0.5;
    fcw_plan* tx = nullptr;  // cp = 0, B_tx symbols
    fcw_plan* rx = nullptr;  // cp = 0, B_rx symbols
    int B_tx = 0, B_rx = 0;
    int64_t tx_len = 0, tx_Q = 0, useful0 = 0;
    int64_t rx_wave_len = 0, rx_pad_len = 0, rx_out_total = 0, stream_total = 0;
    std::vector<int> L, c, full_off, R_tx, R_rx;
    std::vector<int64_t> len, stream_off, out_off;
    std::vector<fcw::fc_col> h_cols;
    fcw::fc_col* d_cols = nullptr;  // per-subband column descriptors
    float2* d_tw = nullptr;         // exp(-2 pi i k / Lmax)
    int row_full = 0;
    // time-domain I/O of the fused kernels (no column passes, no grid round
    // trip, no RX staging copy).  FCW_CONT_COLUMNS=1 forces the column
    // passes.
    bool td_tx = false, td_rx = false;
};

namespace fcw {
namespace {

// One column = (unit u, symbol n, subband m); blockIdx.y = unit.
// Warp per column for L >= 64 (team FFT through a per-warp SMEM buffer),
// thread per column for L <= 32 (register FFT).
template <int L, bool PRE>
__global__ void __launch_bounds__(256) cont_cols_kernel(const fc_col* __restrict__ cols, int n_sub_in_group,
                                                        const int* __restrict__ group, int B,
                                                        const float2* __restrict__ tw, int tw_stride,
                                                        const float2* __restrict__ in, long long in_stride,
                                                        float2* __restrict__ out, long long out_stride) {
    const long long u = blockIdx.y;
    const long long ncols = (long long)B * n_sub_in_group;
    const float sc = rsqrtf((float)L);
    if constexpr (L <= 32) {
        for (long long col = blockIdx.x * (long long)blockDim.x + threadIdx.x; col < ncols;
             col += (long long)gridDim.x * blockDim.x) {
            const int n = (int)(col / n_sub_in_group);
            const fc_col d = cols[group[col - (long long)n * n_sub_in_group]];
            float2 v[L];
            if constexpr (PRE) {
                const float2* s = in + u * in_stride + d.in_off;
                const long long base = 2LL * n * (L / 2) - d.lt;
#pragma unroll
                for (int i = 0; i < L; ++i) {
                    const long long j = base + i;
                    v[i] = (j >= 0 && j < d.len) ? s[j] : make_float2(0.f, 0.f);
                }
                fft_reg<L, -1>(v);
                float2* g = out + u * out_stride + (long long)n * d.row + d.full_off;
#pragma unroll
                for (int i = 0; i < L; ++i) g[i] = cscale(v[i], sc);
            } else {
                const float2* g = in + u * in_stride + (long long)n * d.row + d.full_off;
#pragma unroll
                for (int i = 0; i < L; ++i) v[i] = g[i];
                fft_reg<L, +1>(v);
                float2* o = out + u * out_stride + d.out_off;
                const long long base = 2LL * n * (L / 2);
#pragma unroll
                for (int i = 0; i < L; ++i)
                    if (base + i < d.len_out) o[base + i] = cscale(v[i], sc);
            }
        }
    } else {
        constexpr int PPT = L / 32;
        extern __shared__ float2 cont_smem[];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        float2* buf = cont_smem + warp * (L + L / 16 + 2);
        float2* const bufs[1] = {buf};
        const long long wpb = blockDim.x / 32;
        for (long long col = blockIdx.x * wpb + warp; col < ncols; col += (long long)gridDim.x * wpb) {
            const int n = (int)(col / n_sub_in_group);
            const fc_col d = cols[group[col - (long long)n * n_sub_in_group]];
            float2 v[1][PPT];
            if constexpr (PRE) {
                const float2* s = in + u * in_stride + d.in_off;
                const long long base = 2LL * n * (L / 2) - d.lt;
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    const long long j = base + lane + 32 * k;
                    v[0][k] = (j >= 0 && j < d.len) ? s[j] : make_float2(0.f, 0.f);
                }
                team_fft<L, 32, PPT, -1, 1, false>(v, bufs, tw, tw_stride, lane, true);
                float2* g = out + u * out_stride + (long long)n * d.row + d.full_off + lane;
#pragma unroll
                for (int k = 0; k < PPT; ++k) g[32 * k] = cscale(v[0][k], sc);
            } else {
                const float2* g = in + u * in_stride + (long long)n * d.row + d.full_off + lane;
#pragma unroll
                for (int k = 0; k < PPT; ++k) v[0][k] = g[32 * k];
                team_fft<L, 32, PPT, +1, 1, false>(v, bufs, tw, tw_stride, lane, true);
                float2* o = out + u * out_stride + d.out_off;
                const long long base = 2LL * n * (L / 2);
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    const long long i = base + lane + 32 * k;
                    if (i < d.len_out) o[i] = cscale(v[0][k], sc);
                }
            }
            __syncwarp();
        }
    }
}

template <bool PRE>
cudaError_t launch_cols_L(int L, const fc_col* cols, int nsub, const int* group, int B, const float2* tw, int Lmax,
                          const float2* in, long long in_stride, float2* out, long long out_stride, int S,
                          cudaStream_t st) {
    const long long ncols = (long long)B * nsub;
    const int per_cta = L <= 32 ? 256 : 8;
    const int grid_x = (int)std::max(1LL, std::min((ncols + per_cta - 1) / per_cta, 4096LL));
    const size_t smem = L <= 32 ? 0 : (size_t)8 * (L + L / 16 + 2) * sizeof(float2);
    const dim3 grid(grid_x, S);
#define FCW_CONT_CASE(LL)                                                                                       \
    case LL: {                                                                                                  \
        auto k = cont_cols_kernel<LL, PRE>;                                                                     \
        if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        k<<<grid, 256, smem, st>>>(cols, nsub, group, B, tw, Lmax / LL, in, in_stride, out, out_stride);      \
        break;                                                                                                  \
    }
    switch (L) {
        FCW_CONT_CASE(4)
        FCW_CONT_CASE(8)
        FCW_CONT_CASE(16)
        FCW_CONT_CASE(32)
        FCW_CONT_CASE(64)
        FCW_CONT_CASE(128)
        FCW_CONT_CASE(256)
        FCW_CONT_CASE(512)
        FCW_CONT_CASE(1024)
        default: return cudaErrorInvalidValue;
    }
#undef FCW_CONT_CASE
    return cudaGetLastError();
}

}  // namespace

// Pre (TX) / post (RX) column transforms over every subband, grouped by L.
cudaError_t cont_columns(const fcw_cont_plan& p, bool pre, const float2* in, long long in_stride, float2* out,
                         long long out_stride, int S, int B, cudaStream_t st) {
    std::vector<int> Ls = p.L;
    std::sort(Ls.begin(), Ls.end());
    Ls.erase(std::unique(Ls.begin(), Ls.end()), Ls.end());
    int start = 0;
    for (int L : Ls) {
        int cnt = 0;
        for (int m = 0; m < p.M; ++m) cnt += p.L[m] == L;
        const int* group = reinterpret_cast<const int*>(p.d_cols + p.M) + start;
        const cudaError_t e =
            pre ? launch_cols_L<true>(L, p.d_cols, cnt, group, B, p.d_tw, p.Lmax, in, in_stride, out, out_stride, S, st)
                : launch_cols_L<false>(L, p.d_cols, cnt, group, B, p.d_tw, p.Lmax, in, in_stride, out, out_stride, S,
                                       st);
        if (e != cudaSuccess) return e;
        start += cnt;
    }
    return cudaSuccess;
}

}  // namespace fcw

// ------------------------------------------------------------------ C ABI
namespace {

int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace

extern "C" {

int fcw_cont_plan_create(fcw_cont_plan** out, int N, double overlap, const fcw_subband* sbs, int M,
                         const int64_t* stream_len, int64_t rx_wave_len, int l_cp0) {
    using fcw::set_error;
    if (!out) return set_error(FCW_EINVAL, "null plan pointer");
    *out = nullptr;
    if (M < 1 || !sbs) return set_error(FCW_EINVAL, "one config per subband signal required");  // fc_core.cpp:166
    if (!stream_len) return set_error(FCW_EINVAL, "stream lengths required");
    auto* p = new (std::nothrow) fcw_cont_plan();
    if (!p) return set_error(FCW_ENOMEM, "host allocation failed");
    p->N = N;
    p->M = M;
    p->overlap = overlap;
    std::vector<fcw_fc_params> prm(M);
    int B_tx = 1, B_rx = 1;
    int64_t tx_len = 0, rx_total = 0, soff = 0;
    for (int m = 0; m < M; ++m) {
        int rc = fcw_derive_fc_params(N, sbs[m].L, overlap, &prm[m]);
        if (rc != FCW_OK) {
            delete p;
            return rc;
        }
        if (stream_len[m] < 0) {
            delete p;
            return set_error(FCW_EINVAL, "negative stream length");
        }
        const fcw_fc_params& q = prm[m];
        // continuous_block_count (fc_core.cpp:155-161)
        const int R_tx = ceil_div(stream_len[m] + q.L_O - q.L_L, q.L_S);
        tx_len = std::max<int64_t>(tx_len, (int64_t)(R_tx - 1) * q.N_S + q.N);
        // rx_continuous block count (fc_core.cpp:202-205)
        if (rx_wave_len < N) {
            delete p;
            return set_error(FCW_EINVAL, "waveform shorter than one FC block");  // fc_core.cpp:201
        }
        const int64_t nlow = (rx_wave_len + q.I - 1) / q.I + q.L;
        const int R_rx = ceil_div(nlow, q.L_S);
        B_tx = std::max(B_tx, (R_tx + 1) / 2);
        B_rx = std::max(B_rx, (R_rx + 1) / 2);
        p->L.push_back(sbs[m].L);
        p->c.push_back(sbs[m].c);
        p->R_tx.push_back(R_tx);
        p->R_rx.push_back(R_rx);
        p->len.push_back(stream_len[m]);
        p->stream_off.push_back(soff);
        p->out_off.push_back(rx_total);
        soff += stream_len[m];
        rx_total += (int64_t)R_rx * q.L_S;
        p->Lmax = std::max(p->Lmax, sbs[m].L);
    }
    p->tx_len = tx_len;
    p->stream_total = soff;
    p->rx_out_total = rx_total;
    p->rx_wave_len = rx_wave_len;
    p->B_tx = B_tx;
    p->B_rx = B_rx;
    p->useful0 = (int64_t)std::llround(overlap * N) + (int64_t)prm[0].I * l_cp0;  // fc_core.cpp:192-196
    // the two cp = 0 symbol plans with every DFT bin in the (full) grid
    std::vector<std::vector<int>> bins(M);
    std::vector<fcw_subband> d(M);
    for (int m = 0; m < M; ++m) {
        bins[m].resize(sbs[m].L);
        for (int b = 0; b < sbs[m].L; ++b) bins[m][b] = b;
        d[m] = sbs[m];
        d[m].l_ofdm = sbs[m].L;
        d[m].n_active = sbs[m].L;
        d[m].active_bins = bins[m].data();
    }
    std::vector<int> cp_tx(B_tx, 0), cp_rx(B_rx, 0);
    int rc = fcw_plan_create(&p->tx, N, overlap, cp_tx.data(), B_tx, d.data(), M, 0);
    if (rc == FCW_OK) rc = fcw_plan_create(&p->rx, N, overlap, cp_rx.data(), B_rx, d.data(), M, 0);
    if (rc != FCW_OK) {
        fcw_cont_plan_destroy(p);
        return rc;
    }
    fcw_plan_info ti{}, ri{};
    fcw_plan_get_info(p->tx, &ti);
    fcw_plan_get_info(p->rx, &ri);
    p->tx_Q = ti.Q;
    p->row_full = ti.row_full;
    // RX input: N_L zeros, the waveform, zeros up to the last block pair
    p->rx_pad_len = std::max<int64_t>(ri.Q, prm[0].N_L + rx_wave_len);
    {
        const char* e = std::getenv("FCW_CONT_COLUMNS");
        const bool cols = e && std::atoi(e) != 0;
        bool uni = true, big = false;
        for (int m = 0; m < M; ++m) {
            uni = uni && sbs[m].L == sbs[0].L;
            big = big || sbs[m].L >= 512;
        }
        p->td_tx = !cols;
        p->td_rx = !cols;
        // the TX thread (L <= 32) and warp (L >= 512) paths carry the
        // time-domain input in the generic kernels only (tx_short_one)
        if (p->td_tx && (big || (uni && sbs[0].L <= 32))) fcw::plan_force_generic(p->tx);
        // the zv / nb kernel variants carry no time-domain I/O (nor the
        // bounded window load that replaces rx_continuous's zero padding)
        if (p->td_tx) fcw::plan_clear_special(p->tx);
        if (p->td_rx) fcw::plan_clear_special(p->rx);
    }
    int off = 0;
    for (int m = 0; m < M; ++m) {
        fcw::fc_col c{};
        c.in_off = p->stream_off[m];
        c.len = p->len[m];
        c.out_off = p->out_off[m];
        c.len_out = (long long)p->R_rx[m] * prm[m].L_S;
        c.lt = prm[m].L_T;
        c.row = ti.row_full;
        c.full_off = off;
        off += sbs[m].L;
        p->h_cols.push_back(c);
        p->full_off.push_back(c.full_off);
    }
    // columns, then subband ids grouped by ascending L (fcw::cont_columns)
    std::vector<int> group;
    std::vector<int> Ls = p->L;
    std::sort(Ls.begin(), Ls.end());
    Ls.erase(std::unique(Ls.begin(), Ls.end()), Ls.end());
    for (int L : Ls)
        for (int m = 0; m < M; ++m)
            if (p->L[m] == L) group.push_back(m);
    const size_t cb = sizeof(fcw::fc_col) * M, gb = sizeof(int) * M;
    std::vector<float2> tw(p->Lmax);
    for (int k = 0; k < p->Lmax; ++k) {
        const double a = -2.0 * 3.14159265358979323846 * k / p->Lmax;
        tw[k] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&p->d_cols), cb + gb);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&p->d_tw), sizeof(float2) * p->Lmax);
    if (e == cudaSuccess) e = cudaMemcpy(p->d_cols, p->h_cols.data(), cb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(reinterpret_cast<char*>(p->d_cols) + cb, group.data(), gb, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(p->d_tw, tw.data(), sizeof(float2) * p->Lmax, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        fcw_cont_plan_destroy(p);
        return fcw::set_cuda_error(e, "continuous plan tables");
    }
    *out = p;
    return FCW_OK;
}

void fcw_cont_plan_destroy(fcw_cont_plan* p) {
    if (!p) return;
    if (p->tx) fcw_plan_destroy(p->tx);
    if (p->rx) fcw_plan_destroy(p->rx);
    if (p->d_cols) cudaFree(p->d_cols);
    if (p->d_tw) cudaFree(p->d_tw);
    delete p;
}

int fcw_cont_plan_get_info(const fcw_cont_plan* p, fcw_cont_info* info, int64_t* rx_out_len, int64_t* rx_out_off) {
    if (!p || !info) return fcw::set_error(FCW_EINVAL, "null argument");
    info->N = p->N;
    info->M = p->M;
    info->tx_len = p->tx_len;
    info->tx_stride = p->tx_Q;
    info->useful0 = p->useful0;
    info->stream_total = p->stream_total;
    info->rx_wave_len = p->rx_wave_len;
    info->rx_out_total = p->rx_out_total;
    info->tx_pairs = p->B_tx;
    info->rx_pairs = p->B_rx;
    for (int m = 0; m < p->M; ++m) {
        if (rx_out_len) rx_out_len[m] = p->h_cols[m].len_out;
        if (rx_out_off) rx_out_off[m] = p->h_cols[m].out_off;
    }
    return FCW_OK;
}

int fcw_tx_continuous(const fcw_cont_plan* p, const void* streams, void* wave, int S, void* stream) {
    if (!p) return fcw::set_error(FCW_EINVAL, "null plan");
    if (S < 0) return fcw::set_error(FCW_EINVAL, "negative unit count");
    if (S == 0) return FCW_OK;
    if (!streams || !wave) return fcw::set_error(FCW_EINVAL, "null buffer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (p->td_tx)
        return fcw::tx_time_domain(p->tx, p->d_cols, static_cast<const float2*>(streams), p->stream_total,
                                   static_cast<float2*>(wave), p->tx_Q, S, st);
    const long long grid_stride = (long long)p->B_tx * p->row_full;
    float2* grid = nullptr;
    cudaError_t e = fcw::scratch_alloc(&grid, sizeof(float2) * grid_stride * S, st);
    if (e != cudaSuccess) return fcw::set_cuda_error(e, "continuous TX scratch");
    int rc = FCW_OK;
    for (int u0 = 0; u0 < S && rc == FCW_OK; u0 += 65535) {
        const int s = std::min(S - u0, 65535);
        e = fcw::cont_columns(*p, true, static_cast<const float2*>(streams) + (long long)u0 * p->stream_total,
                              p->stream_total, grid + (long long)u0 * grid_stride, grid_stride, s, p->B_tx, st);
        if (e != cudaSuccess) rc = fcw::set_cuda_error(e, "continuous TX columns");
    }
    if (rc == FCW_OK)
        rc = fcw_tx(p->tx, grid, grid_stride, wave, p->tx_Q, S, FCW_GRID_FULL, stream);
    e = cudaFreeAsync(grid, st);
    if (rc == FCW_OK && e != cudaSuccess) rc = fcw::set_cuda_error(e, "continuous TX scratch free");
    return rc;
}

int fcw_rx_continuous(const fcw_cont_plan* p, const void* wave, void* out, int S, void* stream) {
    if (!p) return fcw::set_error(FCW_EINVAL, "null plan");
    if (S < 0) return fcw::set_error(FCW_EINVAL, "negative unit count");
    if (S == 0) return FCW_OK;
    if (!wave || !out) return fcw::set_error(FCW_EINVAL, "null buffer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    fcw_plan_info ri{};
    fcw_plan_get_info(p->rx, &ri);
    if (p->td_rx)
        return fcw::rx_time_domain(p->rx, p->d_cols, static_cast<const float2*>(wave), p->rx_wave_len,
                                   p->rx_wave_len, -(long long)ri.N_L, static_cast<float2*>(out), p->rx_out_total,
                                   S, st);
    const long long grid_stride = (long long)p->B_rx * p->row_full;
    const long long pad = p->rx_pad_len;
    float2 *wp = nullptr, *grid = nullptr;
    cudaError_t e = fcw::scratch_alloc(&wp, sizeof(float2) * pad * S, st);
    if (e == cudaSuccess) e = fcw::scratch_alloc(&grid, sizeof(float2) * grid_stride * S, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(wp, 0, sizeof(float2) * pad * S, st);
    // x = [0_{N_L}, w, 0 ...] (fc_core.cpp:207-208)
    if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(wp + ri.N_L, sizeof(float2) * pad, wave, sizeof(float2) * p->rx_wave_len,
                              sizeof(float2) * p->rx_wave_len, S, cudaMemcpyDeviceToDevice, st);
    int rc = e == cudaSuccess ? FCW_OK : fcw::set_cuda_error(e, "continuous RX staging");
    if (rc == FCW_OK)
        rc = fcw_rx(p->rx, wp, pad, pad, ri.N_L, grid, grid_stride, S, FCW_GRID_FULL, stream);
    for (int u0 = 0; u0 < S && rc == FCW_OK; u0 += 65535) {
        const int s = std::min(S - u0, 65535);
        e = fcw::cont_columns(*p, false, grid + (long long)u0 * grid_stride, grid_stride,
                              static_cast<float2*>(out) + (long long)u0 * p->rx_out_total, p->rx_out_total, s,
                              p->B_rx, st);
        if (e != cudaSuccess) rc = fcw::set_cuda_error(e, "continuous RX columns");
    }
    if (wp) cudaFreeAsync(wp, st);
    if (grid) cudaFreeAsync(grid, st);
    return rc;
}

}  // extern "C"
