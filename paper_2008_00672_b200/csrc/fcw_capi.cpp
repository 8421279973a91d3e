// Host side of the C ABI (include/fcwave_b200.h): integer-exact geometry, the
// immutable device-resident plan, launch configuration and the pipelined
// host-buffer entry points.  Reference anchors are cited per function.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "fcw_internal.hpp"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? FCW_ENOMEM : FCW_ECUDA;
}

bool is_pow2(long long v) { return v >= 1 && (v & (v - 1)) == 0; }
int ilog2(long long v) {
    int l = 0;
    while ((1LL << l) < v) ++l;
    return l;
}
long long mod_ll(long long a, long long m) {
    long long r = a % m;
    return r < 0 ? r + m : r;
}

// numerology.cpp:44-70
int derive(int N, int L, double overlap, fcw_fc_params* p) {
    if (L < 2 || N < L || N % L != 0) return fail(FCW_EINVAL, "L must divide N");
    const double lo = overlap * L;
    const int L_O = (int)std::lround(lo);
    if (std::fabs(lo - L_O) > 1e-9 || L_O <= 0 || L_O >= L)
        return fail(FCW_EINVAL, "overlap*L must be a positive integer < L");
    const double no = overlap * N;
    const int N_O = (int)std::lround(no);
    if (std::fabs(no - N_O) > 1e-9) return fail(FCW_EINVAL, "overlap*N must be an integer");
    p->L = L;
    p->N = N;
    p->overlap = overlap;
    p->I = N / L;
    p->L_O = L_O;
    p->L_S = L - L_O;
    p->L_L = (L_O + 1) / 2;
    p->L_T = L_O / 2;
    p->N_O = N_O;
    p->N_S = N - N_O;
    p->N_L = (N_O + 1) / 2;
    p->N_T = N_O / 2;
    return FCW_OK;
}

long long cp_partial(const std::vector<int>& cp, int n) {
    long long s = 0;
    for (int q = 1; q <= n; ++q) s += cp[q];
    return s;
}

// Work distribution of one launch (see RunSource in fcw_device.cuh):
// static balanced ranges when each resident team gets few symbols (many GPUs,
// small batches: fewest TX run starts, +-1 symbol balance), dynamic runs of
// `chunk` symbols at full load (absorbs CTA speed differences).  FCW_CHUNK /
// FCW_CHUNK_TX / FCW_CHUNK_RX force dynamic mode with that run length (tests
// use it to exercise the TX carry recompute at every run start).
void pick_schedule(const fcw::Plan& p, int S, bool tx, fcw::KParams& kp) {
    kp.chunk = p.B;
    kp.dynamic = 0;
    for (const char* name : {tx ? "FCW_CHUNK_TX" : "FCW_CHUNK_RX", "FCW_CHUNK"})
        if (const char* e = std::getenv(name)) {
            const int c = std::atoi(e);
            if (c > 0) {
                kp.chunk = std::min(c, p.B);
                kp.dynamic = 1;
                break;
            }
        }
    const int G = (p.N >= 512 && p.N <= 4096) ? 4096 / p.N : 1;
    const long long teams = 2LL * fcw::device_sms() * G;  // 2 resident CTAs per SM
    const long long per_team = (long long)p.B * std::max(S, 1) / teams;
    const char* sched = std::getenv("FCW_SCHED");  // dev A/B knob: "static" keeps balanced static ranges
    const bool force_static = sched && std::strcmp(sched, "static") == 0;
    if (!kp.dynamic && per_team >= 200 && !force_static) {
        kp.dynamic = 1;
        kp.chunk = std::min(p.B, tx ? 140 : 28);  // measured (tools/ab.sh): TX 28 -> 140 is -1%; RX 16 -> 28 is -0.8%
    }
    kp.nchunks = (p.B + kp.chunk - 1) / kp.chunk;
}

}  // namespace

namespace fcw {
// shared with the other C-ABI translation units (fcw_cont.cu)
int set_error(int code, const std::string& msg) { return fail(code, msg); }
int set_cuda_error(cudaError_t e, const char* where) { return cuda_fail(e, where); }

}  // namespace fcw

struct fcw_plan : fcw::Plan {};

namespace fcw {
// Generic (mixed-L) kernels: the zero-bin (zv) and narrowband (nb) kernel
// variants and their trimmed zero lists no longer apply.
void plan_force_generic(fcw_plan* p) {
    p->generic = true;
    plan_clear_special(p);
}
// Drop the zv / nb specialisations (their kernels carry no time-domain I/O):
// the plan then runs the plain uniform-L kernels with the full zero list.
void plan_clear_special(fcw_plan* p) {
    p->zv = false;
    p->nb = false;
}

// Continuous FC with time-domain I/O (fcw_cont.cu): the fused kernels read
// the subband streams (TX) or write the output streams (RX) through the
// column descriptors td, instead of a full grid that cont_cols_kernel
// transforms.  p is a cp = 0 plan whose short paths support it (see
// fcw_cont_plan_create).
int tx_time_domain(const fcw_plan* p, const fc_col* td, const float2* streams, long long stream_stride,
                   float2* wave, long long wave_stride, int S, cudaStream_t st) {
    KParams kp{};
    fill_common(*p, kp);
    if ((long long)S * p->B >= (1LL << 31)) return fail(FCW_ENOTSUP, "S*B symbols per launch must be < 2^31");
    pick_schedule(*p, S, true, kp);
    kp.row_len = 0;
    kp.grid_full = 1;
    kp.td = td;
    kp.in = streams;
    kp.in_stride = stream_stride;
    kp.out = wave;
    kp.out_stride = wave_stride;
    const cudaError_t e = launch_tx(*p, kp, S, st);
    return e == cudaSuccess ? FCW_OK : cuda_fail(e, "continuous tx launch");
}

// RX input is the caller's waveform itself: the kernel reads it at
// rx_base + sigma_n with zeros outside [0, wave_len) (rx_base = -N_L: the
// N_L zeros rx_continuous prepends, fc_core.cpp:207-208).
int rx_time_domain(const fcw_plan* p, const fc_col* td, const float2* wave, long long wave_stride,
                   long long wave_len, long long rx_base, float2* out, long long out_stride, int S,
                   cudaStream_t st) {
    KParams kp{};
    fill_common(*p, kp);
    if ((long long)S * p->B >= (1LL << 31)) return fail(FCW_ENOTSUP, "S*B symbols per launch must be < 2^31");
    pick_schedule(*p, S, false, kp);
    kp.row_len = 0;
    kp.grid_full = 1;
    kp.fused = 0;
    kp.td = td;
    kp.rx_base = rx_base;
    kp.wave_len = wave_len;
    kp.in = wave;
    kp.in_stride = wave_stride;
    kp.out = out;
    kp.out_stride = out_stride;
    const cudaError_t e = launch_rx(*p, kp, S, st);
    return e == cudaSuccess ? FCW_OK : cuda_fail(e, "continuous rx launch");
}
}  // namespace fcw

extern "C" {

const char* fcw_last_error(void) { return g_err.c_str(); }
const char* fcw_version(void) { return "fcwave-b200 0.1 (sm_100a)"; }

int fcw_derive_fc_params(int N, int L, double overlap, fcw_fc_params* out) {
    if (!out) return fail(FCW_EINVAL, "null output");
    return derive(N, L, overlap, out);
}

// numerology.cpp:17-42
int fcw_cp_schedule(int scs_khz, int n_fft, int n_symbols, int* out) {
    if (!is_pow2(n_fft) || n_fft < 16) return fail(FCW_EINVAL, "n_fft must be a power of two >= 16");
    if (scs_khz <= 0 || scs_khz % 15 != 0 || !is_pow2(scs_khz / 15))
        return fail(FCW_EINVAL, "scs_khz must be 15*2^k");
    if (n_symbols < 1) return fail(FCW_EINVAL, "n_symbols must be >= 1");
    if ((80LL * n_fft) % 1024 != 0 || (72LL * n_fft) % 1024 != 0)
        return fail(FCW_EINVAL, "n_fft does not scale the CP pattern to integers");
    for (int n = 0; n < n_symbols; ++n) out[n] = (int)((n % 7 == 0 ? 80LL : 72LL) * n_fft / 1024);
    return FCW_OK;
}

int fcw_nr_cp_schedule(int scs_khz, int n_fft, int n_symbols, int* out) {
    if (!is_pow2(n_fft) || n_fft < 16) return fail(FCW_EINVAL, "n_fft must be a power of two >= 16");
    if (scs_khz <= 0 || scs_khz % 15 != 0 || !is_pow2(scs_khz / 15))
        return fail(FCW_EINVAL, "scs_khz must be 15*2^k");
    if (n_symbols < 1) return fail(FCW_EINVAL, "n_symbols must be >= 1");
    const long long mu2 = scs_khz / 15;  // 2^mu
    if ((144LL * n_fft) % 2048 != 0 || (16LL * mu2 * n_fft) % 2048 != 0)
        return fail(FCW_EINVAL, "n_fft does not scale the CP pattern to integers");
    const int short_cp = (int)(144LL * n_fft / 2048);
    const int long_cp = short_cp + (int)(16LL * mu2 * n_fft / 2048);
    const long long period = 7 * mu2;
    for (int n = 0; n < n_symbols; ++n) out[n] = (n % period == 0) ? long_cp : short_cp;
    return FCW_OK;
}

int fcw_cp_truncate(int n_cp_high, int I, int* l_cp, int* extrap) {
    if (I < 1) return fail(FCW_EINVAL, "interpolation factor must be >= 1");
    *l_cp = n_cp_high / I;
    *extrap = n_cp_high - I * *l_cp;
    return FCW_OK;
}

int fcw_first_block_overlap(const fcw_fc_params* p, int l_cp, double* out) {
    if (l_cp < 0 || l_cp > p->L_L) return fail(FCW_EINVAL, "CP does not fit in the leading overlap (L_CP > L_L)");
    *out = 0.5 - (double)l_cp / p->L;
    return FCW_OK;
}

int fcw_design_window(int L, int n_pass, int n_tb, double* w) {
    if (n_pass <= 0 || n_tb < 0 || n_pass + 2 * n_tb > L) return fail(FCW_EINVAL, "window allocation exceeds L");
    for (int i = 0; i < L; ++i) w[i] = 0.0;
    const int lo = L / 2 - n_pass / 2, hi = lo + n_pass - 1;
    for (int i = lo; i <= hi; ++i) w[i] = 1.0;
    for (int k = 0; k < n_tb; ++k) {
        const double v = std::cos(M_PI * (k + 1) / (2.0 * (n_tb + 1)));
        w[lo - 1 - k] = v * v;
        w[hi + 1 + k] = v * v;
    }
    return FCW_OK;
}

int fcw_centered_active_map(int l_ofdm, int n_active, int skip_dc, int* bins) {
    if (n_active <= 0 || n_active > l_ofdm - (skip_dc ? 1 : 0))
        return fail(FCW_EINVAL, "active subcarriers do not fit the transform");
    int k = 0;
    const int lo = n_active / 2;
    if (skip_dc) {
        for (int ls = -lo; ls <= -1; ++ls) bins[k++] = (ls + l_ofdm) % l_ofdm;
        for (int ls = 1; ls <= n_active - lo; ++ls) bins[k++] = ls;
    } else {
        for (int ls = -lo; ls < n_active - lo; ++ls) bins[k++] = (ls + l_ofdm) % l_ofdm;
    }
    return FCW_OK;
}

int64_t fcw_symbol_sigma(int n, const int* cp, int N) {
    int64_t s = (int64_t)n * N;
    for (int q = 1; q <= n; ++q) s += cp[q];
    return s;
}

int64_t fcw_combined_length(int B, const int* cp, const fcw_fc_params* p) {
    int64_t q = (int64_t)p->N_L + p->N_T + (int64_t)B * p->N;
    for (int i = 1; i <= B - 1; ++i) q += cp[i];
    return q;
}

void* fcw_host_alloc(size_t bytes) {
    void* p = nullptr;
    const cudaError_t e = cudaMallocHost(&p, bytes);
    if (e != cudaSuccess) {
        cuda_fail(e, "cudaMallocHost");
        return nullptr;
    }
    return p;
}

void fcw_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

// ------------------------------------------------------------------- plan

int fcw_plan_create(fcw_plan** out, int N, double overlap, const int* cp_high, int B,
                    const fcw_subband* sbs, int M, unsigned flags) {
    (void)flags;
    if (!out) return fail(FCW_EINVAL, "null plan pointer");
    *out = nullptr;
    if (M < 1 || !sbs) return fail(FCW_EINVAL, "one config per grid required");
    if (B < 1 || !cp_high) return fail(FCW_EINVAL, "no symbols");
    for (int n = 0; n < B; ++n)
        if (cp_high[n] < 0) return fail(FCW_EINVAL, "negative CP length");
    // Reference-valid geometry first (same messages as the reference) ...
    std::vector<fcw_fc_params> ps(M);
    for (int m = 0; m < M; ++m) {
        const fcw_subband& s = sbs[m];
        if (s.l_ofdm != 0 && s.l_ofdm != s.L)
            return fail(FCW_EINVAL, "symbol-synchronized TX requires L == L_OFDM");
        if (!s.window) return fail(FCW_EINVAL, "window length must be L");
        if (int rc = derive(N, s.L, overlap, &ps[m])) return rc;
        if (s.n_active < 0 || (s.n_active > 0 && !s.active_bins))
            return fail(FCW_EINVAL, "active bins missing");
        for (int a = 0; a < s.n_active; ++a)
            if (s.active_bins[a] < 0 || s.active_bins[a] >= s.L)
                return fail(FCW_EINVAL, "active bin outside [0, L)");
        for (int n = 0; n < B; ++n) {
            const int lcp = cp_high[n] / ps[m].I;
            if (lcp > ps[m].L_L) return fail(FCW_EINVAL, "CP exceeds leading overlap (L_CP > L_L)");
            if (lcp >= s.L) return fail(FCW_EINVAL, "l_cp out of range");
        }
        if (ps[m].N_L != ps[0].N_L || ps[m].N_T != ps[0].N_T)
            return fail(FCW_EINVAL, "subbands must share N and the overlap factor");
    }
    // ... then this build's envelope.
    if (overlap != 0.5)
        return fail(FCW_ENOTSUP, "symbol-synchronized path is built for overlap 0.5 (the reference's only "
                                 "consistent setting: combine_symbols writes 3N/2 per symbol)");
    if (!is_pow2(N) || N < 16 || N > fcw::kMaxN) return fail(FCW_ENOTSUP, "N must be a power of two in [16, 4096]");
    for (int m = 0; m < M; ++m)
        if (!is_pow2(sbs[m].L) || sbs[m].L < 4 || sbs[m].L > fcw::kMaxL)
            return fail(FCW_ENOTSUP, "L must be a power of two in [4, 1024]");

    fcw_plan* p = new (std::nothrow) fcw_plan();
    if (!p) return fail(FCW_ENOMEM, "host allocation failed");
    cudaGetDevice(&p->device);
    p->N = N;
    p->B = B;
    p->M = M;
    p->overlap = overlap;
    p->pN = ps[0];
    p->cp.assign(cp_high, cp_high + B);
    p->sigma.resize(B);
    for (int n = 0; n < B; ++n) p->sigma[n] = (long long)n * N + cp_partial(p->cp, n);
    p->Q = (long long)ps[0].N_L + ps[0].N_T + (long long)B * N + cp_partial(p->cp, B - 1);
    p->useful0 = ps[0].N_L;
    p->frame_samples = 0;
    for (int n = 0; n < B; ++n) p->frame_samples += N + p->cp[n];

    // subbands, tables
    p->subs.resize(M);
    int act_off = 0, full_off = 0;
    std::vector<int> cnt(N, 0);
    struct Contrib {
        int m, p0, q, rank;
    };
    std::vector<Contrib> secondary;
    p->h_inv.assign(0, 0);
    for (int m = 0; m < M; ++m) {
        const fcw_subband& s = sbs[m];
        auto& S = p->subs[m];
        S.desc = s;
        S.bins.assign(s.active_bins, s.active_bins + s.n_active);
        S.window.assign(s.window, s.window + s.L);
        S.p = ps[m];
        S.desc.active_bins = nullptr;
        S.desc.window = nullptr;
        fcw::SubDev d{};
        d.L = s.L;
        d.logL = ilog2(s.L);
        d.c = s.c;
        d.logI = ilog2(ps[m].I);
        d.act_off = act_off;
        d.n_act = s.n_active;
        d.full_off = full_off;
        d.cmodN = (int)mod_ll(s.c, N);
        // block_phase(1, c, L_S, L) with L_S = L/2: exp(j*pi*(c mod 2))
        d.bp1 = (mod_ll((long long)mod_ll(s.c, s.L) * ps[m].L_S, s.L) == 0) ? 1.0f : -1.0f;
        d.tx_scale = (float)(std::sqrt((double)ps[m].I) / ((double)N * std::sqrt((double)s.L)));
        d.rx_s0 = (float)(std::sqrt((double)ps[m].I) * ((double)s.L / N) / std::sqrt((double)s.L));
        p->h_sub.push_back(d);
        std::vector<int> inv(s.L, -1);
        for (int a = 0; a < s.n_active; ++a) {
            if (inv[s.active_bins[a]] >= 0) {
                delete p;
                return fail(FCW_EINVAL, "duplicate active bin");
            }
            inv[s.active_bins[a]] = a;
        }
        for (int b = 0; b < s.L; ++b) p->h_inv.push_back(inv[b]);
        for (int p0 = 0; p0 < s.L; ++p0) {
            p->h_win.push_back((float)s.window[p0]);
            const int q = (int)mod_ll((long long)s.c - (s.L + 1) / 2 + p0, N);
            if (s.window[p0] == 0.0) {
                p->h_dest.push_back(-1);
            } else if (cnt[q] == 0) {
                p->h_dest.push_back(q);
                cnt[q] = 1;
            } else {
                secondary.push_back({m, p0, q, cnt[q]});
                cnt[q] += 1;
                p->h_dest.push_back(-2);  // patched below
            }
        }
        act_off += s.n_active;
        full_off += s.L;
        p->Lmax = std::max(p->Lmax, s.L);
    }
    p->row_active = act_off;
    p->row_full = full_off;
    // zero-bin kernel variant (tx_short_half / rx_short_half, ZV): uniform
    // L = 256 at N = 4096 where every subband leaves DFT bins b with
    // b / 16 in [5, 10] inactive and outside its window
    p->zv = N == 4096 && M > 0;
    for (int m = 0; m < M && p->zv; ++m) {
        const fcw_subband& s = sbs[m];
        if (s.L != 256) {
            p->zv = false;
            break;
        }
        for (int b = 80; b < 176 && p->zv; ++b) {
            if ((float)s.window[b ^ 128] != 0.0f) p->zv = false;
            if (p->h_inv[(size_t)m * 256 + b] >= 0) p->zv = false;
        }
        // ... and its active map is the centred one (centered_active_map without a DC
        // gap): active index a sits on DFT bin (a - n_act/2) mod L, so the kernels
        // compute the packed-row index of bin b as (b + n_act/2) mod L without a table
        for (int b = 0; b < 256 && p->zv; ++b) {
            const int a = (b + s.n_active / 2) & 255;
            if (p->h_inv[(size_t)m * 256 + b] != (a < s.n_active ? a : -1)) p->zv = false;
        }
    }
    // secondary contributions: ext slots numbered subband-major (a subband's
    // secondary bins are consecutive from its ext_base); the fix-up list is
    // ordered by contributor rank so shared bins are summed in a fixed order.
    int max_rank = 0;
    for (const Contrib& c : secondary) max_rank = std::max(max_rank, c.rank);
    if (N + (long long)secondary.size() >= 32768) {
        delete p;
        return fail(FCW_ENOTSUP, "too many shared transition bins for the 16-bit spectrum slot index");
    }
    if (max_rank > fcw::kMaxLevels) {
        delete p;
        return fail(FCW_ENOTSUP, "more than 9 subbands share one N-grid bin");
    }
    p->n_ext = (int)secondary.size();
    p->n_lvl = max_rank;
    std::vector<int> sec_idx(p->h_dest.size(), -1);
    for (int k = 0; k < p->n_ext; ++k) {
        const Contrib& c = secondary[k];
        fcw::SubDev& d = p->h_sub[c.m];
        if (k == 0 || secondary[k - 1].m != c.m) d.ext_base = k;
        p->h_dest[d.full_off + c.p0] = N + k;
        sec_idx[d.full_off + c.p0] = k - d.ext_base;
    }
    std::vector<int> order(p->n_ext);
    for (int k = 0; k < p->n_ext; ++k) order[k] = k;
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return secondary[a].rank < secondary[b].rank; });
    for (int k : order) {
        p->h_fix.push_back(secondary[k].q);
        p->h_fix_slot.push_back(k);
    }
    {
        // grouped by the thread that loads the target bin in the long transform (q mod N/16):
        // that thread adds its bins' secondary contributions, in rank order, right before it
        // loads them (tx_kernel), so the fix-up needs no phase and no barrier of its own
        const int T = std::max(1, N / 16);
        std::vector<int> by_owner(order);
        std::stable_sort(by_owner.begin(), by_owner.end(),
                         [&](int a, int b) { return secondary[a].q % T < secondary[b].q % T; });
        p->h_own_start.assign(T + 1, 0);
        for (int k : by_owner) {
            p->h_own_tgt.push_back(secondary[k].q);
            p->h_own_slot.push_back(k);
            ++p->h_own_start[secondary[k].q % T + 1];
        }
        for (int t = 0; t < T; ++t) p->h_own_start[t + 1] += p->h_own_start[t];
    }
    p->lvl_start.assign(max_rank + 1, 0);
    for (int l = 0; l <= max_rank; ++l) {
        int k = 0;
        while (k < p->n_ext && secondary[order[k]].rank < l + 1) ++k;
        p->lvl_start[l] = k;
    }
    // bins no subband touches; with the zero-bin variant the guard band
    // [7N/16, 9N/16) is never read by the long transform (kernel skips it),
    // so those bins go last and are not zero-filled (n_zero_core)
    // (every bin a subband's L-span reads or writes lies outside the guard band)
    p->zv = p->zv && [&] {
        for (int m = 0; m < M; ++m)
            for (int p0 = 0; p0 < sbs[m].L; ++p0) {
                const int q = (int)mod_ll((long long)sbs[m].c - sbs[m].L / 2 + p0, N);
                if (q >= 7 * N / 16 && q < 9 * N / 16) return false;
            }
        return true;
    }();
    // narrowband plans (config 1): every subband span inside 16 bins [k0, k0 + 16)
    // of N = 1024 with L = 16 -> per-thread 16-point long transforms (ZV = 2)
    p->nb = false;
    if (N == 1024) {
        bool uni16 = true;
        for (int m = 0; m < M; ++m) uni16 = uni16 && sbs[m].L == 16;
        if (uni16) {
            std::vector<int> span;
            for (int m = 0; m < M; ++m)
                for (int p0 = 0; p0 < 16; ++p0) span.push_back((int)mod_ll((long long)sbs[m].c - 8 + p0, N));
            for (int k0 : span) {
                bool ok = true;
                for (int q : span) ok = ok && mod_ll((long long)q - k0, N) < 16;
                if (ok) {
                    p->nb = true;
                    p->nb_k0 = k0;
                    break;
                }
            }
        }
    }
    auto core = [&](int q) {
        if (p->nb) return mod_ll((long long)q - p->nb_k0, N) < 16;
        return !(p->zv && q >= 7 * N / 16 && q < 9 * N / 16);
    };
    for (int q = 0; q < N; ++q)
        if (cnt[q] == 0 && core(q)) p->h_zero.push_back(q);
    p->n_zero_core = (int)p->h_zero.size();
    for (int q = 0; q < N; ++q)
        if (cnt[q] == 0 && !core(q)) p->h_zero.push_back(q);
    // L groups
    std::map<int, std::vector<int>> groups;
    for (int m = 0; m < M; ++m) groups[sbs[m].L].push_back(m);
    p->n_groups = 0;
    for (auto& kv : groups) {
        p->grp_L[p->n_groups] = kv.first;
        p->grp_start[p->n_groups] = (int)p->h_grp_sub.size();
        p->grp_count[p->n_groups] = (int)kv.second.size();
        for (int m : kv.second) p->h_grp_sub.push_back(m);
        ++p->n_groups;
    }
    // symbols
    p->h_sym.resize(B);
    for (int n = 0; n < B; ++n) {
        fcw::SymDev s{};
        s.sigma = p->sigma[n];
        s.cp = p->cp[n];
        s.own_len = (n < B - 1) ? N + p->cp[n + 1] : 3 * N / 2;
        s.carry_len = n > 0 ? N / 2 - p->cp[n] : 0;
        s.smodN = (int)mod_ll(cp_partial(p->cp, n), N);
        p->h_sym[n] = s;
    }
    // Bin-class table: per DFT bin b (p0 = b ^ L/2) the active index, the
    // secondary-slot index relative to the subband's ext_base (-1 primary,
    // -2 zero weight) and the window.  Subbands with identical rows share one
    // class (regular allocations have 2-3 classes), so the table stays in L1.
    {
        std::map<std::vector<int>, int> classes;
        for (int m = 0; m < M; ++m) {
            fcw::SubDev& d = p->h_sub[m];
            std::vector<int> key;
            key.push_back(d.L);
            std::vector<int2> rows(d.L);
            for (int b = 0; b < d.L; ++b) {
                const int p0 = b ^ (d.L / 2);
                const float w = p->h_win[d.full_off + p0];
                const int inv = p->h_inv[d.full_off + b];
                const int dst = p->h_dest[d.full_off + p0];
                const int sec = dst < 0 ? -2 : (dst >= N ? sec_idx[d.full_off + p0] : -1);
                int2 e;
                e.x = (inv & 0xffff) | (int)((unsigned)sec << 16);
                std::memcpy(&e.y, &w, 4);
                rows[b] = e;
                key.push_back(e.x);
                key.push_back(e.y);
            }
            auto it = classes.find(key);
            if (it == classes.end()) {
                it = classes.emplace(key, (int)p->h_cls.size()).first;
                p->h_cls.insert(p->h_cls.end(), rows.begin(), rows.end());
            }
            d.cls_off = it->second;
        }
        // The zv kernels keep per-lane (weight, slot code) rows of the classes in TMEM
        // (tmem_tables in fcw_device.cuh).  Both half-warps of a warp read their row with one
        // tcgen05.ld, so a row holds a PAIR of classes: the classes of the two subbands the fixed
        // schedule puts side by side in one warp (TX: pair rounds (done + 2w, done + 2w + 1) while
        // more than one subband per warp remains, then one subband per warp; RX: pair rounds
        // throughout; a missing partner repeats the last subband).  At most kMaxTmemClasses rows.
        if (p->zv) {
            const int W = fcw::kWarps;
            std::vector<std::pair<int, int>> rows;
            auto cls = [&](int m) { return p->h_sub[std::min(m, M - 1)].cls_off / 256; };
            auto row_of = [&](int a, int b) {
                const std::pair<int, int> key(cls(a), cls(b));
                for (size_t j = 0; j < rows.size(); ++j)
                    if (rows[j] == key) return (int)j;
                rows.push_back(key);
                return (int)rows.size() - 1;
            };
            for (int done = 0; done < M;) {  // TX (tx_short_half)
                const bool pair = M - done > W;
                for (int w = 0; w < W; ++w) {
                    const int a = pair ? done + 2 * w : done + w, b = pair ? a + 1 : a;
                    if (a >= M) break;
                    const int j = row_of(a, b);
                    p->h_sub[a].row_tx = j;
                    if (b < M) p->h_sub[b].row_tx = j;
                }
                done += pair ? 2 * W : W;
            }
            for (int done = 0; done < M; done += 2 * W)  // RX (rx_short_half)
                for (int w = 0; w < W; ++w) {
                    const int a = done + 2 * w, b = a + 1;
                    if (a >= M) break;
                    const int j = row_of(a, b);
                    p->h_sub[a].row_rx = j;
                    if (b < M) p->h_sub[b].row_rx = j;
                }
            if ((int)rows.size() > fcw::kMaxTmemClasses) {
                p->zv = false;
            } else {
                for (const auto& r : rows) {
                    p->h_combo.push_back(r.first);
                    p->h_combo.push_back(r.second);
                }
            }
        }
    }
    // device tables in one blob
    std::vector<float2> tw(N);
    for (int k = 0; k < N; ++k) {
        const double a = -2.0 * M_PI * (double)k / N;
        tw[k] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
    auto align = [](size_t v) { return (v + 255) & ~size_t(255); };
    size_t off = 0;
    const size_t o_sub = off;
    off = align(off + sizeof(fcw::SubDev) * M);
    const size_t o_sym = off;
    off = align(off + sizeof(fcw::SymDev) * B);
    const size_t o_bin = off;
    off = align(off + sizeof(int2) * p->h_cls.size());
    const size_t o_fslot = off;
    off = align(off + sizeof(int) * std::max<size_t>(1, p->h_fix_slot.size()));
    const size_t o_inv = off;
    off = align(off + sizeof(int) * p->h_inv.size());
    const size_t o_grp = off;
    off = align(off + sizeof(int) * p->h_grp_sub.size());
    const size_t o_fix = off;
    off = align(off + sizeof(int) * std::max<size_t>(1, p->h_fix.size()));
    const size_t o_zero = off;
    off = align(off + sizeof(int) * std::max<size_t>(1, p->h_zero.size()));
    const size_t o_ostart = off;
    off = align(off + sizeof(int) * p->h_own_start.size());
    const size_t o_otgt = off;
    off = align(off + sizeof(int) * std::max<size_t>(1, p->h_own_tgt.size()));
    const size_t o_oslot = off;
    off = align(off + sizeof(int) * std::max<size_t>(1, p->h_own_slot.size()));
    const size_t o_tw = off;
    off = align(off + sizeof(float2) * N);
    std::vector<unsigned char> host(off, 0);
    std::memcpy(&host[o_sub], p->h_sub.data(), sizeof(fcw::SubDev) * M);
    std::memcpy(&host[o_sym], p->h_sym.data(), sizeof(fcw::SymDev) * B);
    std::memcpy(&host[o_bin], p->h_cls.data(), sizeof(int2) * p->h_cls.size());
    if (!p->h_fix_slot.empty())
        std::memcpy(&host[o_fslot], p->h_fix_slot.data(), sizeof(int) * p->h_fix_slot.size());
    std::memcpy(&host[o_inv], p->h_inv.data(), sizeof(int) * p->h_inv.size());
    std::memcpy(&host[o_grp], p->h_grp_sub.data(), sizeof(int) * p->h_grp_sub.size());
    if (!p->h_fix.empty()) std::memcpy(&host[o_fix], p->h_fix.data(), sizeof(int) * p->h_fix.size());
    if (!p->h_zero.empty()) std::memcpy(&host[o_zero], p->h_zero.data(), sizeof(int) * p->h_zero.size());
    std::memcpy(&host[o_ostart], p->h_own_start.data(), sizeof(int) * p->h_own_start.size());
    if (!p->h_own_tgt.empty()) {
        std::memcpy(&host[o_otgt], p->h_own_tgt.data(), sizeof(int) * p->h_own_tgt.size());
        std::memcpy(&host[o_oslot], p->h_own_slot.data(), sizeof(int) * p->h_own_slot.size());
    }
    std::memcpy(&host[o_tw], tw.data(), sizeof(float2) * N);
    cudaError_t e = cudaMalloc(&p->d_blob, off);
    if (e != cudaSuccess) {
        delete p;
        return cuda_fail(e, "cudaMalloc(plan tables)");
    }
    e = cudaMemcpy(p->d_blob, host.data(), off, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(p->d_blob);
        delete p;
        return cuda_fail(e, "cudaMemcpy(plan tables)");
    }
    auto* base = static_cast<unsigned char*>(p->d_blob);
    p->d_sub = reinterpret_cast<fcw::SubDev*>(base + o_sub);
    p->d_sym = reinterpret_cast<fcw::SymDev*>(base + o_sym);
    p->d_cls = reinterpret_cast<int2*>(base + o_bin);
    p->d_fix_slot = reinterpret_cast<int*>(base + o_fslot);
    p->d_inv = reinterpret_cast<int*>(base + o_inv);
    p->d_grp_sub = reinterpret_cast<int*>(base + o_grp);
    p->d_fix = reinterpret_cast<int*>(base + o_fix);
    p->d_zero = reinterpret_cast<int*>(base + o_zero);
    p->d_own_start = reinterpret_cast<int*>(base + o_ostart);
    p->d_own_tgt = reinterpret_cast<int*>(base + o_otgt);
    p->d_own_slot = reinterpret_cast<int*>(base + o_oslot);
    p->d_tw = reinterpret_cast<float2*>(base + o_tw);
    // SMEM envelope check (one CTA must fit)
    int dev_smem = 0;
    cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device);
    const size_t need = std::max(fcw::tx_smem_bytes(*p), fcw::rx_smem_bytes(*p));
    if ((size_t)dev_smem < need) {
        cudaFree(p->d_blob);
        delete p;
        return fail(FCW_ENOTSUP, "plan exceeds the per-CTA shared-memory envelope");
    }
    p->chunk = p->B;
    *out = p;
    return FCW_OK;
}

void fcw_plan_destroy(fcw_plan* p) {
    if (!p) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(p->device);
    for (int i = 0; i < 2; ++i) {
        for (int j = 0; j < 2; ++j)
            if (p->stage[i][j]) cudaFree(p->stage[i][j]);
        if (p->streams[i]) cudaStreamDestroy(p->streams[i]);
    }
    if (p->d_blob) cudaFree(p->d_blob);
    cudaSetDevice(cur);
    delete p;
}

int fcw_plan_get_info(const fcw_plan* p, fcw_plan_info* info) {
    if (!p || !info) return fail(FCW_EINVAL, "null argument");
    info->N = p->N;
    info->B = p->B;
    info->M = p->M;
    info->overlap = p->overlap;
    info->Q = p->Q;
    info->useful0 = p->useful0;
    info->frame_samples = p->frame_samples;
    info->row_active = p->row_active;
    info->row_full = p->row_full;
    info->N_L = p->pN.N_L;
    info->N_T = p->pN.N_T;
    info->chunk = p->chunk;
    info->kernel_variant = p->zv ? 1 : (p->nb ? 2 : (fcw::plan_team_only(*p) ? 3 : 0));
    info->tmem_rows = p->zv ? (int)p->h_combo.size() / 2 : 0;
    return FCW_OK;
}

int fcw_plan_sigma(const fcw_plan* p, int64_t* sigma) {
    if (!p || !sigma) return fail(FCW_EINVAL, "null argument");
    for (int n = 0; n < p->B; ++n) sigma[n] = p->sigma[n];
    return FCW_OK;
}

int fcw_plan_cp_split(const fcw_plan* p, int m, int* l_cp, int* extrap) {
    if (!p || !l_cp || !extrap) return fail(FCW_EINVAL, "null argument");
    if (m < 0 || m >= p->M) return fail(FCW_ERANGE, "subband index");
    const int I = p->subs[m].p.I;
    for (int n = 0; n < p->B; ++n) {
        l_cp[n] = p->cp[n] / I;
        extrap[n] = p->cp[n] - I * l_cp[n];
    }
    return FCW_OK;
}

int fcw_plan_bin_map(const fcw_plan* p, int m, int* q, int* b) {
    if (!p) return fail(FCW_EINVAL, "null argument");
    if (m < 0 || m >= p->M) return fail(FCW_ERANGE, "subband index");
    const auto& s = p->subs[m];
    const int L = s.desc.L;
    for (int p0 = 0; p0 < L; ++p0) {
        if (q) q[p0] = (int)mod_ll((long long)s.desc.c - (L + 1) / 2 + p0, p->N);
        if (b) b[p0] = (p0 + L / 2) % L;
    }
    return FCW_OK;
}

int fcw_plan_rx_starts(const fcw_plan* p, int64_t useful0, int64_t* starts) {
    if (!p || !starts) return fail(FCW_EINVAL, "null argument");
    for (int n = 0; n < p->B; ++n) starts[n] = useful0 - p->pN.N_L + p->sigma[n];
    return FCW_OK;
}

int fcw_plan_fc_params(const fcw_plan* p, int m, fcw_fc_params* out) {
    if (!p || !out) return fail(FCW_EINVAL, "null argument");
    if (m < 0 || m >= p->M) return fail(FCW_ERANGE, "subband index");
    *out = p->subs[m].p;
    return FCW_OK;
}

// --------------------------------------------------------- device entry points

int fcw_tx(const fcw_plan* p, const void* grid, int64_t grid_stride, void* wave, int64_t wave_stride, int S,
           unsigned flags, void* stream) {
    if (!p) return fail(FCW_EINVAL, "null plan");
    if (S < 0) return fail(FCW_EINVAL, "negative unit count");
    if (S == 0) return FCW_OK;
    if (!grid || !wave) return fail(FCW_EINVAL, "null buffer");
    const int row = (flags & FCW_GRID_FULL) ? p->row_full : p->row_active;
    if (grid_stride == 0) grid_stride = (int64_t)p->B * row;
    if (wave_stride == 0) wave_stride = p->Q;
    if (grid_stride < (int64_t)p->B * row) return fail(FCW_EINVAL, "grid unit stride too small");
    if (wave_stride < p->Q) return fail(FCW_EINVAL, "waveform unit stride smaller than Q");
    fcw::KParams kp{};
    fcw::fill_common(*p, kp);
    if ((long long)S * p->B >= (1LL << 31)) return fail(FCW_ENOTSUP, "S*B symbols per launch must be < 2^31");
    pick_schedule(*p, S, true, kp);
    kp.row_len = row;
    kp.grid_full = (flags & FCW_GRID_FULL) ? 1 : 0;
    kp.accumulate = (flags & FCW_TX_ACCUMULATE) ? 1 : 0;
    kp.in = static_cast<const float2*>(grid);
    kp.in_stride = grid_stride;
    kp.out = static_cast<float2*>(wave);
    kp.out_stride = wave_stride;
    const cudaError_t e = fcw::launch_tx(*p, kp, S, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "tx launch");
    return FCW_OK;
}

int fcw_rx(const fcw_plan* p, const void* wave, int64_t wave_stride, int64_t wave_len, int64_t useful0,
           void* grid, int64_t grid_stride, int S, unsigned flags, void* stream) {
    if (!p) return fail(FCW_EINVAL, "null plan");
    if (S < 0) return fail(FCW_EINVAL, "negative unit count");
    if (S == 0) return FCW_OK;
    if (!grid || !wave) return fail(FCW_EINVAL, "null buffer");
    if (wave_stride == 0) wave_stride = wave_len;
    if (wave_stride < wave_len) return fail(FCW_EINVAL, "waveform unit stride smaller than its length");
    // rx_segment bounds (fc_sync.cpp:146-151), checked for every symbol
    for (int n = 0; n < p->B; ++n) {
        const long long start = useful0 - p->pN.N_L + p->sigma[n];
        if (start < 0 || start + 3LL * p->N / 2 > wave_len)
            return fail(FCW_EINVAL, "waveform too short for symbol window");
    }
    const int row = (flags & FCW_GRID_FULL) ? p->row_full : p->row_active;
    if (grid_stride == 0) grid_stride = (int64_t)p->B * row;
    if (grid_stride < (int64_t)p->B * row) return fail(FCW_EINVAL, "grid unit stride too small");
    fcw::KParams kp{};
    fcw::fill_common(*p, kp);
    if ((long long)S * p->B >= (1LL << 31)) return fail(FCW_ENOTSUP, "S*B symbols per launch must be < 2^31");
    pick_schedule(*p, S, false, kp);
    kp.row_len = row;
    kp.grid_full = (flags & FCW_GRID_FULL) ? 1 : 0;
    kp.fused = (flags & FCW_RX_FUSED) ? 1 : 0;
    kp.rx_base = useful0 - p->pN.N_L;
    kp.wave_len = wave_len;
    kp.in = static_cast<const float2*>(wave);
    kp.in_stride = wave_stride;
    kp.out = static_cast<float2*>(grid);
    kp.out_stride = grid_stride;
    const cudaError_t e = fcw::launch_rx(*p, kp, S, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "rx launch");
    return FCW_OK;
}

// ----------------------------------------------- per-symbol entry points
namespace {
constexpr double kTwoPi = 6.283185307179586476925286766559;

// symbol_phase (fc_sync.cpp:45-50): exp(+j 2 pi ((c mod N)(S_n mod N) mod N) / N)
void symbol_phase_d(int n, int c, const std::vector<int>& cp, int N, double* re, double* im) {
    long long sn = 0;
    for (int q = 1; q <= n; ++q) sn += cp[(size_t)q];
    const long long num = ((long long)c % N) * (sn % N) % N;
    const double a = kTwoPi * (double)num / N;
    *re = std::cos(a);
    *im = std::sin(a);
}
// block_phase (fc_core.cpp:41-44): exp(+j 2 pi (r c mod L) L_S mod L / L)
void block_phase_d(long long r, int c, int L_S, int L, double* re, double* im) {
    const long long num = r * c % L * L_S % L;
    const double a = kTwoPi * (double)num / L;
    *re = std::cos(a);
    *im = std::sin(a);
}
float2 f2(double re, double im) { return make_float2((float)re, (float)im); }
int check_sym(const fcw_plan* p, int m, int S) {
    if (!p) return fail(FCW_EINVAL, "null plan");
    if (m < 0 || m >= p->M) return fail(FCW_ERANGE, "subband index");
    if (S < 0) return fail(FCW_EINVAL, "negative unit count");
    return FCW_OK;
}
}  // namespace

int fcw_symbol_phase(int n, int c, const int* cp_high, int B, int N, double* re, double* im) {
    if (!re || !im || (n > 0 && !cp_high)) return fail(FCW_EINVAL, "null argument");
    if (n < 0) return fail(FCW_EINVAL, "symbol index");  // fc_sync.cpp:46
    if (n >= B && n > 0) return fail(FCW_ERANGE, "symbol index outside CP schedule");
    if (N <= 0) return fail(FCW_EINVAL, "N must be positive");
    std::vector<int> cp(cp_high, cp_high + (n > 0 ? B : 0));
    symbol_phase_d(n, c, cp, N, re, im);
    return FCW_OK;
}

int fcw_block_phase(int64_t r, int c, int L_S, int L, double* re, double* im) {
    if (!re || !im) return fail(FCW_EINVAL, "null argument");
    if (L <= 0) return fail(FCW_EINVAL, "L must be positive");
    block_phase_d(r, c, L_S, L, re, im);
    return FCW_OK;
}

int fcw_tx_symbol(const fcw_plan* p, int m, int n, const void* sym, int64_t sym_stride, int l_cp, void* out,
                  int64_t out_stride, int S, void* stream) {
    if (int rc = check_sym(p, m, S)) return rc;
    if (n < 0 || n >= p->B) return fail(FCW_ERANGE, "symbol index outside CP schedule");
    if (S == 0) return FCW_OK;
    if (!sym || !out) return fail(FCW_EINVAL, "null buffer");
    const auto& sb = p->subs[m];
    if (sb.desc.l_ofdm != sb.desc.L) return fail(FCW_EINVAL, "symbol-synchronized TX requires L == L_OFDM");
    if (l_cp < 0 || l_cp > sb.p.L_L) return fail(FCW_EINVAL, "CP exceeds leading overlap (L_CP > L_L)");  // fc_sync.cpp:35
    if (sym_stride == 0) sym_stride = sb.desc.L + l_cp;
    if (out_stride == 0) out_stride = 3LL * p->N / 2;
    if (sym_stride < sb.desc.L + l_cp || out_stride < 3LL * p->N / 2) return fail(FCW_EINVAL, "stride too small");
    double tr, ti, b1r, b1i;
    symbol_phase_d(n, sb.desc.c, p->cp, p->N, &tr, &ti);
    block_phase_d(1, sb.desc.c, sb.p.L_S, sb.desc.L, &b1r, &b1i);  // block_phase(0) = 1
    const cudaError_t e = fcw::sym_tx_symbol(*p, m, static_cast<const float2*>(sym), sym_stride, l_cp, f2(tr, ti),
                                             f2(b1r * tr - b1i * ti, b1r * ti + b1i * tr),
                                             (float)std::sqrt((double)sb.p.I), static_cast<float2*>(out), out_stride,
                                             S, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "tx_symbol");
    return FCW_OK;
}

int fcw_combine_symbols(const fcw_plan* p, const void* syms, int64_t sym_unit_stride, void* wave,
                        int64_t wave_stride, int S, void* stream) {
    if (!p) return fail(FCW_EINVAL, "null plan");
    if (S < 0) return fail(FCW_EINVAL, "negative unit count");
    if (S == 0) return FCW_OK;
    if (!syms || !wave) return fail(FCW_EINVAL, "null buffer");
    const long long per = (long long)p->B * (3LL * p->N / 2);
    if (sym_unit_stride == 0) sym_unit_stride = per;
    if (wave_stride == 0) wave_stride = p->Q;
    if (sym_unit_stride < per || wave_stride < p->Q) return fail(FCW_EINVAL, "stride too small");
    const cudaError_t e = fcw::sym_combine(*p, static_cast<const float2*>(syms), sym_unit_stride,
                                           static_cast<float2*>(wave), wave_stride, S,
                                           static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "combine_symbols");
    return FCW_OK;
}

int fcw_rx_segment(const fcw_plan* p, const void* wave, int64_t wave_stride, int64_t wave_len, int64_t useful0,
                   int n, void* y0, void* y1, int64_t y_stride, int S, void* stream) {
    if (!p) return fail(FCW_EINVAL, "null plan");
    if (n < 0 || n >= p->B) return fail(FCW_ERANGE, "symbol index outside CP schedule");  // fc_sync.cpp:146-147
    if (S < 0) return fail(FCW_EINVAL, "negative unit count");
    const long long start = useful0 - p->pN.N_L + p->sigma[(size_t)n];
    if (start < 0 || start + 3LL * p->N / 2 > wave_len)
        return fail(FCW_EINVAL, "waveform too short for symbol window");  // fc_sync.cpp:149-151
    if (S == 0) return FCW_OK;
    if (!wave || !y0 || !y1) return fail(FCW_EINVAL, "null buffer");
    if (wave_stride == 0) wave_stride = wave_len;
    if (y_stride == 0) y_stride = p->N;
    if (wave_stride < wave_len || y_stride < p->N) return fail(FCW_EINVAL, "stride too small");
    const size_t b = sizeof(float2);
    auto st = static_cast<cudaStream_t>(stream);
    const float2* w = static_cast<const float2*>(wave) + start;
    cudaError_t e = cudaMemcpy2DAsync(y0, b * y_stride, w, b * wave_stride, b * p->N, S, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(y1, b * y_stride, w + p->N / 2, b * wave_stride, b * p->N, S, cudaMemcpyDeviceToDevice,
                              st);
    if (e != cudaSuccess) return cuda_fail(e, "rx_segment");
    return FCW_OK;
}

int fcw_rx_block_freq(const fcw_plan* p, int m, const void* y, int64_t y_stride, double phase_re, double phase_im,
                      void* g, int64_t g_stride, int S, void* stream) {
    if (int rc = check_sym(p, m, S)) return rc;
    if (S == 0) return FCW_OK;
    if (!y || !g) return fail(FCW_EINVAL, "null buffer");
    const int L = p->subs[m].desc.L;
    if (y_stride == 0) y_stride = p->N;
    if (g_stride == 0) g_stride = L;
    if (y_stride < p->N || g_stride < L) return fail(FCW_EINVAL, "stride too small");
    const cudaError_t e = fcw::sym_rx_block_freq(*p, m, static_cast<const float2*>(y), y_stride, f2(phase_re, -phase_im),
                                                 static_cast<float2*>(g), g_stride, S,
                                                 static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "rx_block_freq");
    return FCW_OK;
}

int fcw_rx_symbol_simplified(const fcw_plan* p, int m, const void* g0, const void* g1, int64_t g_stride, void* out,
                             int64_t out_stride, int S, void* stream) {
    if (int rc = check_sym(p, m, S)) return rc;
    const auto& sb = p->subs[m];
    if (sb.p.L_S * 2 != sb.desc.L) return fail(FCW_EINVAL, "fused RX path requires 50 % overlap");  // fc_sync.cpp:199
    if (S == 0) return FCW_OK;
    if (!g0 || !g1 || !out) return fail(FCW_EINVAL, "null buffer");
    const int L = sb.desc.L;
    if (g_stride == 0) g_stride = L;
    if (out_stride == 0) out_stride = L;
    if (g_stride < L || out_stride < L) return fail(FCW_EINVAL, "stride too small");
    const double scale = std::sqrt((double)sb.p.I) * ((double)L / p->N) / std::sqrt((double)L);
    const cudaError_t e = fcw::sym_rx_simplified(*p, m, static_cast<const float2*>(g0), static_cast<const float2*>(g1),
                                                 g_stride, (float)scale, static_cast<float2*>(out), out_stride, S,
                                                 static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "rx_symbol_simplified");
    return FCW_OK;
}

int fcw_rx_symbol_direct(const fcw_plan* p, int m, int n, const void* y0, const void* y1, int64_t y_stride, void* out,
                         int64_t out_stride, int S, void* stream) {
    if (int rc = check_sym(p, m, S)) return rc;
    if (n < 0 || n >= p->B) return fail(FCW_ERANGE, "symbol index outside CP schedule");
    const auto& sb = p->subs[m];
    if (sb.desc.l_ofdm != sb.desc.L) return fail(FCW_EINVAL, "symbol-synchronized RX requires L == L_OFDM");
    if (S == 0) return FCW_OK;
    if (!y0 || !y1 || !out) return fail(FCW_EINVAL, "null buffer");
    const int L = sb.desc.L;
    if (y_stride == 0) y_stride = p->N;
    if (out_stride == 0) out_stride = L;
    if (y_stride < p->N || out_stride < L) return fail(FCW_EINVAL, "stride too small");
    double tr, ti, b1r, b1i;
    symbol_phase_d(n, sb.desc.c, p->cp, p->N, &tr, &ti);
    block_phase_d(1, sb.desc.c, sb.p.L_S, L, &b1r, &b1i);
    const double p1r = b1r * tr - b1i * ti, p1i = b1r * ti + b1i * tr;
    const cudaError_t e = fcw::sym_rx_direct(*p, m, static_cast<const float2*>(y0), static_cast<const float2*>(y1),
                                             y_stride, f2(tr, -ti), f2(p1r, -p1i), (float)std::sqrt((double)sb.p.I),
                                             static_cast<float2*>(out), out_stride, S,
                                             static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "rx_symbol_direct");
    return FCW_OK;
}

int fcw_gen_qam(const fcw_plan* p, uint64_t seed, int64_t unit0, int S, int bits, void* grid, void* stream) {
    if (!p || !grid) return fail(FCW_EINVAL, "null argument");
    if (bits != 2 && bits != 4 && bits != 6 && bits != 8) return fail(FCW_EINVAL, "bits_per_symbol must be 2,4,6,8");
    if (S <= 0) return FCW_OK;
    const cudaError_t e =
        fcw::launch_gen_qam(*p, seed, unit0, S, bits, static_cast<float2*>(grid), static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "gen_qam launch");
    return FCW_OK;
}

// ------------------------------------------------------------- link step

int fcw_link_stats(const fcw_plan* p, const void* grid, int64_t grid_stride, int S, uint64_t seed, int64_t unit0,
                   int bits, fcw_link_stat* stats, void* stream) {
    if (!p || !grid || !stats) return fail(FCW_EINVAL, "null argument");
    if (bits != 2 && bits != 4 && bits != 6 && bits != 8) return fail(FCW_EINVAL, "bits_per_symbol must be 2,4,6,8");
    if (S < 0) return fail(FCW_EINVAL, "negative unit count");
    if (S == 0) return FCW_OK;
    const int64_t per_unit = (int64_t)p->B * p->row_active;
    if (grid_stride == 0) grid_stride = per_unit;
    if (grid_stride < per_unit) return fail(FCW_EINVAL, "grid unit stride too small");
    std::vector<double> num(S), den(S);
    std::vector<long long> err(S);
    const cudaError_t e = fcw::link_stats(*p, static_cast<const float2*>(grid), grid_stride, S, seed, unit0, bits,
                                          num.data(), den.data(), err.data(), static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "link_stats");
    for (int u = 0; u < S; ++u) stats[u] = fcw_link_stat{num[u], den[u], err[u], per_unit * bits};
    return FCW_OK;
}

int fcw_awgn(const fcw_plan* p, void* wave, int64_t wave_stride, int64_t wave_len, int S, double sigma2,
             uint64_t seed, int64_t unit0, void* stream) {
    if (!p || !wave) return fail(FCW_EINVAL, "null argument");
    if (S < 0 || wave_len < 0) return fail(FCW_EINVAL, "negative size");
    if (!(sigma2 >= 0.0)) return fail(FCW_EINVAL, "noise variance must be >= 0");
    if (wave_stride == 0) wave_stride = wave_len;
    if (wave_stride < wave_len) return fail(FCW_EINVAL, "waveform unit stride smaller than its length");
    if (S == 0 || wave_len == 0) return FCW_OK;
    const cudaError_t e = fcw::awgn(static_cast<float2*>(wave), wave_stride, wave_len, S, sigma2, seed, unit0,
                                    static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "awgn launch");
    return FCW_OK;
}

int fcw_wave_power(const fcw_plan* p, const void* wave, int64_t wave_stride, int64_t wave_len, int S, int64_t begin,
                   int64_t end, double* power, void* stream) {
    if (!p || !wave || !power) return fail(FCW_EINVAL, "null argument");
    if (S < 0) return fail(FCW_EINVAL, "negative unit count");
    if (wave_stride == 0) wave_stride = wave_len;
    if (wave_stride < wave_len) return fail(FCW_EINVAL, "waveform unit stride smaller than its length");
    begin = std::max<int64_t>(begin, 0);
    end = std::min<int64_t>(end, wave_len);
    if (end <= begin) return fail(FCW_EINVAL, "empty measurement span");  // channel.cpp:151
    if (S == 0) return FCW_OK;
    const cudaError_t e = fcw::wave_power(static_cast<const float2*>(wave), wave_stride, S, begin, end, power,
                                          static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "wave_power");
    return FCW_OK;
}

int fcw_wave_zero(void* wave, int64_t wave_stride, int S, int64_t begin, int64_t end, void* stream) {
    if (!wave && S > 0) return fail(FCW_EINVAL, "null argument");
    if (S < 0 || begin < 0 || end < begin || (S > 1 && wave_stride < end))
        return fail(FCW_EINVAL, "invalid zero span");
    if (S == 0 || end == begin) return FCW_OK;
    const size_t pitch = sizeof(float2) * (size_t)(S > 1 ? wave_stride : end);
    const cudaError_t e = cudaMemset2DAsync(static_cast<float2*>(wave) + begin, pitch, 0,
                                            sizeof(float2) * (size_t)(end - begin), (size_t)S,
                                            static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "wave_zero");
    return FCW_OK;
}

int fcw_draw_tdl(const double* delay_ns, const double* power_lin, int n_taps, double fs_hz, uint64_t seed,
                 int* delays, double* gains) {
    if (n_taps < 0 || (n_taps > 0 && (!delay_ns || !power_lin || !delays || !gains)))
        return fail(FCW_EINVAL, "null argument");
    uint64_t st = seed ? seed : 0x1234567890abcdefULL;  // GaussianRng ctor (channel.cpp:26)
    auto next = [&]() {
        uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    };
    for (int k = 0; k < n_taps; ++k) {
        delays[k] = (int)std::lround(delay_ns[k] * 1e-9 * fs_hz);
        const double u1 = ((double)(next() >> 11) + 1.0) * 0x1p-53;
        const double u2 = (double)(next() >> 11) * 0x1p-53;
        const double r = std::sqrt(-std::log(u1)), a = std::sqrt(power_lin[k]);
        gains[2 * k] = a * (r * std::cos(2.0 * 3.14159265358979323846 * u2));
        gains[2 * k + 1] = a * (r * std::sin(2.0 * 3.14159265358979323846 * u2));
    }
    return FCW_OK;
}

int fcw_apply_channel(const void* in, void* out, int64_t stride, int64_t len, int S, const int* delays,
                      const double* gains, int n_taps, void* stream) {
    if (!in || !out || (n_taps > 0 && (!delays || !gains))) return fail(FCW_EINVAL, "null argument");
    if (in == out) return fail(FCW_EINVAL, "apply_channel is out of place");
    if (S < 0 || len < 0 || n_taps < 0) return fail(FCW_EINVAL, "negative size");
    if (n_taps > 64) return fail(FCW_ENOTSUP, "at most 64 taps");
    if (S > 65535) return fail(FCW_ENOTSUP, "at most 65535 units per call");
    if (stride == 0) stride = len;
    if (stride < len) return fail(FCW_EINVAL, "waveform unit stride smaller than its length");
    if (S == 0 || len == 0) return FCW_OK;
    for (long long i = 0; i < (long long)S * n_taps; ++i)
        if (delays[i] < 0) return fail(FCW_EINVAL, "negative tap delay");
    std::vector<float2> g((size_t)S * n_taps);
    for (size_t i = 0; i < g.size(); ++i) g[i] = make_float2((float)gains[2 * i], (float)gains[2 * i + 1]);
    const cudaError_t e = fcw::apply_channel(static_cast<const float2*>(in), static_cast<float2*>(out), stride, len, S,
                                             delays, g.data(), n_taps, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "apply_channel");
    return FCW_OK;
}

int fcw_psd(const void* wave, int64_t wave_stride, int64_t wave_len, int S, int seg_len, double overlap,
            double* out, void* stream) {
    if (!wave || !out) return fail(FCW_EINVAL, "null argument");
    if (seg_len <= 0 || seg_len > wave_len) return fail(FCW_EINVAL, "waveform shorter than one segment");
    if (overlap < 0.0 || overlap >= 1.0) return fail(FCW_EINVAL, "overlap fraction in [0,1)");  // metrics.cpp:131
    if (!is_pow2(seg_len) || seg_len < 64 || seg_len > 4096)
        return fail(FCW_ENOTSUP, "seg_len must be a power of two in [64, 4096]");
    if (S < 0) return fail(FCW_EINVAL, "negative unit count");
    if (wave_stride == 0) wave_stride = wave_len;
    if (wave_stride < wave_len) return fail(FCW_EINVAL, "waveform unit stride smaller than its length");
    if (S == 0) return FCW_OK;
    if (S > 65535) return fail(FCW_ENOTSUP, "at most 65535 units per call");
    const cudaError_t e = fcw::psd(static_cast<const float2*>(wave), wave_stride, wave_len, S, seg_len, overlap, out,
                                   static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "psd");
    return FCW_OK;
}

// ------------------------------------------------------ host-buffer pipeline

namespace {

int ensure_stage(fcw_plan* p, int set, int which, size_t bytes) {
    if (p->stage_bytes[set][which] >= bytes) return FCW_OK;
    if (p->stage[set][which]) cudaFree(p->stage[set][which]);
    p->stage[set][which] = nullptr;
    p->stage_bytes[set][which] = 0;
    cudaError_t e = cudaMalloc(&p->stage[set][which], bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(staging)");
    p->stage_bytes[set][which] = bytes;
    return FCW_OK;
}

int ensure_streams(fcw_plan* p) {
    for (int i = 0; i < 2; ++i)
        if (!p->streams[i]) {
            cudaError_t e = cudaStreamCreateWithFlags(&p->streams[i], cudaStreamNonBlocking);
            if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
        }
    return FCW_OK;
}

// Units per pipeline chunk: ~256 MiB of staging per direction and set.
int units_per_chunk(size_t in_unit, size_t out_unit, int S) {
    const size_t budget = 256u << 20;
    size_t u = budget / std::max<size_t>(1, std::max(in_unit, out_unit));
    if (u < 1) u = 1;
    // at least 4 chunks when there is enough work, so copies overlap kernels
    const size_t quarter = (S + 3) / 4;
    if (quarter >= 1 && u > quarter) u = quarter;
    return (int)std::min<size_t>(u, (size_t)S);
}

}  // namespace

int fcw_tx_host(fcw_plan* p, const void* grid_host, void* wave_host, int S, unsigned flags) {
    if (!p) return fail(FCW_EINVAL, "null plan");
    if (S <= 0) return S == 0 ? FCW_OK : fail(FCW_EINVAL, "negative unit count");
    if (!grid_host || !wave_host) return fail(FCW_EINVAL, "null buffer");
    std::lock_guard<std::mutex> lk(p->host_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(p->device);
    const int row = (flags & FCW_GRID_FULL) ? p->row_full : p->row_active;
    const size_t in_unit = sizeof(float2) * (size_t)p->B * row;
    const size_t out_unit = sizeof(float2) * (size_t)p->Q;
    const int U = units_per_chunk(in_unit, out_unit, S);
    int rc = ensure_streams(p);
    for (int s = 0; rc == FCW_OK && s < 2; ++s) {
        rc = ensure_stage(p, s, 0, in_unit * U);
        if (rc == FCW_OK) rc = ensure_stage(p, s, 1, out_unit * U);
    }
    for (int u0 = 0, c = 0; rc == FCW_OK && u0 < S; u0 += U, ++c) {
        const int n = std::min(U, S - u0);
        const int set = c & 1;
        cudaStream_t st = p->streams[set];
        cudaError_t e = cudaMemcpyAsync(p->stage[set][0], static_cast<const char*>(grid_host) + in_unit * u0,
                                        in_unit * n, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) {
            rc = cuda_fail(e, "H2D");
            break;
        }
        rc = fcw_tx(p, p->stage[set][0], 0, p->stage[set][1], 0, n, flags, st);
        if (rc) break;
        e = cudaMemcpyAsync(static_cast<char*>(wave_host) + out_unit * u0, p->stage[set][1], out_unit * n,
                            cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) rc = cuda_fail(e, "D2H");
    }
    for (int s = 0; s < 2; ++s) {
        const cudaError_t e = cudaStreamSynchronize(p->streams[s]);
        if (e != cudaSuccess && rc == FCW_OK) rc = cuda_fail(e, "tx_host sync");
    }
    cudaSetDevice(cur);
    return rc;
}

int fcw_rx_host(fcw_plan* p, const void* wave_host, int64_t wave_len, int64_t useful0, void* grid_host, int S,
                unsigned flags) {
    if (!p) return fail(FCW_EINVAL, "null plan");
    if (S <= 0) return S == 0 ? FCW_OK : fail(FCW_EINVAL, "negative unit count");
    if (!grid_host || !wave_host) return fail(FCW_EINVAL, "null buffer");
    std::lock_guard<std::mutex> lk(p->host_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(p->device);
    const int row = (flags & FCW_GRID_FULL) ? p->row_full : p->row_active;
    const size_t in_unit = sizeof(float2) * (size_t)wave_len;
    const size_t out_unit = sizeof(float2) * (size_t)p->B * row;
    const int U = units_per_chunk(in_unit, out_unit, S);
    int rc = ensure_streams(p);
    for (int s = 0; rc == FCW_OK && s < 2; ++s) {
        rc = ensure_stage(p, s, 0, in_unit * U);
        if (rc == FCW_OK) rc = ensure_stage(p, s, 1, out_unit * U);
    }
    for (int u0 = 0, c = 0; rc == FCW_OK && u0 < S; u0 += U, ++c) {
        const int n = std::min(U, S - u0);
        const int set = c & 1;
        cudaStream_t st = p->streams[set];
        cudaError_t e = cudaMemcpyAsync(p->stage[set][0], static_cast<const char*>(wave_host) + in_unit * u0,
                                        in_unit * n, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) {
            rc = cuda_fail(e, "H2D");
            break;
        }
        rc = fcw_rx(p, p->stage[set][0], 0, wave_len, useful0, p->stage[set][1], 0, n, flags, st);
        if (rc) break;
        e = cudaMemcpyAsync(static_cast<char*>(grid_host) + out_unit * u0, p->stage[set][1], out_unit * n,
                            cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) rc = cuda_fail(e, "D2H");
    }
    for (int s = 0; s < 2; ++s) {
        const cudaError_t e = cudaStreamSynchronize(p->streams[s]);
        if (e != cudaSuccess && rc == FCW_OK) rc = cuda_fail(e, "rx_host sync");
    }
    cudaSetDevice(cur);
    return rc;
}

}  // extern "C"
