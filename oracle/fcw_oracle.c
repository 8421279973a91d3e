/*
 * TEST INFRASTRUCTURE ONLY — see fcw_oracle.h for the rules and the pins.
 *
 * Plain-C restatement of the reference's symbol-synchronized FC TX/RX
 * (fcwave, arXiv 2008.00672) in double precision.  Each function names the
 * reference file:line it restates.  The FFT is this file's own radix-2
 * transform; the reference delegates to FFTW (proj/src/fft.cpp:47-61), whose
 * DFT definition (forward unscaled e^{-j}, inverse e^{+j} scaled 1/n) is what
 * fco_fft implements.
 */
#include "fcw_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.14159265358979323846264338327950288;

static int is_pow2(int v) { return v >= 1 && (v & (v - 1)) == 0; }
static int64_t mod64(int64_t a, int64_t m) {
    int64_t r = a % m;
    return r < 0 ? r + m : r;
}

/* numerology.cpp:44-70 */
int fco_derive_params(int N, int L, double overlap, fco_params* p) {
    if (L < 2 || N < L || N % L != 0) return 1;
    const double lo = overlap * L;
    const int L_O = (int)lround(lo);
    if (fabs(lo - L_O) > 1e-9 || L_O <= 0 || L_O >= L) return 1;
    const double no = overlap * N;
    const int N_O = (int)lround(no);
    if (fabs(no - N_O) > 1e-9) return 1;
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
    return 0;
}

/* numerology.cpp:17-42 (make_numerology validation + cp_schedule) */
int fco_cp_schedule(int scs_khz, int n_fft, int n_symbols, int* out) {
    if (!is_pow2(n_fft) || n_fft < 16) return 1;
    if (scs_khz <= 0 || scs_khz % 15 != 0 || !is_pow2(scs_khz / 15)) return 1;
    if (n_symbols < 1) return 1;
    if ((80LL * n_fft) % 1024 != 0 || (72LL * n_fft) % 1024 != 0) return 1;
    for (int n = 0; n < n_symbols; ++n) out[n] = (int)((n % 7 == 0 ? 80LL : 72LL) * n_fft / 1024);
    return 0;
}

/* fc_sync.cpp:26-32 */
void fco_cp_truncate(int n_cp_high, int I, int* l_cp, int* extrap) {
    *l_cp = n_cp_high / I;
    *extrap = n_cp_high - I * *l_cp;
}

/* fc_sync.cpp:18-23: sum over symbols 1..n */
int64_t fco_cp_partial_sum(const int* cp, int n) {
    int64_t s = 0;
    for (int q = 1; q <= n; ++q) s += cp[q];
    return s;
}

/* fc_sync.cpp:86-88 */
int64_t fco_symbol_sigma(int n, const int* cp, int N) { return (int64_t)n * N + fco_cp_partial_sum(cp, n); }

/* fc_sync.cpp:90-94 */
int64_t fco_combined_length(int B, const int* cp, const fco_params* p) {
    return (int64_t)p->N_L + p->N_T + (int64_t)B * p->N + fco_cp_partial_sum(cp, B - 1);
}

/* fc_core.cpp:25-39 */
int fco_design_window(int L, int n_pass, int n_tb, double* w) {
    if (n_pass <= 0 || n_tb < 0 || n_pass + 2 * n_tb > L) return 1;
    for (int i = 0; i < L; ++i) w[i] = 0.0;
    const int lo = L / 2 - n_pass / 2;
    const int hi = lo + n_pass - 1;
    for (int i = lo; i <= hi; ++i) w[i] = 1.0;
    for (int k = 0; k < n_tb; ++k) {
        const double v = cos(kPi * (k + 1) / (2.0 * (n_tb + 1)));
        w[lo - 1 - k] = v * v;
        w[hi + 1 + k] = v * v;
    }
    return 0;
}

/* ofdm.cpp:80-95 */
int fco_centered_active_map(int l_ofdm, int n_active, int skip_dc, int* bins) {
    if (n_active <= 0 || n_active > l_ofdm - (skip_dc ? 1 : 0)) return 1;
    int k = 0;
    const int lo = n_active / 2;
    if (skip_dc) {
        const int hi = n_active - lo;
        for (int ls = -lo; ls <= -1; ++ls) bins[k++] = (ls + l_ofdm) % l_ofdm;
        for (int ls = 1; ls <= hi; ++ls) bins[k++] = ls;
    } else {
        for (int ls = -lo; ls < n_active - lo; ++ls) bins[k++] = (ls + l_ofdm) % l_ofdm;
    }
    return 0;
}

/* fc_core.cpp:41-44: exp(+j 2 pi ((r c mod L) L_S mod L) / L) */
void fco_block_phase(int64_t r, int c, int L_S, int L, double* re, double* im) {
    const int64_t num = mod64(mod64(r * c, L) * L_S, L);
    const double a = 2.0 * kPi * (double)num / L;
    *re = cos(a);
    *im = sin(a);
}

/* fc_sync.cpp:45-50: exp(+j 2 pi ((c mod N)(S_n mod N) mod N) / N) */
void fco_symbol_phase(int n, int c, const int* cp, int N, double* re, double* im) {
    const int64_t s = fco_cp_partial_sum(cp, n);
    const int64_t num = mod64(mod64(c, N) * mod64(s, N), N);
    const double a = 2.0 * kPi * (double)num / N;
    *re = cos(a);
    *im = sin(a);
}

/* fc_sync.cpp:34-43 */
int fco_zero_pad_symbol(const double* sym, int sym_len, const fco_params* p, int l_cp, double* z) {
    if (l_cp > p->L_L) return 1;
    if (sym_len != p->L + l_cp) return 1;
    const int s_l = p->L_L - l_cp;
    memset(z, 0, sizeof(double) * 2 * (size_t)(3 * p->L / 2));
    memcpy(z + 2 * s_l, sym, sizeof(double) * 2 * (size_t)sym_len);
    return 0;
}

/* fc_sync.cpp:52-58: passes [S_L, S_L + L_S + l_cp) */
int fco_first_block_window(const fco_params* p, int l_cp, double* a) {
    if (l_cp > p->L_L) return 1;
    const int s_l = p->L_L - l_cp;
    for (int i = 0; i < p->L; ++i) a[i] = (i >= s_l && i < s_l + p->L_S + l_cp) ? 1.0 : 0.0;
    return 0;
}

/* DFT definition of proj/src/fft.cpp:47-61 (FFTW forward/backward). */
void fco_fft(double* d, int n, int inverse) {
    if (n <= 1) return;
    for (int i = 1, j = 0; i < n; ++i) {
        int bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) {
            double t0 = d[2 * i], t1 = d[2 * i + 1];
            d[2 * i] = d[2 * j];
            d[2 * i + 1] = d[2 * j + 1];
            d[2 * j] = t0;
            d[2 * j + 1] = t1;
        }
    }
    const double sgn = inverse ? 1.0 : -1.0;
    for (int len = 2; len <= n; len <<= 1) {
        const int half = len >> 1;
        for (int k = 0; k < half; ++k) {
            const double a = 2.0 * kPi * (double)k / len;
            const double wr = cos(a), wi = sgn * sin(a);
            for (int s = 0; s < n; s += len) {
                double* x = d + 2 * (s + k);
                double* y = d + 2 * (s + k + half);
                const double br = y[0] * wr - y[1] * wi;
                const double bi = y[0] * wi + y[1] * wr;
                y[0] = x[0] - br;
                y[1] = x[1] - bi;
                x[0] += br;
                x[1] += bi;
            }
        }
    }
    if (inverse) {
        const double s = 1.0 / n;
        for (int i = 0; i < 2 * n; ++i) d[i] *= s;
    }
}

static double* zalloc(size_t ncomplex) { return (double*)calloc(ncomplex * 2 + 2, sizeof(double)); }

/* The subband bin map of synth_core / rx_block_freq (fc_core.cpp:80-84,
 * fc_sync.cpp:183-187): shifted index p0 in [0, L) sits on long-transform bin
 * q = (c - ceil(L/2) + p0) mod N and carries short-transform bin
 * b = (p0 + L/2) mod L. */
void fco_bin_map(int L, int c, int N, int* q, int* b) {
    const int half = (L + 1) / 2;
    for (int p0 = 0; p0 < L; ++p0) {
        b[p0] = (p0 + L / 2) % L;
        q[p0] = (int)mod64((int64_t)c - half + p0, N);
    }
}

/* rx_segment's window start (fc_sync.cpp:148): useful0 - N_L + sigma_n */
int64_t fco_rx_start(int64_t useful0, int N_L, int n, const int* cp, int N) {
    return useful0 - N_L + fco_symbol_sigma(n, cp, N);
}

/* fc_core.cpp:76-90 synth_core after the OLA analysis window
 * (sfb_block_ola, fc_core.cpp:115-124).  out: N complex. */
static void synth_block(const double* xw, int L, int c, const double* window, int N, double pr,
                        double pi, double* out) {
    double* X = zalloc((size_t)L);
    memcpy(X, xw, sizeof(double) * 2 * (size_t)L);
    fco_fft(X, L, 0);
    memset(out, 0, sizeof(double) * 2 * (size_t)N);
    int* qm = (int*)malloc(sizeof(int) * 2 * (size_t)L);
    fco_bin_map(L, c, N, qm, qm + L);
    for (int p0 = 0; p0 < L; ++p0) {
        const int b = qm[L + p0], q = qm[p0];
        const double wr = window[p0] * X[2 * b], wi = window[p0] * X[2 * b + 1];
        out[2 * q] = pr * wr - pi * wi;
        out[2 * q + 1] = pr * wi + pi * wr;
    }
    fco_fft(out, N, 1);
    free(qm);
    free(X);
}

/* fc_sync.cpp:60-84 (tx_symbol) with zero_pad_symbol :34-43 and
 * first_block_analysis_window :52-58. */
int fco_tx_symbol(const double* sym, int sym_len, int L, int c, const double* window,
                  const fco_params* p, const int* cp, int n, double* out3n2) {
    const int l_cp = sym_len - p->L;
    if (l_cp > p->L_L) return 1;
    if (l_cp < 0) return 1;
    const int N = p->N;
    const int s_l = p->L_L - l_cp;
    double* z = zalloc((size_t)(3 * L / 2));
    for (int i = 0; i < sym_len; ++i) {
        z[2 * (s_l + i)] = sym[2 * i];
        z[2 * (s_l + i) + 1] = sym[2 * i + 1];
    }
    double thr, thi;
    fco_symbol_phase(n, c, cp, N, &thr, &thi);
    const double scale = sqrt((double)p->I);
    double* xw = zalloc((size_t)L);
    double* blk = zalloc((size_t)N);
    memset(out3n2, 0, sizeof(double) * 2 * (size_t)(3 * N / 2));
    for (int r = 0; r < 2; ++r) {
        /* analysis windows: a0 passes [S_L, S_L+L_S+l_cp), a1 passes [L_L, L_L+L_S) */
        const int lo = r == 0 ? s_l : p->L_L;
        const int hi = r == 0 ? s_l + p->L_S + l_cp : p->L_L + p->L_S;
        for (int i = 0; i < L; ++i) {
            const int src = r * (L / 2) + i;
            const int keep = i >= lo && i < hi;
            xw[2 * i] = keep ? z[2 * src] : 0.0;
            xw[2 * i + 1] = keep ? z[2 * src + 1] : 0.0;
        }
        double br, bi;
        fco_block_phase(r, c, p->L_S, L, &br, &bi);
        const double pr = br * thr - bi * thi, pi = br * thi + bi * thr;
        synth_block(xw, L, c, window, N, pr, pi, blk);
        for (int t = 0; t < N; ++t) {
            out3n2[2 * (r * N / 2 + t)] += scale * blk[2 * t];
            out3n2[2 * (r * N / 2 + t) + 1] += scale * blk[2 * t + 1];
        }
    }
    free(z);
    free(xw);
    free(blk);
    return 0;
}

/* fc_sync.cpp:114-143 with ofdm_modulate (ofdm.cpp:97-106), cp_insert
 * (ofdm.cpp:108-116) and combine_symbols (fc_sync.cpp:96-112). */
int fco_tx_discontinuous(int N, double overlap, const int* cp, int B, int M, const int* Ls,
                         const int* cs, const double* windows, const double* grids, double* wave,
                         int64_t cap, int64_t* Q, int64_t* useful0) {
    if (M < 1 || B < 1) return 1;
    size_t woff = 0, goff = 0;
    int64_t q_len = -1;
    for (int m = 0; m < M; ++m) {
        const int L = Ls[m];
        fco_params p;
        if (fco_derive_params(N, L, overlap, &p)) return 1;
        const int64_t qm = fco_combined_length(B, cp, &p);
        if (m == 0) {
            q_len = qm;
            *useful0 = p.N_L;
            if (qm > cap) return 1;
            memset(wave, 0, sizeof(double) * 2 * (size_t)qm);
        } else if (qm != q_len || p.N_L != *useful0) {
            return 1;
        }
        double* x = zalloc((size_t)L);
        double* sym = zalloc((size_t)(2 * L));
        double* out = zalloc((size_t)(3 * N / 2));
        for (int n = 0; n < B; ++n) {
            int l_cp, ex;
            fco_cp_truncate(cp[n], p.I, &l_cp, &ex);
            if (l_cp < 0 || l_cp >= L) goto fail;
            memcpy(x, grids + 2 * (goff + (size_t)n * L), sizeof(double) * 2 * (size_t)L);
            fco_fft(x, L, 1);
            const double s = sqrt((double)L);
            for (int i = 0; i < 2 * L; ++i) x[i] *= s;
            for (int i = 0; i < l_cp; ++i) {
                sym[2 * i] = x[2 * (L - l_cp + i)];
                sym[2 * i + 1] = x[2 * (L - l_cp + i) + 1];
            }
            memcpy(sym + 2 * l_cp, x, sizeof(double) * 2 * (size_t)L);
            if (fco_tx_symbol(sym, L + l_cp, L, cs[m], windows + woff, &p, cp, n, out)) goto fail;
            const int64_t sigma = fco_symbol_sigma(n, cp, N);
            for (int t = 0; t < 3 * N / 2; ++t) {
                wave[2 * (sigma + t)] += out[2 * t];
                wave[2 * (sigma + t) + 1] += out[2 * t + 1];
            }
        }
        free(x);
        free(sym);
        free(out);
        woff += (size_t)L;
        goff += (size_t)B * L;
        continue;
    fail:
        free(x);
        free(sym);
        free(out);
        return 1;
    }
    *Q = q_len;
    return 0;
}

/* fc_sync.cpp:178-193 */
int fco_rx_block_freq(const double* y, int L, int c, const double* window, const fco_params* p,
                      double ph_re, double ph_im, double* g) {
    const int N = p->N;
    double* Y = zalloc((size_t)N);
    memcpy(Y, y, sizeof(double) * 2 * (size_t)N);
    fco_fft(Y, N, 0);
    int* qm = (int*)malloc(sizeof(int) * 2 * (size_t)L);
    fco_bin_map(L, c, N, qm, qm + L);
    for (int p0 = 0; p0 < L; ++p0) {
        const int b = qm[L + p0], q = qm[p0];
        const double vr = window[p0] * Y[2 * q], vi = window[p0] * Y[2 * q + 1];
        /* conj(phase) * v */
        g[2 * b] = ph_re * vr + ph_im * vi;
        g[2 * b + 1] = ph_re * vi - ph_im * vr;
    }
    free(qm);
    free(Y);
    return 0;
}

/* fc_core.cpp:94-111 analysis_core + fc_core.cpp:144-153 afb_block_ols
 * (synthesis_window_low = analysis_window, fc_core.cpp:57-69). */
static void afb_ols(const double* y, int L, int c, const double* window, const fco_params* p,
                    double pr, double pi, double* z) {
    fco_rx_block_freq(y, L, c, window, p, pr, pi, z);
    fco_fft(z, L, 1);
    const double s = (double)L / p->N;
    for (int i = 0; i < L; ++i) {
        const double keep = (i >= p->L_L && i < p->L_L + p->L_S) ? s : 0.0;
        z[2 * i] *= keep;
        z[2 * i + 1] *= keep;
    }
}

/* fc_sync.cpp:158-176 + ofdm_demodulate (ofdm.cpp:125-131) */
int fco_rx_symbol_direct(const double* y0, const double* y1, int L, int c, const double* window,
                         const fco_params* p, const int* cp, int n, double* out) {
    double thr, thi;
    fco_symbol_phase(n, c, cp, p->N, &thr, &thi);
    const double scale = sqrt((double)p->I);
    double* z = zalloc((size_t)L);
    for (int r = 0; r < 2; ++r) {
        double br, bi;
        fco_block_phase(r, c, p->L_S, L, &br, &bi);
        afb_ols(r == 0 ? y0 : y1, L, c, window, p, br * thr - bi * thi, br * thi + bi * thr, z);
        for (int i = 0; i < L / 2; ++i) {
            out[2 * (r * L / 2 + i)] = scale * z[2 * (L / 4 + i)];
            out[2 * (r * L / 2 + i) + 1] = scale * z[2 * (L / 4 + i) + 1];
        }
    }
    fco_fft(out, L, 0);
    const double s = 1.0 / sqrt((double)L);
    for (int i = 0; i < 2 * L; ++i) out[i] *= s;
    free(z);
    return 0;
}

/* diag(W_L^(phi q)), W_L = exp(-j 2 pi / L)  (fc_sync.cpp:204-213) */
static void omega(int phi, int L, double* v) {
    for (int q = 0; q < L; ++q) {
        const int64_t e = mod64((int64_t)phi * q, L);
        const double a = -2.0 * kPi * (double)e / L;
        const double cr = cos(a), ci = sin(a);
        const double vr = v[2 * q], vi = v[2 * q + 1];
        v[2 * q] = cr * vr - ci * vi;
        v[2 * q + 1] = cr * vi + ci * vr;
    }
}

/* fc_sync.cpp:195-243 (Eq. 30 transform decomposition) */
int fco_rx_symbol_simplified(const double* g0, const double* g1, const fco_params* p, double* out) {
    const int L = p->L;
    if (p->L_S * 2 != L) return 1;
    double* t = zalloc((size_t)L);
    double* f = zalloc((size_t)L);
    memcpy(t, g1, sizeof(double) * 2 * (size_t)L);
    omega(L / 2, L, t);
    for (int i = 0; i < 2 * L; ++i) f[i] = g0[i] - t[i];
    omega(-L / 4, L, f);
    fco_fft(f, L, 1);
    for (int i = 0; i < L; ++i) {
        /* S-hat[i] = s[(i + L/4) mod L], s = [0_{L_L} 1_{L_S} 0_{L_T}] */
        const int j = (i + L / 4) % L;
        const double sh = (j >= p->L_L && j < p->L_L + p->L_S) ? 1.0 : 0.0;
        f[2 * i] *= sh;
        f[2 * i + 1] *= sh;
    }
    fco_fft(f, L, 0);
    omega(L / 4, L, f);
    for (int i = 0; i < 2 * L; ++i) f[i] += t[i];
    omega(-L / 4, L, f);
    const double scale = sqrt((double)p->I) * ((double)p->L / p->N) / sqrt((double)L);
    for (int i = 0; i < 2 * L; ++i) out[i] = f[i] * scale;
    free(t);
    free(f);
    return 0;
}

/* fc_sync.cpp:245-264 with rx_segment :145-156 */
int fco_rx_discontinuous(const double* wave, int64_t len, int64_t useful0, int N, double overlap,
                         const int* cp, int B, int L, int c, const double* window, int simplified,
                         double* out) {
    fco_params p;
    if (fco_derive_params(N, L, overlap, &p)) return 1;
    double* g0 = zalloc((size_t)L);
    double* g1 = zalloc((size_t)L);
    int rc = 0;
    for (int n = 0; n < B; ++n) {
        const int64_t start = fco_rx_start(useful0, p.N_L, n, cp, N);
        if (start < 0 || start + 3 * N / 2 > len) {
            rc = 1;
            break;
        }
        const double* y0 = wave + 2 * start;
        const double* y1 = wave + 2 * (start + N / 2);
        double* o = out + 2 * (size_t)n * L;
        if (!simplified) {
            fco_rx_symbol_direct(y0, y1, L, c, window, &p, cp, n, o);
        } else {
            double thr, thi, br, bi;
            fco_symbol_phase(n, c, cp, N, &thr, &thi);
            fco_block_phase(0, c, p.L_S, L, &br, &bi);
            fco_rx_block_freq(y0, L, c, window, &p, br * thr - bi * thi, br * thi + bi * thr, g0);
            fco_block_phase(1, c, p.L_S, L, &br, &bi);
            fco_rx_block_freq(y1, L, c, window, &p, br * thr - bi * thi, br * thi + bi * thr, g1);
            if (fco_rx_symbol_simplified(g0, g1, &p, o)) {
                rc = 1;
                break;
            }
        }
    }
    free(g0);
    free(g1);
    return rc;
}

/* channel.cpp:19-24 */
uint64_t fco_splitmix64(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* channel.cpp:45-48 */
uint64_t fco_derive_seed(uint64_t seed, uint64_t index) {
    uint64_t s = seed ^ (0x9e3779b97f4a7c15ULL * (index + 1));
    return fco_splitmix64(&s);
}

/* ofdm.cpp:55-65 (Gray square QAM, unit average power), extended to k=8
 * (256-QAM, levels=16) with the same formulas. */
void fco_qam_map(int bits_per_symbol, unsigned symbol_bits, double* re, double* im) {
    const int k = bits_per_symbol / 2;
    const int levels = 1 << k;
    const unsigned mask = (1u << k) - 1u;
    unsigned bi = symbol_bits & mask, bq = (symbol_bits >> k) & mask;
    unsigned li = 0, lq = 0;
    for (unsigned g = bi; g; g >>= 1) li ^= g;
    for (unsigned g = bq; g; g >>= 1) lq ^= g;
    const double s = 1.0 / sqrt(2.0 * ((double)levels * levels - 1.0) / 3.0);
    *re = s * (2.0 * li + 1 - levels);
    *im = s * (2.0 * lq + 1 - levels);
}

/* scenario.cpp:110-128 bit drawing (one splitmix64 draw per bit, LSB first),
 * per-unit stream seeded with derive_seed(seed, unit).  Packed row order is
 * [B][A], i.e. symbol-major over the plan's active bins. */
void fco_gen_grid(uint64_t seed, int64_t unit0, int units, int B, int A, int bits_per_symbol,
                  double* packed) {
    for (int u = 0; u < units; ++u) {
        uint64_t st = fco_derive_seed(seed, (uint64_t)(unit0 + u));
        if (st == 0) st = 0x1234567890abcdefULL; /* GaussianRng ctor, channel.cpp:26 */
        double* dst = packed + 2 * (size_t)u * B * A;
        for (int64_t i = 0; i < (int64_t)B * A; ++i) {
            unsigned sym = 0;
            for (int b = 0; b < bits_per_symbol; ++b) sym |= (unsigned)(fco_splitmix64(&st) & 1u) << b;
            fco_qam_map(bits_per_symbol, sym, &dst[2 * i], &dst[2 * i + 1]);
        }
    }
}

/* ------------------------------------------------------------ link step (f1)
 * The step on either side of the path in the reference's link simulation
 * (scenario.cpp:469-494): hard-decision demap, bit errors and EVM sums.   */

/* ofdm.cpp:67-78 (qam_demap): per-axis slice with lround, clamp, Gray encode;
 * extended to k=4 (256-QAM) with the same formulas. */
unsigned fco_qam_demap(int bits_per_symbol, double re, double im) {
    const int k = bits_per_symbol / 2;
    const int levels = 1 << k;
    const double s = 1.0 / sqrt(2.0 * ((double)levels * levels - 1.0) / 3.0);
    unsigned out[2];
    const double v[2] = {re, im};
    for (int a = 0; a < 2; ++a) {
        /* static_cast<int>(std::lround(...)) as in the reference: the long
         * result is narrowed to int (modular) before the clamp */
        int idx = (int)lround((v[a] / s - 1.0 + levels) / 2.0);
        if (idx < 0) idx = 0;
        if (idx >= levels) idx = levels - 1;
        out[a] = (unsigned)idx ^ ((unsigned)idx >> 1);
    }
    return out[0] | (out[1] << k);
}

/* Per-unit link statistics of a received packed grid against the seeded
 * transmit grid of fco_gen_grid: EVM numerator/denominator sums
 * (metrics.cpp:115-127 evm_db, scenario.cpp:481-484) and bit errors of the
 * hard decisions (metrics.cpp:105-113 ber, scenario.cpp:486-491).  The
 * transmitted bits are re-drawn from the same splitmix64 streams.
 * out: per unit {evm_num, evm_den}; errs: per unit bit errors.  The sums run
 * in element order. */
void fco_link_stats(const double* rx, uint64_t seed, int64_t unit0, int units, int B, int A,
                    int bits_per_symbol, double* out, int64_t* errs) {
    for (int u = 0; u < units; ++u) {
        uint64_t st = fco_derive_seed(seed, (uint64_t)(unit0 + u));
        if (st == 0) st = 0x1234567890abcdefULL;
        const double* y = rx + 2 * (size_t)u * B * A;
        double num = 0.0, den = 0.0;
        int64_t e = 0;
        for (int64_t i = 0; i < (int64_t)B * A; ++i) {
            unsigned sym = 0;
            for (int b = 0; b < bits_per_symbol; ++b) sym |= (unsigned)(fco_splitmix64(&st) & 1u) << b;
            double xr, xi;
            fco_qam_map(bits_per_symbol, sym, &xr, &xi);
            const double dr = y[2 * i] - xr, di = y[2 * i + 1] - xi;
            num += dr * dr + di * di;
            den += xr * xr + xi * xi;
            const unsigned got = fco_qam_demap(bits_per_symbol, y[2 * i], y[2 * i + 1]);
            unsigned diff = got ^ sym;
            for (int b = 0; b < bits_per_symbol; ++b) e += (diff >> b) & 1u;
        }
        out[2 * u] = num;
        out[2 * u + 1] = den;
        errs[u] = e;
    }
}

/* channel.cpp:37-42 (GaussianRng::next_complex): two draws, Box-Muller with
 * variance 1/2 per axis. */
void fco_gauss_complex(uint64_t* state, double* re, double* im) {
    const double u1 = ((double)(fco_splitmix64(state) >> 11) + 1.0) * 0x1p-53;
    const double u2 = (double)(fco_splitmix64(state) >> 11) * 0x1p-53;
    const double r = sqrt(-log(u1));
    const double pi = 3.14159265358979323846;
    *re = r * cos(2.0 * pi * u2);
    *im = r * sin(2.0 * pi * u2);
}

/* channel.cpp:136-141 (awgn_with_variance): v += sqrt(sigma2) * n, one
 * GaussianRng(seed) stream over the samples in order. */
void fco_awgn(double* wave, int64_t len, double sigma2, uint64_t seed) {
    uint64_t st = seed ? seed : 0x1234567890abcdefULL;
    const double s = sqrt(sigma2);
    for (int64_t t = 0; t < len; ++t) {
        double nr, ni;
        fco_gauss_complex(&st, &nr, &ni);
        wave[2 * t] += s * nr;
        wave[2 * t + 1] += s * ni;
    }
}

/* channel.cpp:148-155 (measure_power): mean |v|^2 over [begin, end) clipped
 * to the waveform; -1 for an empty span (the reference throws). */
double fco_measure_power(const double* wave, int64_t len, int64_t begin, int64_t end) {
    if (begin < 0) begin = 0;
    if (end > len) end = len;
    if (end <= begin) return -1.0;
    double p = 0.0;
    for (int64_t t = begin; t < end; ++t) p += wave[2 * t] * wave[2 * t] + wave[2 * t + 1] * wave[2 * t + 1];
    return p / (double)(end - begin);
}

/* ------------------------------------------------ continuous FC (row f2) */

/* fc_core.cpp:155-161 */
int fco_continuous_block_count(int stream_len, const fco_params* p) {
    const int need = stream_len + p->L_O - p->L_L;
    return (need + p->L_S - 1) / p->L_S;
}

/* fc_core.cpp:163-198 tx_continuous: per subband, the stream is padded with
 * L_O leading zeros, cut into blocks hopping L_S, each block goes through
 * sfb_block_ola (analysis window, synth_core with block_phase(R)) and is
 * overlap-added at R*N_S scaled by sqrt(I); subbands are summed.
 * streams: concatenated per subband (lens[m] complex each).  Returns 1 on the
 * reference's invalid_argument cases; *out_len, *useful0 as the reference. */
int fco_tx_continuous(int N, double overlap, int M, const int* Ls, const int* cs, const double* windows,
                      const double* streams, const int64_t* lens, int l_cp0, double* wave, int64_t cap,
                      int64_t* out_len, int64_t* useful0) {
    if (M < 1) return 1;
    int64_t qlen = 0;
    size_t woff = 0, soff = 0;
    memset(wave, 0, sizeof(double) * 2 * (size_t)cap);
    for (int m = 0; m < M; ++m) {
        const int L = Ls[m];
        fco_params p;
        if (fco_derive_params(N, L, overlap, &p)) return 1;
        const int len = (int)lens[m];
        const int R_tot = fco_continuous_block_count(len, &p);
        const int64_t ol = (int64_t)(R_tot - 1) * p.N_S + p.N;
        if (ol > cap) return 2;
        if (ol > qlen) qlen = ol;
        const double scale = sqrt((double)p.I);
        double* xw = zalloc((size_t)L);
        double* blk = zalloc((size_t)N);
        for (int R = 0; R < R_tot; ++R) {
            /* padded[R L_S + i] = stream[R L_S + i - L_O]; a passes [L_L, L_L + L_S) */
            for (int i = 0; i < L; ++i) {
                const int64_t j = (int64_t)R * p.L_S + i - p.L_O;
                const int keep = i >= p.L_L && i < p.L_L + p.L_S && j >= 0 && j < len;
                xw[2 * i] = keep ? streams[2 * (soff + (size_t)j)] : 0.0;
                xw[2 * i + 1] = keep ? streams[2 * (soff + (size_t)j) + 1] : 0.0;
            }
            double pr, pi;
            fco_block_phase(R, cs[m], p.L_S, L, &pr, &pi);
            synth_block(xw, L, cs[m], windows + woff, N, pr, pi, blk);
            for (int t = 0; t < N; ++t) {
                wave[2 * ((int64_t)R * p.N_S + t)] += scale * blk[2 * t];
                wave[2 * ((int64_t)R * p.N_S + t) + 1] += scale * blk[2 * t + 1];
            }
        }
        if (m == 0) *useful0 = (int64_t)llround(overlap * N) + (int64_t)p.I * l_cp0;
        free(xw);
        free(blk);
        woff += (size_t)L;
        soff += (size_t)len;
    }
    *out_len = qlen;
    return 0;
}

/* fc_core.cpp:200-223 rx_continuous for one subband: the waveform is
 * prefixed with N_L zeros, blocks hop N_S, each goes through afb_block_ols
 * with block_phase(R) and the central L_S samples (x sqrt(I)) are kept.
 * out: R_tot * L_S complex (*n_out = that count). */
int fco_rx_continuous(const double* wave, int64_t len, int N, double overlap, int L, int c,
                      const double* window, double* out, int64_t cap, int64_t* n_out) {
    fco_params p;
    if (fco_derive_params(N, L, overlap, &p)) return 1;
    if (len < p.N) return 1;
    const int64_t nlow = (len + p.I - 1) / p.I + p.L;
    const int64_t R_tot = (nlow + p.L_S - 1) / p.L_S;
    if (R_tot * p.L_S > cap) return 2;
    const double scale = sqrt((double)p.I);
    double* y = zalloc((size_t)N);
    double* z = zalloc((size_t)L);
    for (int64_t R = 0; R < R_tot; ++R) {
        for (int t = 0; t < N; ++t) {
            const int64_t j = R * p.N_S + t - p.N_L;  /* x[N_L + t] = w[t] */
            const int in = j >= 0 && j < len;
            y[2 * t] = in ? wave[2 * j] : 0.0;
            y[2 * t + 1] = in ? wave[2 * j + 1] : 0.0;
        }
        double pr, pi;
        fco_block_phase(R, c, p.L_S, L, &pr, &pi);
        afb_ols(y, L, c, window, &p, pr, pi, z);
        for (int u = 0; u < p.L_S; ++u) {
            out[2 * (R * p.L_S + u)] = scale * z[2 * (p.L_L + u)];
            out[2 * (R * p.L_S + u) + 1] = scale * z[2 * (p.L_L + u) + 1];
        }
    }
    *n_out = R_tot * p.L_S;
    free(y);
    free(z);
    return 0;
}

/* ------------------------------------------------------ Welch PSD (row f4) */

/* metrics.cpp:128-155 (psd): Hann-windowed segments of seg_len hopping
 * lround(seg_len (1 - overlap)), |FFT|^2 accumulated, scaled by
 * 1 / (n_seg sum win^2).  Returns 1 for the reference's invalid_argument. */
int fco_psd(const double* x, int64_t len, int seg_len, double overlap_frac, double* out) {
    if (seg_len <= 0 || seg_len > len) return 1;
    if (overlap_frac < 0.0 || overlap_frac >= 1.0) return 1;
    long hop = lround(seg_len * (1.0 - overlap_frac));
    if (hop < 1) hop = 1;
    double* win = (double*)malloc(sizeof(double) * (size_t)seg_len);
    double wpow = 0.0;
    for (int i = 0; i < seg_len; ++i) {
        win[i] = 0.5 - 0.5 * cos(2.0 * kPi * i / seg_len);
        wpow += win[i] * win[i];
    }
    double* seg = zalloc((size_t)seg_len);
    for (int i = 0; i < seg_len; ++i) out[i] = 0.0;
    int n_seg = 0;
    for (int64_t start = 0; start + seg_len <= len; start += hop) {
        for (int i = 0; i < seg_len; ++i) {
            seg[2 * i] = x[2 * (start + i)] * win[i];
            seg[2 * i + 1] = x[2 * (start + i) + 1] * win[i];
        }
        fco_fft(seg, seg_len, 0);
        for (int i = 0; i < seg_len; ++i) out[i] += seg[2 * i] * seg[2 * i] + seg[2 * i + 1] * seg[2 * i + 1];
        ++n_seg;
    }
    const double scale = 1.0 / ((double)n_seg * wpow);
    for (int i = 0; i < seg_len; ++i) out[i] *= scale;
    free(win);
    free(seg);
    return 0;
}

/* ---------------------------------------------------- TDL channel (row f3) */

/* channel.cpp:101-111 draw_tdl: delays lround(delay_ns 1e-9 fs), gains
 * sqrt(power) * GaussianRng(seed).next_complex() per tap in order. */
void fco_draw_tdl(const double* delay_ns, const double* power_lin, int n_taps, double fs_hz, uint64_t seed,
                  int* delays, double* gains) {
    uint64_t st = seed ? seed : 0x1234567890abcdefULL;
    for (int k = 0; k < n_taps; ++k) {
        delays[k] = (int)lround(delay_ns[k] * 1e-9 * fs_hz);
        double nr, ni;
        fco_gauss_complex(&st, &nr, &ni);
        const double a = sqrt(power_lin[k]);
        gains[2 * k] = a * nr;
        gains[2 * k + 1] = a * ni;
    }
}

/* channel.cpp:113-124 apply_channel: out[t] = sum_k g_k w[t - d_k] (t >= d_k),
 * taps accumulated in tap order. */
void fco_apply_channel(const double* w, int64_t len, const int* delays, const double* gains, int n_taps,
                       double* out) {
    for (int64_t t = 0; t < 2 * len; ++t) out[t] = 0.0;
    for (int k = 0; k < n_taps; ++k) {
        const int64_t d = delays[k];
        const double gr = gains[2 * k], gi = gains[2 * k + 1];
        for (int64_t t = d; t < len; ++t) {
            const double xr = w[2 * (t - d)], xi = w[2 * (t - d) + 1];
            out[2 * t] += gr * xr - gi * xi;
            out[2 * t + 1] += gr * xi + gi * xr;
        }
    }
}
