/*
 * TEST INFRASTRUCTURE ONLY — see fftw3.h.
 *
 * DFT of length n: out[k] = sum_j in[j] * exp(sign * 2*pi*i*j*k/n), unscaled
 * (FFTW's documented definition).  Power-of-two n runs an iterative radix-2
 * decimation-in-time transform with double-precision twiddles computed from
 * exactly reduced integer angles; any other n falls back to the direct sum.
 */
#include "fftw3.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

struct fcw_shim_plan_s {
    int n;
    int sign;
    int log2n; /* -1 when n is not a power of two */
    double* tw; /* n/2 complex twiddles exp(sign*2*pi*i*k/n) (pow2) or n (direct) */
    fftw_complex* in;
    fftw_complex* out;
};

static const double kTwoPi = 6.283185307179586476925286766559;

static int ilog2_exact(int n) {
    int l = 0;
    if (n <= 0 || (n & (n - 1)) != 0) return -1;
    while ((1 << l) < n) ++l;
    return l;
}

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags) {
    (void)flags;
    if (n <= 0) return NULL;
    fftw_plan p = (fftw_plan)calloc(1, sizeof(*p));
    if (!p) return NULL;
    p->n = n;
    p->sign = sign < 0 ? -1 : 1;
    p->log2n = ilog2_exact(n);
    p->in = in;
    p->out = out;
    const int ntw = p->log2n >= 0 ? (n / 2 > 0 ? n / 2 : 1) : n;
    p->tw = (double*)malloc(sizeof(double) * 2 * (size_t)ntw);
    if (!p->tw) {
        free(p);
        return NULL;
    }
    for (int k = 0; k < ntw; ++k) {
        const double a = kTwoPi * (double)k / (double)n;
        p->tw[2 * k] = cos(a);
        p->tw[2 * k + 1] = p->sign * sin(a);
    }
    return p;
}

static void run_pow2(const fftw_plan p, double* d) {
    const int n = p->n;
    /* bit-reversal permutation */
    for (int i = 1, j = 0; i < n; ++i) {
        int bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) {
            double tr = d[2 * i], ti = d[2 * i + 1];
            d[2 * i] = d[2 * j];
            d[2 * i + 1] = d[2 * j + 1];
            d[2 * j] = tr;
            d[2 * j + 1] = ti;
        }
    }
    for (int len = 2; len <= n; len <<= 1) {
        const int half = len >> 1;
        const int step = n / len;
        for (int s = 0; s < n; s += len) {
            for (int k = 0; k < half; ++k) {
                const double wr = p->tw[2 * (k * step)], wi = p->tw[2 * (k * step) + 1];
                double* a = d + 2 * (s + k);
                double* b = d + 2 * (s + k + half);
                const double br = b[0] * wr - b[1] * wi;
                const double bi = b[0] * wi + b[1] * wr;
                b[0] = a[0] - br;
                b[1] = a[1] - bi;
                a[0] += br;
                a[1] += bi;
            }
        }
    }
}

static void run_direct(const fftw_plan p, const double* src, double* dst) {
    const int n = p->n;
    for (int k = 0; k < n; ++k) {
        double ar = 0.0, ai = 0.0;
        for (int j = 0; j < n; ++j) {
            const int e = (int)(((long long)j * k) % n);
            const double wr = p->tw[2 * e], wi = p->tw[2 * e + 1];
            ar += src[2 * j] * wr - src[2 * j + 1] * wi;
            ai += src[2 * j] * wi + src[2 * j + 1] * wr;
        }
        dst[2 * k] = ar;
        dst[2 * k + 1] = ai;
    }
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    if (!p) return;
    const size_t bytes = sizeof(double) * 2 * (size_t)p->n;
    if (p->log2n >= 0) {
        if (out != in) memcpy(out, in, bytes);
        run_pow2(p, (double*)out);
    } else {
        double* tmp = (double*)malloc(bytes);
        if (!tmp) return;
        run_direct(p, (const double*)in, tmp);
        memcpy(out, tmp, bytes);
        free(tmp);
    }
}

void fftw_execute(const fftw_plan p) {
    if (p) fftw_execute_dft(p, p->in, p->out);
}

void fftw_destroy_plan(fftw_plan p) {
    if (!p) return;
    free(p->tw);
    free(p);
}
