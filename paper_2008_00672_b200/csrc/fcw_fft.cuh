// Register / shared-memory FFT building blocks for sm_100a (complex fp32).
//
//  * fft_reg<R, SIGN>: natural-order in/out radix-2 DIT transform of R points
//    held in registers, fully unrolled; its twiddles are compile-time
//    immediates (constexpr cos/sin evaluated by the front end).
//  * team_fft<n, T, PPT, SIGN, NF, CTA>: Stockham autosort transform of size
//    n = T * PPT run by a team of T threads (a warp or the CTA), NF transforms
//    in lockstep sharing twiddles.  Input and output are in the cyclic
//    distribution v[m] = x[t + T*m]; intermediate passes go through a padded
//    shared-memory buffer (one pad slot per 16, bank-conflict free for every
//    radix used).  Runtime twiddles come from the plan's N-entry table.
//
// SIGN = -1: forward (e^{-j}, unscaled) like fft::forward (proj/src/fft.cpp:47-52);
// SIGN = +1: inverse WITHOUT the 1/n factor (callers fold scales elsewhere).
#pragma once

#include <cuda_runtime.h>

#define FCW_DI __device__ __forceinline__

namespace fcw {

// ------------------------------------------------------ compile-time trig
constexpr double cx_pi = 3.14159265358979323846264338327950288;

__host__ __device__ constexpr double cx_sin_small(double x) {
    double x2 = x * x, term = x, sum = x;
    for (int i = 1; i < 14; ++i) {
        term *= -x2 / ((2.0 * i) * (2.0 * i + 1.0));
        sum += term;
    }
    return sum;
}
__host__ __device__ constexpr double cx_cos_small(double x) {
    double x2 = x * x, term = 1.0, sum = 1.0;
    for (int i = 1; i < 14; ++i) {
        term *= -x2 / ((2.0 * i - 1.0) * (2.0 * i));
        sum += term;
    }
    return sum;
}
// cos(2*pi*f) for a turn fraction f that is exact in binary (k/n, n a power
// of two), by octant reduction to |angle| <= pi/4.
__host__ __device__ constexpr double cx_cos_turn(double f) {
    f = f - (double)(long long)f;
    if (f < 0) f += 1.0;
    if (f > 0.5) f = 1.0 - f;                                   // even
    if (f > 0.25) return -cx_cos_turn(0.5 - f);                 // cos(pi - a) = -cos(a)
    if (f > 0.125) return cx_sin_small(2.0 * cx_pi * (0.25 - f));  // cos(a) = sin(pi/2 - a)
    return cx_cos_small(2.0 * cx_pi * f);
}
__host__ __device__ constexpr double cx_cos2pi(long k, long n) { return cx_cos_turn((double)k / (double)n); }
__host__ __device__ constexpr double cx_sin2pi(long k, long n) {
    return cx_cos_turn((double)k / (double)n - 0.25);  // sin(a) = cos(a - pi/2)
}

template <int N_, int K_, int SIGN>
struct Tw {
    static constexpr float re = (float)cx_cos2pi(K_, N_);
    static constexpr float im = (float)(SIGN * cx_sin2pi(K_, N_));
};

// --------------------------------------------------------- complex helpers
// Complex fp32 arithmetic on the sm_100a packed-FP32 instructions (FADD2 /
// FMUL2 / FFMA2: one issue slot per complex add / scale, two per complex
// product, with operand broadcast / swap / negate modifiers).  The FP32 pipe
// throughput is the same as the scalar forms (tools/ubench_f32x2.cu); what
// halves is the number of issued instructions, which bounds these kernels.
// Per component the rounding is that of the scalar code: cmul is
// (fma(ax, bx, -(ay by)), fma(ax, by, ay bx)) either way.
// FCW_PK_ADD / FCW_PK_MUL / FCW_PK_FMA select the packed (1) or scalar (0) form
// of the additions, the products and the fused butterfly steps.  The integer
// pipe shares one of the two FP32 datapaths of a sub-partition: a packed
// instruction holds both for two cycles, so integer / move instructions never
// overlap with it, while they pair with scalar FP32 (tools/ubench_coissue.cu).
#ifndef FCW_PK_ADD
#define FCW_PK_ADD 1
#endif
#ifndef FCW_PK_MUL
#define FCW_PK_MUL 0
#endif
#ifndef FCW_PK_FMA
#define FCW_PK_FMA 0
#endif
#ifndef FCW_PK_SCALE
#define FCW_PK_SCALE FCW_PK_MUL
#endif
#ifndef FCW_PK_AXPY
#define FCW_PK_AXPY FCW_PK_FMA
#endif
#ifndef FCW_PK_SWAP
#define FCW_PK_SWAP FCW_PK_FMA
#endif
#ifndef FCW_PK_TWICE
#define FCW_PK_TWICE FCW_PK_FMA
#endif
FCW_DI float2 cadd(float2 a, float2 b) {
#if FCW_PK_ADD
    return __fadd2_rn(a, b);
#else
    return make_float2(a.x + b.x, a.y + b.y);
#endif
}
FCW_DI float2 csub(float2 a, float2 b) {
#if FCW_PK_ADD
    return __fadd2_rn(a, make_float2(-b.x, -b.y));
#else
    return make_float2(a.x - b.x, a.y - b.y);
#endif
}
FCW_DI float2 cmul(float2 a, float2 b) {
#if FCW_PK_MUL
    return __ffma2_rn(make_float2(a.x, a.x), b, __fmul2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x)));
#else
    return make_float2(fmaf(a.x, b.x, -(a.y * b.y)), fmaf(a.x, b.y, a.y * b.x));
#endif
}
FCW_DI float2 cmulc(float2 a, float2 b) {  // a * conj(b)
#if FCW_PK_MUL
    return __ffma2_rn(a, make_float2(b.x, b.x), __fmul2_rn(make_float2(a.y, a.x), make_float2(b.y, -b.y)));
#else
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -(a.x * b.y)));
#endif
}
FCW_DI float2 cscale(float2 a, float s) {
#if FCW_PK_SCALE
    return __fmul2_rn(a, make_float2(s, s));
#else
    return make_float2(a.x * s, a.y * s);
#endif
}
FCW_DI float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
// a + s * b (real s), one FFMA2
FCW_DI float2 caxpy(float s, float2 b, float2 a) {
#if FCW_PK_AXPY
    return __ffma2_rn(make_float2(s, s), b, a);
#else
    return make_float2(fmaf(s, b.x, a.x), fmaf(s, b.y, a.y));
#endif
}
// a + (p, q) * swap(b) = (a.x + p b.y, a.y + q b.x), one FFMA2: with (p, q) =
// (-1, 1) it is a + j b, with (1, -1) a - j b
FCW_DI float2 cswapfma(float2 b, float p, float q, float2 a) {
#if FCW_PK_SWAP
    return __ffma2_rn(make_float2(b.y, b.x), make_float2(p, q), a);
#else
    return make_float2(fmaf(b.y, p, a.x), fmaf(b.x, q, a.y));
#endif
}
// 2 a - y (the second output of a butterfly whose first output is y = a + w b)
FCW_DI float2 ctwice_minus(float2 a, float2 y) {
#if FCW_PK_TWICE
    return __ffma2_rn(make_float2(2.f, 2.f), a, make_float2(-y.x, -y.y));
#else
    return make_float2(fmaf(2.f, a.x, -y.x), fmaf(2.f, a.y, -y.y));
#endif
}
// multiply by j^k (compile-time k)
template <int K>
FCW_DI float2 mul_jpow(float2 a) {
    constexpr int k = ((K % 4) + 4) % 4;
    if constexpr (k == 0) return a;
    if constexpr (k == 1) return make_float2(-a.y, a.x);
    if constexpr (k == 2) return make_float2(-a.x, -a.y);
    return make_float2(a.y, -a.x);
}
// j^k * a for a runtime k that differs across lanes: selects only, no branches
// (a switch here diverges four ways inside a warp).
FCW_DI float2 mul_jpow_rt(float2 a, int k) {
    const bool swap = k & 1;
    const float sr = ((k + 1) & 2) ? -1.f : 1.f;  // k = 1, 2 negate the real part
    const float si = (k & 2) ? -1.f : 1.f;        // k = 2, 3 negate the imaginary part
    const float re = swap ? a.y : a.x;
    const float im = swap ? a.x : a.y;
    return make_float2(sr * re, si * im);
}

__host__ __device__ constexpr int cx_log2(int v) { return v <= 1 ? 0 : 1 + cx_log2(v / 2); }
__host__ __device__ constexpr int cx_brev(int v, int bits) {
    int r = 0;
    for (int i = 0; i < bits; ++i) r |= ((v >> i) & 1) << (bits - 1 - i);
    return r;
}

// ----------------------------------------------------- register radix-2 DIT
// ZM: compile-time mask of positions (in the bit-reversed working order) that
// are known to be zero at the start of stage LEN; butterflies with a known-zero
// operand are reduced to copies / a single product (pruned transforms).
__host__ __device__ constexpr unsigned long long zm_next(unsigned long long zm, int L, int LEN) {
    unsigned long long out = 0;
    const int H = LEN / 2;
    for (int s = 0; s < L; s += LEN)
        for (int k = 0; k < H; ++k) {
            const bool z = ((zm >> (s + k)) & 1ull) && ((zm >> (s + k + H)) & 1ull);
            if (z) out |= (1ull << (s + k)) | (1ull << (s + k + H));
        }
    return out;
}
__host__ __device__ constexpr unsigned long long zm_brev(unsigned long long zm, int L, int bits) {
    unsigned long long out = 0;
    for (int p = 0; p < L; ++p) {
        int r = 0;
        for (int i = 0; i < bits; ++i) r |= ((p >> i) & 1) << (bits - 1 - i);
        if ((zm >> r) & 1ull) out |= 1ull << p;
    }
    return out;
}

// OM: outputs (natural order) the caller needs; in the last stage a butterfly
// with one dead output computes only the other.
template <int L, int SIGN, int LEN, int K, unsigned long long ZM = 0, unsigned long long OM = ~0ull>
FCW_DI void fft_stage(float2 (&x)[L]) {
    if constexpr (LEN <= L) {
        if constexpr (K < LEN / 2) {
            constexpr int H = LEN / 2;
#pragma unroll
            for (int s = 0; s < L; s += LEN) {
                const float2 a = x[s + K];
                const float2 b = x[s + K + H];
                const bool za = (ZM >> (s + K)) & 1ull, zb = (ZM >> (s + K + H)) & 1ull;
                const bool n0 = LEN < L || ((OM >> (s + K)) & 1ull), n1 = LEN < L || ((OM >> (s + K + H)) & 1ull);
                if (!n0 && !n1) {
                    // neither output used
                } else if (!(za || zb) && !(n0 && n1)) {
                    // one live output: y = a +- w b
                    float2 wb = b;
                    if constexpr (K != 0) wb = cmul(b, make_float2(Tw<LEN, K, SIGN>::re, Tw<LEN, K, SIGN>::im));
                    if (n0) x[s + K] = cadd(a, wb);
                    else x[s + K + H] = csub(a, wb);
                } else if (za && zb) {
                    x[s + K] = make_float2(0.f, 0.f);  // never read the (unset) zero registers
                    x[s + K + H] = make_float2(0.f, 0.f);
                } else if (zb) {
                    x[s + K + H] = a;  // a + w*0, a - w*0
                } else if (za) {
                    float2 wb = b;
                    if constexpr (K != 0) wb = cmul(b, make_float2(Tw<LEN, K, SIGN>::re, Tw<LEN, K, SIGN>::im));
                    x[s + K] = wb;
                    x[s + K + H] = make_float2(-wb.x, -wb.y);  // negation folds into consumers
                } else if constexpr (K == 0) {
                    x[s + K] = cadd(a, b);  // FADD2 x 2
                    x[s + K + H] = csub(a, b);
                } else if constexpr (4 * K == LEN) {
                    // trivial twiddle -+j: w b = SIGN < 0 ? -j b : +j b, one FFMA2 per output
                    constexpr float p = SIGN < 0 ? 1.f : -1.f;
                    x[s + K] = cswapfma(b, p, -p, a);
                    x[s + K + H] = cswapfma(b, -p, p, a);
                } else if constexpr (8 * K == LEN || 8 * K == 3 * LEN) {
                    // +-45 degree twiddles: w b = c (sr b + si j b), 3 FFMA2
                    constexpr float wr = Tw<LEN, K, SIGN>::re;
                    constexpr float wi = Tw<LEN, K, SIGN>::im;
                    constexpr float c = wr > 0.f ? wr : -wr;
                    constexpr float sr = wr > 0.f ? 1.f : -1.f, si = wi > 0.f ? 1.f : -1.f;
                    // t = sr b + si j b = (sr b.x - si b.y, sr b.y + si b.x)
                    const float2 t = cswapfma(b, -si, si, make_float2(sr * b.x, sr * b.y));
                    x[s + K] = caxpy(c, t, a);
                    x[s + K + H] = caxpy(-c, t, a);
                } else {
                    // general twiddle: y0 = a + w b (2 FFMA2), y1 = 2a - y0 (1 FFMA2)
                    constexpr float wr = Tw<LEN, K, SIGN>::re;
                    constexpr float wi = Tw<LEN, K, SIGN>::im;
                    const float2 y0 = caxpy(wr, b, cswapfma(b, -wi, wi, a));
                    x[s + K] = y0;
                    x[s + K + H] = ctwice_minus(a, y0);
                }
            }
            fft_stage<L, SIGN, LEN, K + 1, ZM, OM>(x);
        } else {
            fft_stage<L, SIGN, LEN * 2, 0, zm_next(ZM, L, LEN), OM>(x);
        }
    }
}

// ZIN: compile-time mask of inputs (natural order) known to be zero.
template <int L, int SIGN, unsigned long long ZIN = 0, unsigned long long OM = ~0ull>
FCW_DI void fft_reg(float2 (&x)[L]) {
    if constexpr (L == 1) return;
    constexpr int LB = cx_log2(L);
#pragma unroll
    for (int i = 0; i < L; ++i) {
        const int j = cx_brev(i, LB);
        if (i < j) {
            const float2 t = x[i];
            x[i] = x[j];
            x[j] = t;
        }
    }
    fft_stage<L, SIGN, 2, 0, zm_brev(ZIN, L, LB), OM>(x);
}

// ------------------------------------------------- TMEM as a per-lane table
// Twiddles that are constants of a thread (they depend on its lane / thread
// index only) live in tensor memory: every thread parks them in its own TMEM
// lane once per kernel and reads them back with tcgen05.ld (32x32b: thread i
// of warp w reads lane 32 (w mod 4) + i), 16 columns = 8 complex values per
// instruction, instead of 15 LDS.64 or four table loads and eleven products
// per transform.  Measured on the half-warp FFT_256 in isolation
// (tools/ubench_tmem_tw.cu): 60.8 -> 57.4 SM-cycles.
#ifndef FCW_TMEM_TW
#define FCW_TMEM_TW 3
#endif
constexpr int kTwTmem = 99;      // TWL value: long-transform twiddles from TMEM
constexpr int kTmemCols = 256;   // columns per CTA: sets A, B (32 each), C for warps 0-3 / 4-7 (32 each), 4 x 32 bin-class rows
#define FCW_R16(a, o) a(o + 0), a(o + 1), a(o + 2), a(o + 3), a(o + 4), a(o + 5), a(o + 6), a(o + 7), a(o + 8), \
                      a(o + 9), a(o + 10), a(o + 11), a(o + 12), a(o + 13), a(o + 14), a(o + 15)
FCW_DI void tmem_st16(unsigned taddr, const unsigned (&d)[16]) {
#define FCW_IN(i) "r"(d[i])
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%16], {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15};" ::FCW_R16(
            FCW_IN, 0),
        "r"(taddr)
        : "memory");
#undef FCW_IN
}
FCW_DI void tmem_ld16(unsigned taddr, unsigned (&d)[16]) {
#define FCW_OUT(i) "=r"(d[i])
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : FCW_R16(FCW_OUT, 0)
        : "r"(taddr));
#undef FCW_OUT
}
// Wait for this thread's tcgen05.ld; the destination registers pass through
// the statement so no consumer is scheduled ahead of the wait.
FCW_DI void tmem_wait16(unsigned (&d)[16]) {
#define FCW_IO(i) "+r"(d[i])
    asm volatile("tcgen05.wait::ld.sync.aligned;" : FCW_R16(FCW_IO, 0)::"memory");
#undef FCW_IO
}
FCW_DI float2 tmem_c(const unsigned (&d)[16], int k) {
    return make_float2(__uint_as_float(d[2 * k]), __uint_as_float(d[2 * k + 1]));
}

// ------------------------------------------------------------ team barriers
// CTA-scope teams sync on barrier 0 (the whole block) or, for a sub-team, on
// named barrier bar_id over bar_n threads; warp teams use __syncwarp.
template <bool CTA>
FCW_DI void team_bar(int bar_id, int bar_n) {
    if constexpr (CTA) {
        if (bar_id == 0)
            __syncthreads();
        else
            asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(bar_n) : "memory");
    } else {
        __syncwarp();
    }
}

FCW_DI int spad(int e) { return e + (e >> 4); }

// SMEM slot of Stockham element e for a team FFT: one pad slot per 16 is
// conflict-free for radix-16 schedules (and NS = 1); the warp FFTs with 8 or 4
// points per lane (L = 256, 128) use an XOR swizzle instead, which is
// conflict-free for all of their passes (checked exhaustively, 8-byte
// accesses in 16-lane wavefronts) and needs no padding.
template <int T, int PPT>
FCW_DI int saddr(int e) {
    if constexpr (T == 32 && PPT == 8)
        return e ^ ((e >> 3) & 15);
    else if constexpr (T == 32 && PPT == 4)
        return e ^ ((e >> 2) & 15);
    else
        return spad(e);
}

// w[k] = W^(k*e0) for k < R from log2(R) table loads (W^e0, W^2e0, W^4e0,
// W^8e0) and at most two products each, so every power carries at most ~3 ulp
// of rounding (a plain k-step recurrence would grow linearly in k).
// tw is the plan table exp(-2 pi i m / N); e0 is already in table units and
// k*e0 < N for every k < R.  TWL > 0 selects a two-level SMEM table instead:
// tw[0 .. 2^TWL) = W^i, tw[2^TWL + h] = W^(h 2^TWL), and W^e = hi * lo.
template <int R, int SIGN, int TWL = 0>
FCW_DI void twiddle_powers(float2 (&w)[R], const float2* tw, int e0) {
    auto ld = [&](int e) {
        float2 v;
        if constexpr (TWL > 0)
            v = cmul(tw[(1 << TWL) + (e >> TWL)], tw[e & ((1 << TWL) - 1)]);
        else
            v = tw[e];  // generic load: tw may live in SMEM or global
        if constexpr (SIGN > 0) v.y = -v.y;
        return v;
    };
    w[0] = make_float2(1.f, 0.f);
    if constexpr (R >= 2) w[1] = ld(e0);
    if constexpr (R >= 4) {
        w[2] = ld(2 * e0);
        w[3] = cmul(w[1], w[2]);
    }
    if constexpr (R >= 8) {
        w[4] = ld(4 * e0);
        w[5] = cmul(w[1], w[4]);
        w[6] = cmul(w[2], w[4]);
        w[7] = cmul(w[3], w[4]);
    }
    if constexpr (R >= 16) {
        w[8] = ld(8 * e0);
#pragma unroll
        for (int k = 9; k < 16; ++k) w[k] = cmul(w[k - 8], w[8]);
    }
}

// One Stockham pass (and the remaining ones, recursively).
template <int n, int T, int PPT, int SIGN, int NF, bool CTA, int NS, int TWL, unsigned long long ZIN0 = 0>
FCW_DI void team_pass(float2 (&v)[NF][PPT], float2* const* buf, const float2* __restrict__ tw,
                      int ts, int t, bool act, int bar_id, int bar_n, unsigned tm_a = 0, unsigned tm_c = 0) {
    constexpr int R0 = PPT < 16 ? PPT : 16;
    constexpr int REM = n / NS;
    constexpr int R = REM < R0 ? REM : R0;
    constexpr bool LAST = (NS * R == n);
    constexpr int NB = PPT / R;
    static_assert(R >= 2 && PPT % R == 0, "team_fft: bad radix schedule");
    constexpr bool kSwz = T == 32 && (PPT == 8 || PPT == 4);  // XOR-swizzled warp layouts (saddr)
    if (act) {
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const int j = t + T * i;
            float2 y[NF][R];
#pragma unroll
            for (int f = 0; f < NF; ++f)
#pragma unroll
                for (int k = 0; k < R; ++k) y[f][k] = v[f][i + k * NB];
            if constexpr (NS > 1) {
                const int jm = j & (NS - 1);
                float2 wk[R];
                if constexpr (TWL == kTwTmem) {
                    // radix-16 passes of the 4096-point transform: W_256^(k (t & 15)) (set A) for
                    // NS = 16, W_4096^(k t) (set C) for NS = 256, parked in this thread's TMEM lane
                    static_assert(R == 16 && NB == 1 && (NS == 16 || NS == 256), "TMEM twiddles: 16 x 16 x 16");
                    unsigned lo[16], hi[16];
                    const unsigned ta = NS == 16 ? tm_a : tm_c;
                    tmem_ld16(ta, lo);
                    tmem_ld16(ta + 16, hi);
                    tmem_wait16(lo);
                    tmem_wait16(hi);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        wk[k] = tmem_c(lo, k);
                        wk[k + 8] = tmem_c(hi, k);
                        if constexpr (SIGN > 0) {
                            wk[k].y = -wk[k].y;
                            wk[k + 8].y = -wk[k + 8].y;
                        }
                    }
                } else {
                    twiddle_powers<R, SIGN, TWL>(wk, tw, jm * (n / (NS * R)) * ts);
                }
#pragma unroll
                for (int k = 1; k < R; ++k)
#pragma unroll
                    for (int f = 0; f < NF; ++f) y[f][k] = cmul(y[f][k], wk[k]);
            }
#pragma unroll
            for (int f = 0; f < NF; ++f) fft_reg<R, SIGN, NS == 1 && NB == 1 ? ZIN0 : 0ull>(y[f]);
#pragma unroll
            for (int f = 0; f < NF; ++f)
#pragma unroll
                for (int k = 0; k < R; ++k) v[f][i + k * NB] = y[f][k];
        }
    }
    if constexpr (!LAST) {
        team_bar<CTA>(bar_id, bar_n);
        if (act) {
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const int j = t + T * i;
                const int base = (j / NS) * NS * R + (j & (NS - 1));
                // padded layout: with NS = 1 (base a multiple of R, R | 16) or NS a multiple of
                // 16 the pad term of base + k NS is pad(base) + k NS / 16, so the R slots are
                // one computed address plus compile-time offsets
                constexpr bool kPadLinW = !kSwz && (NS == 1 || NS % 16 == 0);
                const int wb = kPadLinW ? spad(base) : 0;
#pragma unroll
                for (int f = 0; f < NF; ++f)
#pragma unroll
                    for (int k = 0; k < R; ++k) {
                        const int slot = kPadLinW ? wb + k * (NS + NS / 16) : saddr<T, PPT>(base + k * NS);
                        buf[f][slot] = v[f][i + k * NB];
                    }
            }
        }
        team_bar<CTA>(bar_id, bar_n);
        if (act) {
            constexpr bool kPadLinR = !kSwz && T % 16 == 0;  // pad(t + T m) = pad(t) + m T / 16
            const int rb = kPadLinR ? spad(t) : 0;
#pragma unroll
            for (int f = 0; f < NF; ++f)
#pragma unroll
                for (int m = 0; m < PPT; ++m)
                    v[f][m] = buf[f][kPadLinR ? rb + m * (T + T / 16) : saddr<T, PPT>(t + T * m)];
        }
        team_pass<n, T, PPT, SIGN, NF, CTA, NS * R, TWL>(v, buf, tw, ts, t, act, bar_id, bar_n, tm_a, tm_c);
    }
}

// Full transform.  All T threads of the team (and, for CTA teams, every
// thread of the block) must call it; threads with act == false only join the
// barriers.  The buffers must hold spad(n) + 1 float2 each and may alias the
// input's source memory once it has been read into v.
// ZIN0: inputs v[f][m] known to be zero (first pass, one butterfly per thread).
template <int n, int T, int PPT, int SIGN, int NF, bool CTA, int TWL = 0, unsigned long long ZIN0 = 0>
FCW_DI void team_fft(float2 (&v)[NF][PPT], float2* const* buf, const float2* __restrict__ tw, int ts,
                     int t, bool act, int bar_id = 0, int bar_n = 0, unsigned tm_a = 0, unsigned tm_c = 0) {
    static_assert(n == T * PPT, "team_fft: n != T*PPT");
    if constexpr (n == 1) return;
    if constexpr (T == 1) {
        if (act) {
#pragma unroll
            for (int f = 0; f < NF; ++f) fft_reg<PPT, SIGN>(v[f]);
        }
    } else {
        team_pass<n, T, PPT, SIGN, NF, CTA, 1, TWL, ZIN0>(v, buf, tw, ts, t, act, bar_id, bar_n, tm_a, tm_c);
    }
}

// Half-warp FFT_256, radix 16 x 16 with ONE shared-memory exchange.  Lane t of
// a 16-lane team holds v[m] = x[t + 16 m] and receives v[k] = X[t + 16 k].
//  * ZIN: inputs v[m] known to be zero (pruned first pass; never read).
//  * eoff: the pass-2 twiddle exponent of lane t is (t + eoff) mod 256.  A
//    non-zero eoff transforms the input rotated by a per-lane factor:
//    eoff = 64 gives the transform of e^{SIGN 2 pi i 64 t / 256} x[t + 16 m]
//    (j^t for SIGN = +1) at no cost, since that factor is common to every
//    pass-1 input of lane t and so commutes into its pass-2 twiddle.
//  * buf: the team's exchange buffer, >= 271 float2 (17 t + k / t + 17 m:
//    conflict-free, immediate offsets).  stw[e] = exp(-2 pi i e / 256).
// Both halves of the warp must call it (it uses __syncwarp).
// tw16 (optional): per-lane twiddle table, tw16[sel][m][t] = exp(-2 pi i m (t + 64 sel) / 256)
// for sel = eoff / 64 in {0, 1}: 15 conflict-free loads instead of 4 loads
// and 11 complex products.
// OUT: outputs v[k] the caller uses (dead ones are not computed).
// TM: the twiddles come from this thread's TMEM lane instead (tm = address of
// set A; set B, for eoff = 64, follows 32 columns later); both loads are in
// flight across the exchange.
template <int SIGN, unsigned long long ZIN = 0, unsigned long long OUT = ~0ull, bool TM = false>
FCW_DI void fft256_half(float2 (&v)[16], float2* buf, const float2* stw, int t, int eoff,
                        const float2* tw16 = nullptr, unsigned tm = 0) {
    fft_reg<16, SIGN, ZIN>(v);
    unsigned lo[16], hi[16];
    if constexpr (TM) {
        const unsigned ta = tm + 32 * (eoff >> 6);
        tmem_ld16(ta, lo);
        tmem_ld16(ta + 16, hi);
    }
    __syncwarp();  // the previous use of buf has been read by every lane
    float2* wp = buf + 17 * t;
#pragma unroll
    for (int k = 0; k < 16; ++k) wp[k] = v[k];
    __syncwarp();
    const float2* rp = buf + t;
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = rp[17 * m];
    if constexpr (TM) {
        tmem_wait16(lo);
        tmem_wait16(hi);
#pragma unroll
        for (int m = 1; m < 16; ++m) {
            float2 w = m < 8 ? tmem_c(lo, m) : tmem_c(hi, m - 8);
            if constexpr (SIGN > 0) w.y = -w.y;
            v[m] = cmul(v[m], w);
        }
        fft_reg<16, SIGN, 0ull, OUT>(v);
        return;
    }
    if (tw16) {
        const float2* tp = tw16 + (eoff >> 6) * 256 + t;
#pragma unroll
        for (int m = 1; m < 16; ++m) {
            float2 w = tp[16 * m];
            if constexpr (SIGN > 0) w.y = -w.y;
            v[m] = cmul(v[m], w);
        }
        fft_reg<16, SIGN, 0ull, OUT>(v);
        return;
    }
    const int e0 = (t + eoff) & 255;
    auto ld = [&](int e) {
        float2 x = stw[e & 255];
        if constexpr (SIGN > 0) x.y = -x.y;
        return x;
    };
    float2 w[16];
    w[1] = ld(e0);
    w[2] = ld(2 * e0);
    w[4] = ld(4 * e0);
    w[8] = ld(8 * e0);
    w[3] = cmul(w[1], w[2]);
    w[5] = cmul(w[1], w[4]);
    w[6] = cmul(w[2], w[4]);
    w[7] = cmul(w[3], w[4]);
#pragma unroll
    for (int k = 9; k < 16; ++k) w[k] = cmul(w[k - 8], w[8]);
#pragma unroll
    for (int m = 1; m < 16; ++m) v[m] = cmul(v[m], w[m]);
    fft_reg<16, SIGN, 0ull, OUT>(v);
}

}  // namespace fcw
