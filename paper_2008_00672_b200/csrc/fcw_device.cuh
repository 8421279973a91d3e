// sm_100a kernels of the symbol-synchronized FC-F-OFDM hot path (templates;
// instantiated per long-transform size N in fcw_k_*.cu).
//
//  K-TX  tx_kernel<N, LU>: fused TX synthesis (replaces tx_discontinuous,
//        proj/src/fc_sync.cpp:114-143 and everything under it:
//        ofdm_modulate ofdm.cpp:97, cp_insert :108, zero_pad_symbol
//        fc_sync.cpp:34, tx_symbol :60, sfb_block_ola/synth_core
//        fc_core.cpp:115,76, combine_symbols fc_sync.cpp:96, subband sum :139).
//  K-RX  rx_kernel<N, LU>: fused RX analysis for all subbands (replaces
//        rx_discontinuous fc_sync.cpp:245 with rx_segment :145, rx_block_freq
//        :178, rx_symbol_simplified :195 / rx_symbol_direct :158 +
//        afb_block_ols fc_core.cpp:144 + ofdm_demodulate ofdm.cpp:125).
//  LU = the plan's uniform short-transform size (specialised, 2 CTAs/SM), or
//  0 for plans mixing several L (generic: one branch per L group).
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
#pragma once

#include "fcw_fft.cuh"
#include "fcw_internal.hpp"

namespace fcw {

constexpr int kPPT = 16;  // long-transform points per thread and block

// Dev-only stage-timing knob (FCW_DEBUG_SKIP, bit 1: short stage, bit 2: long
// transform).  Compiled out of the release library (FCW_DEV_KNOBS=0): the
// product kernels always run every stage.
#ifndef FCW_DEV_KNOBS
#define FCW_DEV_KNOBS 0
#endif
#define FCW_SKIP(P, bit) (FCW_DEV_KNOBS && ((P).dbg_skip & (bit)))

// Bounds checks of every computed SMEM / global index on the hot path
// (the `check` library variant, tools/checked_run.sh; compute-sanitizer is
// not available on the GPU pool).  A failed check traps the kernel.
#ifndef FCW_CHECK
#define FCW_CHECK 0
#endif
#define FCW_ASSERT(c)                        \
    do {                                     \
        if (FCW_CHECK && !(c)) __trap();     \
    } while (0)

// Bin-class entry (plan, per class and DFT bin b), 8 bytes:
//   x = (inv[b] & 0xffff) | sec(p0) << 16, y = bits(w[p0]), p0 = b ^ L/2;
//   sec = -2: zero weight (no contribution), -1: primary (spectrum slot q),
//   >= 0: extension slot N + ext_base + sec of a shared transition bin.
struct Bin {
    int inv, dest;
    float w;
};
template <int N, int L>
FCW_DI Bin bin_entry(const KParams& P, const SubDev& sd, int b) {
    const int2 e = __ldg(&P.cls[sd.cls_off + b]);
    const int sec = e.x >> 16;
    const int q = (sd.c - L / 2 + (b ^ (L / 2))) & (N - 1);
    return Bin{(int)(short)(e.x & 0xffff), sec >= 0 ? N + sd.ext_base + sec : (sec == -1 ? q : -1),
               __int_as_float(e.y)};
}

// Decoded class entry for warp-path lane element b = lane + 32k (L >= 64):
// flipping bit L/2 of b only touches k, so the primary slot is qbase + 32 k'.
template <int I>
struct IC {
    static constexpr int value = I;
};
template <int Nn, int I = 0, class F>
FCW_DI void static_for(F&& f) {
    if constexpr (I < Nn) {
        f(IC<I>{});
        static_for<Nn, I + 1>(f);
    }
}

struct BinW {
    int inv;   // active index or -1
    int dest;  // spectrum slot or -1
    float w;
};
template <int N, int L, int K>
FCW_DI BinW bin_warp(const int2 e, int qbase, int ext0) {
    constexpr int KP = K ^ (L / 64);  // (lane + 32K) ^ (L/2) == lane + 32*KP
    const int sec = e.x >> 16;
    const int q = (qbase + 32 * KP) & (N - 1);
    return BinW{(int)(short)(e.x & 0xffff), sec >= 0 ? ext0 + sec : (sec == -1 ? q : -1), __int_as_float(e.y)};
}

// Bulk L2 prefetch of [p, p + bytes) by one thread (cp.async.bulk, sm_90+):
// the next symbol's input is on its way from HBM while this one computes.
FCW_DI void prefetch_l2(const void* p, long long bytes) {
    // the instruction takes a .global-space address, not a generic one
    const unsigned long long g = static_cast<unsigned long long>(__cvta_generic_to_global(p));
    unsigned long long a = g & ~15ull;
    const unsigned long long e = (g + (unsigned long long)bytes + 15ull) & ~15ull;
    while (a < e) {
        const unsigned chunk = (e - a) > (1ull << 20) ? (1u << 20) : (unsigned)(e - a);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(chunk) : "memory");
        a += chunk;
    }
}

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

// spec[slot] = v under a predicate, as ONE predicated st.shared (no branch around the store and
// the products that feed it); sbase = the spectrum's shared-space byte address.
FCW_DI void sts_if(unsigned sbase, int slot, float2 v, bool pred) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t@p st.shared.v2.f32 [%0], {%1, %2};\n\t}" ::"r"(
            sbase + 8u * (unsigned)slot),
        "f"(v.x), "f"(v.y), "r"(0), "r"((int)pred)
        : "memory");
}

// Predicated global stores as single instructions (no branch around the store and the
// arithmetic that feeds it): streaming (.cs), plain, and the L2 reduction.
FCW_DI void stcs_if(float2* p, float2 v, bool pred) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t@p st.global.cs.v2.f32 [%0], {%1, %2};\n\t}" ::"l"(p),
                 "f"(v.x), "f"(v.y), "r"((int)pred)
                 : "memory");
}
FCW_DI void stg_if(float2* p, float2 v, bool pred) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t@p st.global.v2.f32 [%0], {%1, %2};\n\t}" ::"l"(p),
                 "f"(v.x), "f"(v.y), "r"((int)pred)
                 : "memory");
}
FCW_DI void red_add2_if(float2* p, float2 v, bool pred) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t@p red.global.add.v2.f32 [%0], {%1, %2};\n\t}" ::"l"(p),
                 "f"(v.x), "f"(v.y), "r"((int)pred)
                 : "memory");
}

// *p += v as one fire-and-forget L2 reduction (red.global.add.v2.f32, sm_90+):
// FCW_TX_ACCUMULATE adds each sample exactly once onto the stored waveform,
// so the result equals the load-add-store it replaces, bit for bit.
FCW_DI void red_add2(float2* p, float2 v) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}

constexpr int kLtwLen = 64 + 4096 / 64;  // two-level long-transform twiddles (SMEM)
constexpr int kTw16Len = 512;            // fft256_half per-lane twiddles (uniform L = 256 kernels)
#ifndef FCW_TX_TAIL2
#define FCW_TX_TAIL2 1  // TX half-warp tail round: one subband per warp, one block per half
#endif
#ifndef FCW_TW16
#define FCW_TW16 1
#endif
#ifndef FCW_TX_UNROLL_R
#define FCW_TX_UNROLL_R 1  // TX half-warp pair rounds: both blocks unrolled (compile-time renames)
#endif
// The per-lane twiddle table follows the short and long twiddle tables in SMEM
// (filled in the kernel prologue when P.tw16 is set).
FCW_DI const float2* tw16_of(const KParams& P, const float2* stw) {
    return FCW_TW16 ? stw + P.stab_len + kLtwLen : nullptr;
}

// Streaming read of grid data that is used once: read-only path, no L1
// allocation, so the small L1 beside SMEM keeps the class table entries.
FCW_DI float2 ld_stream(const float2* p) {
    float2 v;
    asm("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
}

FCW_DI float2 grid_val(const KParams& P, const SubDev& sd, const float2* __restrict__ row, int b, int inv) {
    if (P.grid_full) return row[sd.full_off + b];
    return inv >= 0 ? row[sd.act_off + inv] : zero2();
}

// The threads that share one symbol's spectra: the whole CTA for N = 4096 (or
// N < 512), else one of G = 4096/N independent sub-teams of N/16 threads.
struct Team {
    int tid, nthr;    // thread index / count within the team
    int warp, nwarp;  // warp index / count within the team
    unsigned tm_a = 0, tm_c = 0;  // this thread's TMEM twiddle sets (TMEM-twiddle kernels, else unused)
    unsigned tm_k = 0;            // ... and its bin-class rows (32 columns per class)
};

// Kernels whose per-lane / per-thread twiddles live in TMEM (fcw_fft.cuh): the
// zero-bin L = 256, N = 4096 variant (config 5).
template <int N, int ZV>
constexpr bool tmem_tw() {
    return FCW_TMEM_TW && ZV == 1 && N == 4096;
}
// FCW_TMEM_TW bit 1: the half-warp FFT_256 twiddles, bit 2: the long-transform twiddles
template <int N, int ZV>
constexpr bool tmem_tw_half() {
    return tmem_tw<N, ZV>() && (FCW_TMEM_TW & 1);
}
template <int N, int ZV>
constexpr bool tmem_tw_long() {
    return tmem_tw<N, ZV>() && (FCW_TMEM_TW & 2);
}

// Allocate kTmemCols TMEM columns for the CTA and park the twiddle sets:
//   A [0, 32):   W_256^(k (lane & 15)), k = 0..15   (half-warp FFT_256; long pass 2)
//   B [32, 64):  W_256^(k ((lane & 15) + 64))       (fused RX: input rotated by j^t)
//   C [64, 96) for warps 0-3, [96, 128) for warps 4-7: W_N^(k tid)  (long pass 3)
//   K [128 + 32 j, + 32), row j < P.n_combo: the bin-class row of class P.combo[j][h] for the
//     threads of half-warp h (the two subbands a warp transforms side by side may differ in
//     class, and the warp reads its row with one tcgen05.ld), for the lane t = lane & 15 — 16 window weights w[t + 16 k] (columns 0-15) and 16 slot codes
//     (columns 16-31) of the bin's shifted position p0 = b ^ 128: rel = p0 - 128 for a primary
//     bin (spectrum slot (c_m + rel) mod N), kCodeExt + s for the subband's s-th secondary bin
//     (extension slot), kCodeNone for a zero-weight bin (tx_short_half scatter, rx_short_half).
// Every thread writes its own lane (warps w and w + 4 share a lane quadrant, and
// write identical A / B / K).  Returns the allocation's base address.
constexpr int kCodeExt = 0x1000, kCodeNone = 0x4000;  // slot codes of the TMEM bin-class rows
template <int N>
FCW_DI unsigned tmem_tables(const KParams& P, unsigned* slot, Team& tm) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (unsigned)__cvta_generic_to_shared(slot)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned base = *slot;
    const unsigned q = base + ((unsigned)((warp & 3) * 32) << 16);
    tm.tm_a = q;
    tm.tm_c = q + 64 + 32 * (warp >> 2);
    const int t16 = lane & 15, tid = threadIdx.x;
#pragma unroll 1
    for (int set = 0; set < 3; ++set) {
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
            unsigned d[16];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int kk = k + 8 * c;
                const int e = set == 0   ? ((kk * t16) & 255) * (N / 256)
                              : set == 1 ? ((kk * (t16 + 64)) & 255) * (N / 256)
                                         : (kk * tid) & (N - 1);
                const float2 w = __ldg(&P.tw[e]);
                d[2 * k] = __float_as_uint(w.x);
                d[2 * k + 1] = __float_as_uint(w.y);
            }
            tmem_st16((set == 2 ? tm.tm_c : q + 32 * set) + 16 * c, d);
        }
    }
    tm.tm_k = q + 128;
    for (int j = 0; j < P.n_combo && j < kMaxTmemClasses; ++j) {
        const int c = P.combo[j][lane >> 4];
        unsigned wv[16], cv[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int b = t16 + 16 * k;
            const int2 e = __ldg(&P.cls[c * 256 + b]);
            const int sec = e.x >> 16;
            wv[k] = (unsigned)e.y;
            cv[k] = (unsigned)(sec >= 0 ? kCodeExt + sec : (sec == -1 ? (b ^ 128) - 128 : kCodeNone));
        }
        tmem_st16(tm.tm_k + 32 * j, wv);
        tmem_st16(tm.tm_k + 32 * j + 16, cv);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    return base;
}
FCW_DI void tmem_release(unsigned base) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if ((threadIdx.x >> 5) == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(kTmemCols));
}

// ---------------------------------------------------------------- K-TX parts

// Short-side TX of one subband-symbol by one thread (L <= 32).
template <int N, int L, bool TDIO = true>  // TDIO: time-domain input compiled in (continuous FC)
FCW_DI void tx_short_thread(const KParams& P, const Team& tm, const SymDev& sy, const float2* __restrict__ row,
                            float2* spec0, float2* spec1, int gstart, int gcount) {
    const unsigned sb0 = (unsigned)__cvta_generic_to_shared(spec0), sb1 = (unsigned)__cvta_generic_to_shared(spec1);
    for (int i = tm.tid; i < gcount; i += tm.nthr) {
        const int m = P.grp_sub ? __ldg(&P.grp_sub[gstart + i]) : gstart + i;
        const SubDev sd = P.sub[m];
        float2 x[L];
        const float2 ph = cscale(tw_conj(P.tw, theta_exp<N>(sd.cmodN, sy.smodN)), sd.tx_scale);
        if (TDIO && P.td) {
            // time-domain input (continuous FC, as tx_short_half): x = sqrt(L) ph stream[n L - L_T + b]
            const fc_col d = P.td[m];
            const long long j0 = (sy.sigma / N) * L - d.lt;
            const float2 phs = cscale(ph, sqrtf((float)L));
#pragma unroll
            for (int b = 0; b < L; ++b)
                x[b] = (j0 + b >= 0 && j0 + b < d.len) ? cmul(row[d.in_off + j0 + b], phs) : zero2();
        } else {
#pragma unroll
            for (int b = 0; b < L; ++b) x[b] = cmul(grid_val(P, sd, row, b, bin_entry<N, L>(P, sd, b).inv), ph);
            fft_reg<L, +1>(x);  // ofdm_modulate (scale folded into ph)
        }
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
        for (int b = 0; b < L; ++b) {
            const Bin e = bin_entry<N, L>(P, sd, b);
            FCW_ASSERT(e.dest < P.spec_stride);
            sts_if(sb0, max(e.dest, 0), cscale(u0[b], e.w), e.dest >= 0);  // predicated stores, no branch
            sts_if(sb1, max(e.dest, 0), cscale(u1[b], e.w * sd.bp1), e.dest >= 0);
        }
    }
}

// Short-side TX of one subband-symbol by one warp (64 <= L <= 256), lane
// holds bins lane + 32k: synchronous gather, the two block DFTs in lockstep
// (shared twiddles, twice the ILP) over two padded scratch buffers.
template <int N, int L>
FCW_DI void tx_short_warp_lockstep(const KParams& P, const Team& tm, const SymDev& sy, const float2* __restrict__ row,
                          float2* spec0, float2* spec1, float2* scr, const float2* stw, int gstart, int gcount) {
    const unsigned sb0 = (unsigned)__cvta_generic_to_shared(spec0), sb1 = (unsigned)__cvta_generic_to_shared(spec1);
    constexpr int PPT = L / 32;
    const int lane = threadIdx.x & 31;
    const int sts = P.stab_len / L;
    float2* const b1[1] = {scr};
    for (int i = tm.warp; i < gcount; i += tm.nwarp) {
        const int m = P.grp_sub ? __ldg(&P.grp_sub[gstart + i]) : gstart + i;
        const SubDev sd = P.sub[m];
        const float2 ph = cscale(tw_conj(P.tw, theta_exp<N>(sd.cmodN, sy.smodN)), sd.tx_scale);
        const int2* ce = P.cls + sd.cls_off + lane;
        const int qbase = sd.c - L / 2 + lane, ext0 = N + sd.ext_base;
        int2 ent[PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) ent[k] = __ldg(&ce[32 * k]);
        float2 v[1][PPT];
        if (P.td) {
            // time-domain input (continuous FC, as tx_short_half): element lane + 32k of x
            const fc_col d = P.td[m];
            const long long j0 = (sy.sigma / N) * L - d.lt + lane;
            const float2 phs = cscale(ph, sqrtf((float)L));
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                const long long j = j0 + 32 * k;
                v[0][k] = (j >= 0 && j < d.len) ? cmul(ld_stream(row + d.in_off + j), phs) : zero2();
            }
        } else {
        if (P.grid_full) {
            const float2* g = row + sd.full_off + lane;
#pragma unroll
            for (int k = 0; k < PPT; ++k) v[0][k] = cmul(g[32 * k], ph);
        } else {
            const float2* g = row + sd.act_off;
#pragma unroll
            for (int k = 0; k < PPT; ++k) v[0][k] = ld_stream(g + max((int)(short)(ent[k].x & 0xffff), 0));
#pragma unroll
            for (int k = 0; k < PPT; ++k) v[0][k] = (short)(ent[k].x & 0xffff) >= 0 ? cmul(v[0][k], ph) : zero2();
        }
        team_fft<L, 32, PPT, +1, 1, false>(v, b1, stw, sts, lane, true);
        }
        const int lcp = sy.cp >> sd.logI;
        float2 uu[2][PPT];  // block-0 / block-1 DFT inputs
        if constexpr (L >= 128) {
            // L/4 is a multiple of 32: the circular shifts are register renames
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                const int e = lane + 32 * k;
                const bool in0 = (e >= L / 4 - lcp) && (e < 3 * L / 4);
                const bool in1 = (e >= L / 4) && (e < 3 * L / 4);
                uu[0][k] = in0 ? v[0][(k - PPT / 4 + PPT) % PPT] : zero2();
                uu[1][k] = in1 ? v[0][(k + PPT / 4) % PPT] : zero2();
            }
        } else {
            __syncwarp();
#pragma unroll
            for (int k = 0; k < PPT; ++k) scr[lane + 32 * k] = v[0][k];
            __syncwarp();
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                const int e = lane + 32 * k;
                const bool in0 = (e >= L / 4 - lcp) && (e < 3 * L / 4);
                const bool in1 = (e >= L / 4) && (e < 3 * L / 4);
                uu[0][k] = in0 ? scr[(e - L / 4) & (L - 1)] : zero2();
                uu[1][k] = in1 ? scr[(e + L / 4) & (L - 1)] : zero2();
            }
        }
        {
            // both block DFTs in lockstep: shared twiddles, twice the ILP
            float2* const b2[2] = {scr, scr + P.scratch_stride / 2};
            team_fft<L, 32, PPT, -1, 2, false>(uu, b2, stw, sts, lane, true);
        }
        const float bp1 = sd.bp1;
        auto scatter = [&](auto kc) {
            constexpr int K = decltype(kc)::value;
            const BinW e = bin_warp<N, L, K>(ent[K], qbase, ext0);
            FCW_ASSERT(e.dest < P.spec_stride);
            sts_if(sb0, max(e.dest, 0), cscale(uu[0][K], e.w), e.dest >= 0);  // predicated stores, no branch
            sts_if(sb1, max(e.dest, 0), cscale(uu[1][K], e.w * bp1), e.dest >= 0);
        };
        static_for<PPT>(scatter);
    }
}

// 8-byte asynchronous global->SMEM copy (zero-fill when !valid); nothing is
// held in registers while it is in flight.
FCW_DI void cp_async8(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(gsrc), "r"(valid ? 8 : 0)
                 : "memory");
}
FCW_DI void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
FCW_DI void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Request one subband's grid column (lane element b = lane + 32k) into the
// warp's staging buffer.
template <int L>
FCW_DI void stage_grid(const KParams& P, int m, const float2* __restrict__ row, float2* stage, int lane) {
    constexpr int PPT = L / 32;
    const SubDev* sd = P.sub + m;
    if (P.grid_full) {
        const float2* g = row + sd->full_off + lane;
#pragma unroll
        for (int k = 0; k < PPT; ++k) cp_async8(&stage[lane + 32 * k], g + 32 * k, true);
    } else {
        const float2* g = row + sd->act_off;
        const int2* ce = P.cls + sd->cls_off + lane;
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
            const int inv = (int)(short)(__ldg(&ce[32 * k]).x & 0xffff);
            cp_async8(&stage[lane + 32 * k], inv >= 0 ? g + inv : g, inv >= 0);
        }
    }
    cp_async_commit();
}

// Time-domain input (continuous FC): request x = stream[n L - L_T + e],
// e = lane + 32k, of subband m into the staging buffer (zero-filled outside
// the stream).
template <int N, int L>
FCW_DI void stage_stream(const KParams& P, int m, const SymDev& sy, const float2* __restrict__ row, float2* stage,
                         int lane) {
    constexpr int PPT = L / 32;
    const fc_col d = P.td[m];
    const long long j0 = (sy.sigma / N) * L - d.lt + lane;
    const float2* x = row + d.in_off;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
        const long long j = j0 + 32 * k;
        const bool ok = j >= 0 && j < d.len;
        cp_async8(&stage[lane + 32 * k], ok ? x + j : x, ok);
    }
    cp_async_commit();
}

// Short-side TX of one subband-symbol by one warp (L >= 64), lane holds bins
// lane + 32k.  One padded scratch buffer per warp plus a staging buffer that
// receives the NEXT subband's grid column by cp.async while this one is
// transformed (the first subband of the next symbol when `row_next` is set;
// `staged` says this symbol's first subband was requested that way).
template <int N, int L, bool TDIO = true>  // TDIO: time-domain input compiled in (continuous FC)
FCW_DI void tx_short_warp(const KParams& P, const Team& tm, const SymDev& sy, const float2* __restrict__ row,
                          const float2* __restrict__ row_next, bool staged, float2* spec0, float2* spec1,
                          float2* scr, const float2* stw, int gstart, int gcount) {
    const unsigned sb0 = (unsigned)__cvta_generic_to_shared(spec0), sb1 = (unsigned)__cvta_generic_to_shared(spec1);
    constexpr int PPT = L / 32;
    const int lane = threadIdx.x & 31;
    const int sts = P.stab_len / L;
    float2* const b1[1] = {scr};
    float2* stage = scr + P.stage_off;
    auto sub_of = [&](int i) { return P.grp_sub ? __ldg(&P.grp_sub[gstart + i]) : gstart + i; };
    if (tm.warp >= gcount) return;
    // time-domain input (continuous FC): the stream column is staged instead
    // of the grid column, within this symbol only (the caller passes no
    // row_next), and the IDFT is skipped (as tx_short_half)
    const bool td = TDIO && P.td != nullptr;
    if (td) stage_stream<N, L>(P, sub_of(tm.warp), sy, row, stage, lane);
    else if (!staged) stage_grid<L>(P, sub_of(tm.warp), row, stage, lane);
    for (int i = tm.warp; i < gcount; i += tm.nwarp) {
        const SubDev sd = P.sub[sub_of(i)];
        const float2 ph = cscale(tw_conj(P.tw, theta_exp<N>(sd.cmodN, sy.smodN)),
                                 td ? sd.tx_scale * sqrtf((float)L) : sd.tx_scale);
        float2 v[1][PPT];
        cp_async_wait_all();
        __syncwarp();
#pragma unroll
        for (int k = 0; k < PPT; ++k) v[0][k] = cmul(stage[lane + 32 * k], ph);
        __syncwarp();  // the staging buffer is free again
        if (td) {
            if (i + tm.nwarp < gcount) stage_stream<N, L>(P, sub_of(i + tm.nwarp), sy, row, stage, lane);
        } else {
            if (i + tm.nwarp < gcount)
                stage_grid<L>(P, sub_of(i + tm.nwarp), row, stage, lane);
            else if (row_next)
                stage_grid<L>(P, sub_of(tm.warp), row_next, stage, lane);
            team_fft<L, 32, PPT, +1, 1, false>(v, b1, stw, sts, lane, true);
        }
        const int lcp = sy.cp >> sd.logI;
        float2 uu[2][PPT];  // block-0 / block-1 DFT inputs (L/4 is a multiple of 32: register renames)
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
            const int e = lane + 32 * k;
            const bool in0 = (e >= L / 4 - lcp) && (e < 3 * L / 4);
            const bool in1 = (e >= L / 4) && (e < 3 * L / 4);
            uu[0][k] = in0 ? v[0][(k - PPT / 4 + PPT) % PPT] : zero2();
            uu[1][k] = in1 ? v[0][(k + PPT / 4) % PPT] : zero2();
        }
        const int2* ce = P.cls + sd.cls_off + lane;
        const int qbase = sd.c - L / 2 + lane, ext0 = N + sd.ext_base;
        const float bp1 = sd.bp1;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            float2 (&u)[1][PPT] = *reinterpret_cast<float2(*)[1][PPT]>(&uu[r]);
            team_fft<L, 32, PPT, -1, 1, false>(u, b1, stw, sts, lane, true);
            float2* spec = r == 0 ? spec0 : spec1;
            const float sgn = r == 0 ? 1.f : bp1;
            static_for<PPT>([&](auto kc) {
                constexpr int K = decltype(kc)::value;
                const BinW e = bin_warp<N, L, K>(__ldg(&ce[32 * K]), qbase, ext0);
                FCW_ASSERT(e.dest < P.spec_stride);
                sts_if(r == 0 ? sb0 : sb1, max(e.dest, 0), cscale(uu[r][K], e.w * sgn), e.dest >= 0);
            });
        }
    }
}

// Short-side TX for L = 256 by half-warps, 16 bins per lane (element
// b = t + 16k), radix-16 x 16 transforms with one exchange each:
// ofdm_modulate IDFT (ofdm.cpp:97-106), the two block windows of tx_symbol
// (fc_sync.cpp:34-84: L/4 is a multiple of 16, so the circular shifts are
// register renames) and the two block DFTs with their known-zero halves
// pruned (block 1 lives on [L/4, 3L/4), block 0 on [L/4 - l_cp, 3L/4)).
// ZV: every subband's bins t + 16m with m in [5, 10] are inactive (and
// outside the window): those IDFT inputs are known zero (C5's centred 144 of
// 256), so their gathers and first butterflies are skipped.
constexpr unsigned long long kZ6 = 0x07E0ull;  // m = 5..10
template <int N, int L, int ZV = 0>
FCW_DI void tx_short_half(const KParams& P, const Team& tm, const SymDev& sy, const float2* __restrict__ row,
                          float2* spec0, float2* spec1, float2* scr, const float2* stw, int gstart, int gcount) {
    constexpr int TW = 16, PPT = L / TW;
    static_assert(L == 256, "half-warp path is built for L = 256");
    const int lane = threadIdx.x & 31, t = lane & (TW - 1), h = lane >> 4;
    float2* buf = scr + h * (P.scratch_stride / 2);
    // Pair rounds while more than one subband per warp remains: one subband
    // per half-warp, both blocks.  Tail round (at most one subband per warp):
    // both halves transform the same subband (redundant IDFT) and each half
    // one block, so the tail's dependent chain is two transforms, not three
    // (balance: 23 subbands = 16 + 7).
    int done = 0;
    while (done < gcount) {
        const bool pair = gcount - done > (FCW_TX_TAIL2 ? tm.nwarp : 0);
        const int i = pair ? done + 2 * tm.warp + h : done + tm.warp;
        done += pair ? 2 * tm.nwarp : tm.nwarp;
        const bool act = i < gcount;
        if (!pair && !act) break;  // warp-uniform in the tail
        // (an idle half repeats the group's last subband: same TMEM row as its partner)
        const int ic = min(i, gcount - 1);
        const int m = P.grp_sub ? __ldg(&P.grp_sub[gstart + ic]) : gstart + ic;
        const SubDev sd = P.sub[m];
        const int2* ce = P.cls + sd.cls_off + t;
        float2 v[PPT];
        bool td = false;  // time-domain input (continuous FC): x itself, no IDFT
        if constexpr (ZV == 0) td = P.td != nullptr;
        if (td) {
            // block pair n carries x = stream[n L - L_T, + L), zero outside the
            // stream (cont_cols_kernel's DFT / sqrt(L) and this IDFT cancel:
            // v = sqrt(L) ph x)
            const fc_col d = P.td[m];
            const long long j0 = (sy.sigma / N) * L - d.lt + t;
            const float2 ph = cscale(tw_conj(P.tw, theta_exp<N>(sd.cmodN, sy.smodN)), sd.tx_scale * 16.f);
            const float2* x = row + d.in_off;
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                const long long j = j0 + TW * k;
                v[k] = (act && j >= 0 && j < d.len) ? cmul(ld_stream(x + j), ph) : zero2();
            }
        } else {
        {
            // theta_n from the two-level SMEM table of the long transform (W^e = W^(64 h) W^l: two
            // LDS and a product) instead of a dependent global table load at the head of the chain
            // (TX 6.43 -> 6.34 ms; the RX chain reads it at its tail, where the load is hidden)
            const int te = theta_exp<N>(sd.cmodN, sy.smodN);
            const float2* ltw = stw + P.stab_len;
            const float2 ph = cscale(cconj(cmul(ltw[64 + (te >> 6)], ltw[te & 63])), sd.tx_scale);
            constexpr unsigned long long ZI = ZV == 1 ? kZ6 : 0ull;
            auto live = [&](int k) { return !((ZI >> k) & 1ull); };
            int inv[PPT];
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                if constexpr (ZV == 1) {
                    // zv plans have centred active maps: no table load ahead of the gather
                    // (no `act` here: an idle half repeats the group's last subband in full, so its
                    // scatter stores the same values as the half that owns that subband)
                    const int a = (t + TW * k + (sd.n_act >> 1)) & (L - 1);
                    inv[k] = (live(k) && a < sd.n_act) ? a : -1;
                } else {
                    inv[k] = (act && live(k)) ? (int)(short)(__ldg(&ce[TW * k]).x & 0xffff) : -1;
                }
            }
            if (P.grid_full) {
                const float2* g = row + sd.full_off + t;
#pragma unroll
                for (int k = 0; k < PPT; ++k)
                    if (live(k)) v[k] = act ? ld_stream(g + TW * k) : zero2();
            } else {
                const float2* g = row + sd.act_off;
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    FCW_ASSERT(!act || sd.act_off + inv[k] < P.row_len);
                    if (live(k)) v[k] = ld_stream(g + max(inv[k], 0));
                }
#pragma unroll
                for (int k = 0; k < PPT; ++k)
                    if (live(k)) v[k] = inv[k] >= 0 ? v[k] : zero2();
            }
#pragma unroll
            for (int k = 0; k < PPT; ++k)
                if (live(k)) v[k] = cmul(v[k], ph);
        }
        fft256_half<+1, ZV == 1 ? kZ6 : 0ull, ~0ull, tmem_tw_half<N, ZV>()>(v, buf, stw, t, 0, tw16_of(P, stw),
                                                                      tm.tm_a);  // x[t + 16 m] (scales in ph)
        }
        const int lcp = sy.cp >> sd.logI;
        const int qbase = sd.c - L / 2 + t, ext0 = N + sd.ext_base;
        // One block: its DFT inputs from x (register renames), the pruned DFT and the scatter.
        // RC < 0: the block index is the runtime value r (tail round: r = h, lane dependent);
        // RC = 0 / 1: compile-time block (pair rounds): plain renames, and block 1's known-zero
        // CP positions (m < 4) join the DFT's zero mask.
        auto block = [&](auto rc_, int r) {
            constexpr int RC = decltype(rc_)::value;
            if constexpr (RC >= 0) r = RC;
            // block 0: e = t + 16 m in [L/4 - lcp, 3L/4) holds x[(e - L/4) mod L] = v[(m - 4) mod 16];
            // block 1: e in [L/4, 3L/4) holds x[e + L/4] = v[m + 4]  (register renames, L/4 = 4 * 16)
            float2 u[PPT];
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                if (k >= 4 && k < 12)
                    u[k] = r ? v[k + 4] : v[k - 4];
                else if (k < 4)
                    u[k] = (r == 0 && t + TW * k >= L / 4 - lcp) ? v[k + 12] : zero2();
                else
                    u[k] = zero2();  // k >= 12: known zero (not read)
            }
            // ZV: block bins t + 16m, m in [5, 10], lie outside every window (never scattered)
            fft256_half<-1, RC == 1 ? 0xF00Full : 0xF000ull, ZV == 1 ? (0xFFFFull & ~kZ6) : ~0ull, tmem_tw_half<N, ZV>()>(
                u, buf, stw, t, 0, tw16_of(P, stw), tm.tm_a);
            float2* spec = r ? spec1 : spec0;
            const float sgn = r ? sd.bp1 : 1.f;
            if constexpr (tmem_tw_half<N, ZV>()) {
                // weights and slot codes of this lane's bins from the class rows in TMEM: no table
                // load and a short decode between the DFT and its stores
                unsigned wv[16], cv[16];
                const unsigned row = tm.tm_k + 32 * sd.row_tx;  // warp-uniform by plan construction
                FCW_ASSERT(__shfl_sync(0xffffffffu, sd.row_tx, 0) == sd.row_tx);
                tmem_ld16(row, wv);
                tmem_ld16(row + 16, cv);
                tmem_wait16(wv);
                tmem_wait16(cv);
                const int extm = ext0 - kCodeExt;
                const unsigned sbase = (unsigned)__cvta_generic_to_shared(spec);
                static_for<PPT>([&](auto kc) {
                    constexpr int K = decltype(kc)::value;
                    if constexpr (!((kZ6 >> K) & 1ull)) {
                        const int code = (int)cv[K];
                        const int dest = code >= kCodeExt ? extm + code : ((sd.c + code) & (N - 1));
                        FCW_ASSERT(code >= kCodeNone || dest < P.spec_stride);
                        sts_if(sbase, dest, cscale(u[K], __uint_as_float(wv[K]) * sgn), code < kCodeNone);  // (idle halves repeat the last subband)
                    }
                });
                return;
            }
            static_for<PPT>([&](auto kc) {
                constexpr int K = decltype(kc)::value;
                constexpr int KP = K ^ (PPT / 2);  // (t + 16K) ^ (L/2) == t + 16*KP
                if constexpr (!(ZV == 1 && ((kZ6 >> K) & 1ull))) {  // ZV: outside every window, no slot
                    const int2 e = __ldg(&ce[TW * K]);
                    const int sec = e.x >> 16;
                    const int dest = sec >= 0 ? ext0 + sec : (sec == -1 ? ((qbase + TW * KP) & (N - 1)) : -1);
                    FCW_ASSERT(dest < P.spec_stride);
                    if (act && dest >= 0) spec[dest] = cscale(u[K], __int_as_float(e.y) * sgn);
                }
            });
        };
        if (FCW_TX_UNROLL_R && pair) {
            block(IC<0>{}, 0);
            block(IC<1>{}, 1);
        } else {
            const int r0 = pair ? 0 : h, r1 = pair ? 2 : h + 1;
#pragma unroll 1
            for (int r = r0; r < r1; ++r) block(IC<-1>{}, r);
        }
    }
}

// HALF: the kernel carries the half-warp twiddle table (the uniform L = 256
// specialisation); generic kernels use the whole-warp lockstep path.
// TDT: the thread and L >= 512 warp paths carry the time-domain input
// (continuous FC).  Kept out of the uniform-L kernels, where it measured +7%
// TX time on config 4 (L = 16) and +3% / +13% on configs 2 / 3 (L >= 512);
// continuous plans with L >= 512 run the generic kernels (Plan::generic).
template <int N, int L, bool HALF = false, int ZV = 0, bool TDT = true>
FCW_DI void tx_short_one(const KParams& P, const Team& tm, const SymDev& sy, const float2* __restrict__ row,
                         const float2* __restrict__ row_next, bool staged, float2* spec0, float2* spec1,
                         float2* scr, const float2* stw, int gs, int gc) {
    if constexpr (L <= N) {
        if constexpr (L <= 32)
            tx_short_thread<N, L, TDT>(P, tm, sy, row, spec0, spec1, gs, gc);
        else if constexpr (L == 256 && HALF)
            tx_short_half<N, L, ZV>(P, tm, sy, row, spec0, spec1, scr, stw, gs, gc);
        else if constexpr (L <= 256)
            tx_short_warp_lockstep<N, L>(P, tm, sy, row, spec0, spec1, scr, stw, gs, gc);
        else
            tx_short_warp<N, L, TDT>(P, tm, sy, row, row_next, staged, spec0, spec1, scr, stw, gs, gc);
    }
}

// Sub-teams per CTA: the long transform of one block needs N/16 threads, so a
// 256-thread CTA runs 4096/N independent teams for 512 <= N <= 4096 (each with
// its own spectra, work items and named barrier); smaller N use one team.
template <int N>
constexpr int teams_per_cta() {
    return (N >= 512 && N <= 4096) ? 4096 / N : 1;
}

// ------------------------------------------ L = 16 on 16-lane groups (C1)
// Narrowband plans (ZV = 2) have at most a handful of L = 16 subbands per
// team; one thread per subband leaves the team waiting on a 3-transform chain.
// Here each subband gets a 16-lane group, one bin per lane, and the 16-point
// transforms run across the lanes (radix-2 DIF by xor shuffles, then one
// bit-reversal shuffle).  Lane b of group i: bin b of subband i.

// X[b] of the 16 values held by the group's lanes (natural order in and out);
// SIGN = -1 forward, +1 inverse (unscaled).  tw = plan table exp(-2 pi i m / N).
template <int N, int SIGN, int NV>
FCW_DI void lane_fft16(float2 (&v)[NV], int b, const float2* __restrict__ tw) {
#pragma unroll
    for (int h = 8; h >= 1; h >>= 1) {
        const bool up = b & h;
        float2 w = __ldg(&tw[(b & (h - 1)) * (8 / h) * (N / 16)]);
        if (SIGN > 0) w.y = -w.y;
#pragma unroll
        for (int f = 0; f < NV; ++f) {
            float2 o;
            o.x = __shfl_xor_sync(0xffffffffu, v[f].x, h);
            o.y = __shfl_xor_sync(0xffffffffu, v[f].y, h);
            v[f] = up ? cmul(csub(o, v[f]), w) : cadd(v[f], o);
        }
    }
    const int src = (threadIdx.x & ~15) | (int)(__brev((unsigned)b) >> 28);  // X[b] sits in lane brev4(b)
#pragma unroll
    for (int f = 0; f < NV; ++f) {
        v[f].x = __shfl_sync(0xffffffffu, v[f].x, src & 31);
        v[f].y = __shfl_sync(0xffffffffu, v[f].y, src & 31);
    }
}

template <int N>
FCW_DI void tx_short_lanes16(const KParams& P, const Team& tm, const SymDev& sy, const float2* __restrict__ row,
                             float2* spec0, float2* spec1) {
    const unsigned sb0 = (unsigned)__cvta_generic_to_shared(spec0), sb1 = (unsigned)__cvta_generic_to_shared(spec1);
    constexpr int L = 16;
    const int b = tm.tid & 15;
    for (int i0 = (tm.tid >> 5) * 2; i0 < P.M; i0 += tm.nthr / 16) {  // warp-uniform: two groups per warp
        const int i = i0 + ((tm.tid >> 4) & 1);
        const bool act = i < P.M;
        const SubDev sd = P.sub[act ? i : i0];
        const Bin e = bin_entry<N, L>(P, sd, b);
        const float2 ph = cscale(tw_conj(P.tw, theta_exp<N>(sd.cmodN, sy.smodN)), sd.tx_scale);
        float2 x[1] = {act ? cmul(grid_val(P, sd, row, b, e.inv), ph) : zero2()};
        lane_fft16<N, +1, 1>(x, b, P.tw);  // ofdm_modulate (scale folded into ph)
        const int lcp = sy.cp >> sd.logI;
        // block windows of tx_symbol (fc_sync.cpp:34-84): element b of block 0 is
        // x[(b - L/4) mod L] on [L/4 - l_cp, 3L/4), of block 1 x[b + L/4] on [L/4, 3L/4)
        const int base = threadIdx.x & ~15;
        float2 u[2];
        u[0].x = __shfl_sync(0xffffffffu, x[0].x, (base | ((b - 4) & 15)) & 31);
        u[0].y = __shfl_sync(0xffffffffu, x[0].y, (base | ((b - 4) & 15)) & 31);
        u[1].x = __shfl_sync(0xffffffffu, x[0].x, (base | ((b + 4) & 15)) & 31);
        u[1].y = __shfl_sync(0xffffffffu, x[0].y, (base | ((b + 4) & 15)) & 31);
        if (!((b >= L / 4 - lcp) && (b < 3 * L / 4))) u[0] = zero2();
        if (!((b >= L / 4) && (b < 3 * L / 4))) u[1] = zero2();
        lane_fft16<N, -1, 2>(u, b, P.tw);
        FCW_ASSERT(e.dest < P.spec_stride);
        sts_if(sb0, max(e.dest, 0), cscale(u[0], e.w), act && e.dest >= 0);  // predicated stores, no branch
        sts_if(sb1, max(e.dest, 0), cscale(u[1], e.w * sd.bp1), act && e.dest >= 0);
    }
}

// Fused RX (Eq. 30, fc_sync.cpp:195-243) on 16-lane groups, as rx_short_thread.
template <int N>
FCW_DI void rx_short_lanes16(const KParams& P, const Team& tm, const SymDev& sy, const float2* spec0,
                             const float2* spec1, float2* __restrict__ orow) {
    constexpr int L = 16;
    const int b = tm.tid & 15;
    for (int i0 = (tm.tid >> 5) * 2; i0 < P.M; i0 += tm.nthr / 16) {
        const int i = i0 + ((tm.tid >> 4) & 1);
        const bool act = i < P.M;
        const SubDev sd = P.sub[act ? i : i0];
        const Bin e = bin_entry<N, L>(P, sd, b);
        const int q = (sd.c - L / 2 + (b ^ (L / 2))) & (N - 1);
        const float2 g0 = cscale(spec0[q], e.w);
        float2 t = cscale(spec1[q], e.w * sd.bp1);
        if (b & 1) t = make_float2(-t.x, -t.y);           // t = Omega_{L/2} g1
        float2 f[1] = {mul_jpow_rt(csub(g0, t), b & 3)};  // f = Omega_{-L/4}(g0 - t)
        lane_fft16<N, +1, 1>(f, b, P.tw);
        if (b >= L / 2) f[0] = zero2();                   // S-hat
        lane_fft16<N, -1, 1>(f, b, P.tw);
        const float2 ph = __ldg(&P.tw[theta_exp<N>(sd.cmodN, sy.smodN)]);  // conj(theta_n)
        const float a = sd.rx_s0 / (float)L, s = sd.rx_s0;
        const float2 tj = mul_jpow_rt(t, b & 3);
        const float2 o = cmul(make_float2(fmaf(f[0].x, a, tj.x * s), fmaf(f[0].y, a, tj.y * s)), ph);
        if (act) {
            if (P.grid_full) orow[sd.full_off + b] = o;
            else if (e.inv >= 0) orow[sd.act_off + e.inv] = o;
        }
    }
}

// ----------------------------------------------- team-wide short transforms
// For few large subbands (M <= warps/2, L >= 512: config 3's single L = 1024 /
// L = 512 banks) one warp per subband would leave the team's other warps
// idle; here the whole team transforms each subband, PPT = L / TT points per
// thread in the cyclic distribution v[k] = x[t + TT k], through the team's
// warp scratch (two buffers) with the team's barrier.
// Uniform L >= 512 kernels may transform on the whole team (when that leaves
// at least 4 points per thread); they do so when the plan has at most one
// subband per two warps of a team (config 3), else one warp per subband.
template <int N, int LU>
constexpr bool use_team_short() {
    return LU >= 512 && LU <= N && LU / (teams_per_cta<N>() == 1 ? kThreads : N / kPPT) >= 4;
}

template <int G>
FCW_DI int team_bar_id(const Team& tm) {
    return G == 1 ? 0 : 1 + (int)(threadIdx.x / tm.nthr);
}

template <int N, int L, int G>
FCW_DI void tx_short_team(const KParams& P, const Team& tm, const SymDev& sy, const float2* __restrict__ row,
                          float2* spec0, float2* spec1, float2* scr) {
    constexpr int TT = G == 1 ? kThreads : N / kPPT;  // threads per team
    constexpr int PPT = L / TT;
    static_assert(PPT >= 4 && PPT % 4 == 0 && PPT <= 16, "team short path: L / team size");
    const int t = tm.tid, bid = team_bar_id<G>(tm);
    float2* sbuf = scr - tm.warp * P.scratch_stride;  // the team's warp scratch, contiguous
    float2* const b1[1] = {sbuf};
    float2* const b2[2] = {sbuf, sbuf + (L + L / 16 + 2)};
    for (int m = 0; m < P.M; ++m) {
        const SubDev sd = P.sub[m];
        const float2 ph = cscale(tw_conj(P.tw, theta_exp<N>(sd.cmodN, sy.smodN)), sd.tx_scale);
        float2 v[1][PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
            const int b = t + TT * k;
            v[0][k] = cmul(grid_val(P, sd, row, b, bin_entry<N, L>(P, sd, b).inv), ph);
        }
        team_fft<L, TT, PPT, +1, 1, true>(v, b1, P.tw, N / L, t, true, bid, TT);  // ofdm_modulate
        const int lcp = sy.cp >> sd.logI;
        float2 uu[2][PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
            // block windows of tx_symbol (fc_sync.cpp:34-84): L/4 = (PPT/4) TT, a register rename
            const int e = t + TT * k;
            const bool in0 = (e >= L / 4 - lcp) && (e < 3 * L / 4);
            const bool in1 = (e >= L / 4) && (e < 3 * L / 4);
            uu[0][k] = in0 ? v[0][(k - PPT / 4 + PPT) % PPT] : zero2();
            uu[1][k] = in1 ? v[0][(k + PPT / 4) % PPT] : zero2();
        }
        team_bar<true>(bid, TT);  // the IDFT's last exchange has been read before the DFTs reuse the buffers
        team_fft<L, TT, PPT, -1, 2, true>(uu, b2, P.tw, N / L, t, true, bid, TT);
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
            const Bin e = bin_entry<N, L>(P, sd, t + TT * k);
            if (e.dest >= 0) {
                FCW_ASSERT(e.dest < P.spec_stride);
                spec0[e.dest] = cscale(uu[0][k], e.w);
                spec1[e.dest] = cscale(uu[1][k], e.w * sd.bp1);
            }
        }
        team_bar<true>(bid, TT);  // next subband reuses the buffers
    }
}

// RX of one subband by the whole team, as tx_short_team: fused Eq. (30)
// (fc_sync.cpp:195-243) or the direct path.
template <int N, int L, int G, bool FUSED>
FCW_DI void rx_short_team(const KParams& P, const Team& tm, const SymDev& sy, const float2* spec0,
                          const float2* spec1, float2* __restrict__ orow, float2* scr) {
    constexpr int TT = G == 1 ? kThreads : N / kPPT;
    constexpr int PPT = L / TT;
    static_assert(PPT >= 4 && PPT % 4 == 0 && PPT <= 16, "team short path: L / team size");
    const int t = tm.tid, bid = team_bar_id<G>(tm);
    float2* sbuf = scr - tm.warp * P.scratch_stride;
    float2* const b1[1] = {sbuf};
    float2* const b2[2] = {sbuf, sbuf + (L + L / 16 + 2)};
    for (int m = 0; m < P.M; ++m) {
        const SubDev sd = P.sub[m];
        float2 g0[1][PPT], g1[PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
            // rx_block_freq (fc_sync.cpp:178-193); b = t (mod 4) since TT is a multiple of 4
            const int b = t + TT * k;
            const float w = bin_entry<N, L>(P, sd, b).w;
            const int q = (sd.c - L / 2 + (b ^ (L / 2))) & (N - 1);
            const float2 a = cscale(spec0[q], w);
            float2 c1 = cscale(spec1[q], w * sd.bp1);
            if (t & 1) c1 = make_float2(-c1.x, -c1.y);  // t = Omega_{L/2} g1
            g1[k] = c1;
            g0[0][k] = mul_jpow_rt(csub(a, c1), t & 3);  // f = Omega_{-L/4}(g0 - t)
        }
        const float2 ph = __ldg(&P.tw[theta_exp<N>(sd.cmodN, sy.smodN)]);  // conj(theta_n)
        const float a = sd.rx_s0 / (float)L, s = sd.rx_s0;
        if (!FUSED) {
            // direct path (rx_symbol_direct fc_sync.cpp:158-176): both analysis
            // blocks, central halves (L/4 = (PPT/4) TT: register renames), OFDM DFT
            float2 gg[2][PPT];
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                const float2 c1 = (t & 1) ? make_float2(-g1[k].x, -g1[k].y) : g1[k];  // undo Omega_{L/2}
                gg[1][k] = c1;
                // g0 = f-rotation undone: a = j^{-t} f + t  ->  recover a from f and c1
                gg[0][k] = cadd(mul_jpow_rt(g0[0][k], (4 - (t & 3)) & 3), g1[k]);
            }
            team_fft<L, TT, PPT, +1, 2, true>(gg, b2, P.tw, N / L, t, true, bid, TT);
#pragma unroll
            for (int k = 0; k < PPT; ++k)
                g0[0][k] = k < PPT / 2 ? gg[0][k + PPT / 4] : gg[1][k - PPT / 4];
            if (P.td) {
                // time-domain output (continuous FC, as rx_short_warp): element t + TT k of x
                const fc_col d = P.td[m];
                const long long base = (sy.sigma / N) * L + t;
                const float2 phs = cscale(ph, sd.rx_s0 * rsqrtf((float)L));
#pragma unroll
                for (int k = 0; k < PPT; ++k)
                    if (base + TT * k < d.len_out) orow[d.out_off + base + TT * k] = cmul(g0[0][k], phs);
                team_bar<true>(bid, TT);  // next subband reuses the buffers
                continue;
            }
            team_bar<true>(bid, TT);
            team_fft<L, TT, PPT, -1, 1, true>(g0, b1, P.tw, N / L, t, true, bid, TT);
        } else {
            team_fft<L, TT, PPT, +1, 1, true>(g0, b1, P.tw, N / L, t, true, bid, TT);
#pragma unroll
            for (int k = PPT / 2; k < PPT; ++k) g0[0][k] = zero2();  // S-hat: e >= L/2
            team_bar<true>(bid, TT);
            team_fft<L, TT, PPT, -1, 1, true>(g0, b1, P.tw, N / L, t, true, bid, TT);
        }
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
            const int b = t + TT * k;
            const float2 tj = FUSED ? mul_jpow_rt(g1[k], t & 3) : zero2();
            const float2 o = cmul(make_float2(fmaf(g0[0][k].x, a, tj.x * s), fmaf(g0[0][k].y, a, tj.y * s)), ph);
            if (P.grid_full) {
                orow[sd.full_off + b] = o;
            } else {
                const int inv = bin_entry<N, L>(P, sd, b).inv;
                if (inv >= 0) orow[sd.act_off + inv] = o;
            }
        }
        team_bar<true>(bid, TT);
    }
}

template <int N, int LU, int ZV = 0>
FCW_DI void tx_short_all(const KParams& P, const Team& tm, const SymDev& sy, const float2* __restrict__ row,
                         const float2* __restrict__ row_next, bool staged, float2* spec0, float2* spec1,
                         float2* scr, const float2* stw) {
    if constexpr (ZV == 2 && LU == 16) {
        tx_short_lanes16<N>(P, tm, sy, row, spec0, spec1);
    } else if constexpr (ZV == 3 && use_team_short<N, LU>()) {
        // team-only kernels: the plan has at most one subband per two warps
        tx_short_team<N, LU, teams_per_cta<N>()>(P, tm, sy, row, spec0, spec1, scr);
    } else if constexpr (use_team_short<N, LU>()) {
        // few subbands: the whole team per subband; else one warp per subband
        if (2 * P.M <= tm.nwarp)
            tx_short_team<N, LU, teams_per_cta<N>()>(P, tm, sy, row, spec0, spec1, scr);
        else
            tx_short_one<N, LU, false, 0, false>(P, tm, sy, row, row_next, staged, spec0, spec1, scr, stw, 0, P.M);
    } else if constexpr (LU > 0) {
        // uniform L: the next symbol's first subband is staged across calls
        tx_short_one<N, LU, LU == 256, ZV, false>(P, tm, sy, row, row_next, staged, spec0, spec1, scr, stw, 0, P.M);
    } else {
        for (int g = 0; g < P.n_groups; ++g) {
            const int gs = P.grp_start[g], gc = P.grp_count[g];
            switch (P.grp_L[g]) {
                case 4: tx_short_one<N, 4>(P, tm, sy, row, nullptr, false, spec0, spec1, scr, stw, gs, gc); break;
                case 8: tx_short_one<N, 8>(P, tm, sy, row, nullptr, false, spec0, spec1, scr, stw, gs, gc); break;
                case 16: tx_short_one<N, 16>(P, tm, sy, row, nullptr, false, spec0, spec1, scr, stw, gs, gc); break;
                case 32: tx_short_one<N, 32>(P, tm, sy, row, nullptr, false, spec0, spec1, scr, stw, gs, gc); break;
                case 64: tx_short_one<N, 64>(P, tm, sy, row, nullptr, false, spec0, spec1, scr, stw, gs, gc); break;
                case 128: tx_short_one<N, 128>(P, tm, sy, row, nullptr, false, spec0, spec1, scr, stw, gs, gc); break;
                case 256: tx_short_one<N, 256>(P, tm, sy, row, nullptr, false, spec0, spec1, scr, stw, gs, gc); break;
                case 512: tx_short_one<N, 512>(P, tm, sy, row, nullptr, false, spec0, spec1, scr, stw, gs, gc); break;
                case 1024: tx_short_one<N, 1024>(P, tm, sy, row, nullptr, false, spec0, spec1, scr, stw, gs, gc); break;
                default: break;
            }
        }
    }
}

// ---------------------------------------------------------------- K-RX parts

template <int N, int L, bool TDIO = true>  // TDIO: time-domain output compiled in (continuous FC)
FCW_DI void rx_short_thread(const KParams& P, const Team& tm, const SymDev& sy, const float2* spec0,
                            const float2* spec1, float2* __restrict__ orow, int gstart, int gcount) {
    for (int i = tm.tid; i < gcount; i += tm.nthr) {
        const int m = P.grp_sub ? __ldg(&P.grp_sub[gstart + i]) : gstart + i;
        const SubDev sd = P.sub[m];
        // rx_block_freq (fc_sync.cpp:178-193) without the per-symbol rotator,
        // which is applied once at the output (linearity)
        float2 g0[L], g1[L];
#pragma unroll
        for (int b = 0; b < L; ++b) {
            const float w = bin_entry<N, L>(P, sd, b).w;
            const int q = (sd.c - L / 2 + (b ^ (L / 2))) & (N - 1);
            g0[b] = cscale(spec0[q], w);
            g1[b] = cscale(spec1[q], w * sd.bp1);
        }
        const float2 ph = __ldg(&P.tw[theta_exp<N>(sd.cmodN, sy.smodN)]);  // conj(theta_n)
        if (P.fused) {
            // Eq. (30): t = Omega_{L/2} g1, f = Omega_{-L/4}(g0 - t), IDFT, S-hat,
            // DFT, Omega_{L/4}, + t, Omega_{-L/4}  (fc_sync.cpp:195-243)
#pragma unroll
            for (int b = 0; b < L; ++b) {
                if (b & 1) g1[b] = make_float2(-g1[b].x, -g1[b].y);  // t
                const float2 f = csub(g0[b], g1[b]);
                switch (b & 3) {
                    case 0: g0[b] = f; break;
                    case 1: g0[b] = mul_jpow<1>(f); break;
                    case 2: g0[b] = mul_jpow<2>(f); break;
                    default: g0[b] = mul_jpow<3>(f); break;
                }
            }
            fft_reg<L, +1>(g0);
#pragma unroll
            for (int k = L / 2; k < L; ++k) g0[k] = zero2();
            fft_reg<L, -1>(g0);
            const float a = sd.rx_s0 / (float)L, s = sd.rx_s0;
#pragma unroll
            for (int b = 0; b < L; ++b) {
                float2 tj = g1[b];
                switch (b & 3) {
                    case 1: tj = mul_jpow<1>(tj); break;
                    case 2: tj = mul_jpow<2>(tj); break;
                    case 3: tj = mul_jpow<3>(tj); break;
                    default: break;
                }
                g0[b] = cmul(make_float2(fmaf(g0[b].x, a, tj.x * s), fmaf(g0[b].y, a, tj.y * s)), ph);
            }
        } else {
            // direct path: two OLS analysis blocks, central halves, OFDM DFT
            fft_reg<L, +1>(g0);
            fft_reg<L, +1>(g1);
            float2 x[L];
#pragma unroll
            for (int k = 0; k < L / 2; ++k) {
                x[k] = g0[L / 4 + k];
                x[L / 2 + k] = g1[L / 4 + k];
            }
            if (TDIO && P.td) {  // time-domain output (continuous FC), as rx_short_warp
                const fc_col d = P.td[m];
                const long long base = (sy.sigma / N) * L;
                const float2 phs = cscale(ph, sd.rx_s0 * rsqrtf((float)L));
                float2* o = orow + d.out_off;
#pragma unroll
                for (int b = 0; b < L; ++b)
                    if (base + b < d.len_out) o[base + b] = cmul(x[b], phs);
                continue;
            }
            fft_reg<L, -1>(x);
            const float2 phs = cscale(ph, sd.rx_s0 / (float)L);
#pragma unroll
            for (int b = 0; b < L; ++b) g0[b] = cmul(x[b], phs);
        }
#pragma unroll
        for (int b = 0; b < L; ++b) {
            if (P.grid_full) {
                orow[sd.full_off + b] = g0[b];
            } else {
                const int a = bin_entry<N, L>(P, sd, b).inv;
                if (a >= 0) orow[sd.act_off + a] = g0[b];
            }
        }
    }
}

template <int N, int L, bool TDIO = true>  // TDIO: time-domain output compiled in (continuous FC)
FCW_DI void rx_short_warp(const KParams& P, const Team& tm, const SymDev& sy, const float2* spec0,
                          const float2* spec1, float2* __restrict__ orow, float2* scr, const float2* stw, int gstart,
                          int gcount) {
    constexpr int PPT = L / 32;
    const int lane = threadIdx.x & 31;
    const int sts = P.stab_len / L;
    float2* const b1[1] = {scr};
    for (int i = tm.warp; i < gcount; i += tm.nwarp) {
        const int m = P.grp_sub ? __ldg(&P.grp_sub[gstart + i]) : gstart + i;
        const SubDev sd = P.sub[m];
        float2 g0[1][PPT], g1[1][PPT];
        int inv[PPT];
        {
            const int2* ce = P.cls + sd.cls_off + lane;
            const int qbase = sd.c - L / 2 + lane;
            const float bp1 = sd.bp1;
            static_for<PPT>([&](auto kc) {
                constexpr int K = decltype(kc)::value;
                constexpr int KP = K ^ (L / 64);  // (lane + 32K) ^ (L/2) == lane + 32*KP
                const int2 e = __ldg(&ce[32 * K]);
                inv[K] = (int)(short)(e.x & 0xffff);
                const float w = __int_as_float(e.y);
                const int q = (qbase + 32 * KP) & (N - 1);
                g0[0][K] = cscale(spec0[q], w);
                g1[0][K] = cscale(spec1[q], w * bp1);
            });
        }
        const float2 ph = __ldg(&P.tw[theta_exp<N>(sd.cmodN, sy.smodN)]);
        if (P.fused) {
            const bool odd = lane & 1;
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                if (odd) g1[0][k] = make_float2(-g1[0][k].x, -g1[0][k].y);  // t
                g0[0][k] = mul_jpow_rt(csub(g0[0][k], g1[0][k]), lane);
            }
            team_fft<L, 32, PPT, +1, 1, false>(g0, b1, stw, sts, lane, true);
#pragma unroll
            for (int k = PPT / 2; k < PPT; ++k) g0[0][k] = zero2();
            team_fft<L, 32, PPT, -1, 1, false>(g0, b1, stw, sts, lane, true);
            const float a = sd.rx_s0 / (float)L, s = sd.rx_s0;
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
                const float2 tj = mul_jpow_rt(g1[0][k], lane);
                g0[0][k] = cmul(make_float2(fmaf(g0[0][k].x, a, tj.x * s), fmaf(g0[0][k].y, a, tj.y * s)), ph);
            }
        } else {
            team_fft<L, 32, PPT, +1, 1, false>(g0, b1, stw, sts, lane, true);
            team_fft<L, 32, PPT, +1, 1, false>(g1, b1, stw, sts, lane, true);
            float2 x[1][PPT];
            if constexpr (L >= 128) {
                // central halves: element L/4 + i of block r -> register rename
#pragma unroll
                for (int k = 0; k < PPT; ++k)
                    x[0][k] = (k < PPT / 2) ? g0[0][k + PPT / 4] : g1[0][k - PPT / 2 + PPT / 4];
            } else {
                float2* s1 = scr + P.scratch_stride / 2;
                __syncwarp();
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    scr[lane + 32 * k] = g0[0][k];
                    s1[lane + 32 * k] = g1[0][k];
                }
                __syncwarp();
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    const int e = lane + 32 * k;
                    x[0][k] = (k < PPT / 2) ? scr[L / 4 + e] : s1[L / 4 + e - L / 2];
                }
            }
            if (TDIO && P.td) {
                // time-domain output (continuous FC): x itself, no OFDM DFT
                // (cont_cols_kernel's IDFT / sqrt(L) would undo it): pair n
                // lands at out[n L, + L) of subband m's output stream
                const fc_col d = P.td[m];
                const long long base = (sy.sigma / N) * L;
                const float2 phs = cscale(ph, sd.rx_s0 * rsqrtf((float)L));
                float2* o = orow + d.out_off;
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    const long long j = base + lane + 32 * k;
                    if (j < d.len_out) o[j] = cmul(x[0][k], phs);
                }
                __syncwarp();
                continue;
            }
            team_fft<L, 32, PPT, -1, 1, false>(x, b1, stw, sts, lane, true);
            const float2 phs = cscale(ph, sd.rx_s0 / (float)L);
#pragma unroll
            for (int k = 0; k < PPT; ++k) g0[0][k] = cmul(x[0][k], phs);
        }
        if (P.grid_full) {
            float2* o = orow + sd.full_off + lane;
#pragma unroll
            for (int k = 0; k < PPT; ++k) o[32 * k] = g0[0][k];
        } else {
            float2* o = orow + sd.act_off;
#pragma unroll
            for (int k = 0; k < PPT; ++k)
                if (inv[k] >= 0) {
                    FCW_ASSERT(sd.act_off + inv[k] < P.row_len);
                    o[inv[k]] = g0[0][k];
                }
        }
        __syncwarp();
    }
}

// Fused RX (Eq. 30) for L = 256 by half-warps, 16 bins per lane (element
// b = t + 16k): both short transforms radix-16 x 16, one exchange each.
// Every per-bin rotation of rx_symbol_simplified (fc_sync.cpp:195-243) is a
// lane constant here, because b = t (mod 16):
//   f = Omega_{-L/4}(g0 - Omega_{L/2} g1) = j^t * w (S0 - (-1)^t bp1 S1):
//     the j^t factor is folded into the IDFT's pass-2 twiddles (eoff = L/4);
//   out = conj(theta) (a G + s j^t t) = P1 G + P2 (w S1), with
//     P1 = a conj(theta), P2 = s bp1 (-j)^t conj(theta) per lane and subband.
// The spectra carry a wrap-around copy of bins [0, L) at [N, N + L), so the
// bin addresses of a subband are one base plus immediate offsets.
template <int N, int L, int ZV = 0>
FCW_DI void rx_short_half(const KParams& P, const Team& tm, const SymDev& sy, const float2* spec0,
                          const float2* spec1, float2* __restrict__ orow, float2* scr, const float2* stw,
                          int gstart, int gcount) {
    constexpr int TW = 16, PPT = L / TW;
    static_assert(L == 256, "half-warp path is built for L = 256");
    const int lane = threadIdx.x & 31, t = lane & (TW - 1), h = lane >> 4;
    float2* buf = scr + h * (P.scratch_stride / 2);
    const float sgn_t = (t & 1) ? -1.f : 1.f;  // (-1)^b
    // Rounds of two subbands per warp (a whole-warp tail round was measured
    // slower here: the chain IDFT -> DFT cannot be split across halves).
    int done = 0;
    while (gcount - done > 0) {
        // a warp with no subband left in this round leaves (warp-uniform): it
        // goes on to the next symbol's window loads instead of transforming
        // discarded data (23 subbands = 16 + 7: warps 4..7 skip round 2)
        if (done + 2 * tm.warp >= gcount) break;
        const int i = done + 2 * tm.warp + h;
        done += 2 * tm.nwarp;
        const bool act = i < gcount;
        // (an idle half repeats the group's last subband: same TMEM row as its partner)
        const int ic = min(i, gcount - 1);
        const int m = P.grp_sub ? __ldg(&P.grp_sub[gstart + ic]) : gstart + ic;
        const SubDev sd = P.sub[m];
        const int2* ce = P.cls + sd.cls_off + t;
        const int q0 = (sd.c - L / 2 + t) & (N - 1);
        const float2* s0 = spec0 + q0;
        const float2* s1 = spec1 + q0;
        const float sig = sgn_t * sd.bp1;
        float2 f[PPT], gw[PPT];
        unsigned wv[16];
        if constexpr (tmem_tw_half<N, ZV>()) {
            FCW_ASSERT(__shfl_sync(0xffffffffu, sd.row_rx, 0) == sd.row_rx);
            tmem_ld16(tm.tm_k + 32 * sd.row_rx, wv);  // this lane's window weights (class row in TMEM)
            tmem_wait16(wv);
        }
        static_for<PPT>([&](auto kc) {
            constexpr int K = decltype(kc)::value;
            constexpr int KP = K ^ (PPT / 2);  // (t + 16K) ^ (L/2) == t + 16*KP
            if constexpr (ZV == 1 && ((kZ6 >> K) & 1ull)) {
                gw[K] = zero2();  // outside every window: zero input, inactive output
            } else {
                float w;
                if constexpr (tmem_tw_half<N, ZV>()) w = __uint_as_float(wv[K]);
                else w = __int_as_float(__ldg(&ce[TW * K]).y);
                const float2 a = s0[TW * KP], b = s1[TW * KP];
                gw[K] = cscale(b, w);
                f[K] = cscale(make_float2(fmaf(-sig, b.x, a.x), fmaf(-sig, b.y, a.y)), w);
            }
        });
        // IDFT of j^t f; S-hat then keeps x[e], e < L/2: outputs m >= 8 are dead
        fft256_half<+1, ZV == 1 ? kZ6 : 0ull, 0x00FFull, tmem_tw_half<N, ZV>()>(f, buf, stw, t, L / 4, tw16_of(P, stw),
                                                                          tm.tm_a);
        // S-hat keeps x[e], e < L/2; DFT
        fft256_half<-1, 0xFF00ull, ~0ull, tmem_tw_half<N, ZV>()>(f, buf, stw, t, 0, tw16_of(P, stw), tm.tm_a);
        const float2 ph = __ldg(&P.tw[theta_exp<N>(sd.cmodN, sy.smodN)]);  // conj(theta_n)
        const float2 P1 = cscale(ph, sd.rx_s0 / (float)L);
        const float2 P2 = mul_jpow_rt(cscale(ph, sd.rx_s0 * sd.bp1), (4 - t) & 3);
        auto outv = [&](int k) {
            return make_float2(fmaf(f[k].x, P1.x, fmaf(-f[k].y, P1.y, fmaf(gw[k].x, P2.x, -gw[k].y * P2.y))),
                               fmaf(f[k].x, P1.y, fmaf(f[k].y, P1.x, fmaf(gw[k].x, P2.y, gw[k].y * P2.x))));
        };
        // (an idle half repeats its partner's subband: it stores the same values to the same places)
        {
            if (P.grid_full) {
                float2* o = orow + sd.full_off + t;
#pragma unroll
                for (int k = 0; k < PPT; ++k) o[TW * k] = outv(k);
            } else {
                float2* o = orow + sd.act_off;
                constexpr unsigned long long ZO = ZV == 1 ? kZ6 : 0ull;  // ZV: inactive bins, nothing to store
                int inv[PPT];  // all entry loads in flight before the first store
#pragma unroll
                for (int k = 0; k < PPT; ++k) {
                    if constexpr (ZV == 1) {
                        // zv plans have centred active maps (see tx_short_half)
                        const int a = (t + TW * k + (sd.n_act >> 1)) & (L - 1);
                        inv[k] = (!((ZO >> k) & 1ull) && a < sd.n_act) ? a : -1;
                    } else {
                        inv[k] = ((ZO >> k) & 1ull) ? -1 : (int)(short)(__ldg(&ce[TW * k]).x & 0xffff);
                    }
                }
#pragma unroll
                for (int k = 0; k < PPT; ++k)
                    if (!((ZO >> k) & 1ull) && inv[k] >= 0) {
                        FCW_ASSERT(sd.act_off + inv[k] < P.row_len);
                        __stcs(&o[inv[k]], outv(k));  // streaming store: the grid is not re-read here
                    }
            }
        }
    }
}

// MIRROR: the kernel keeps the wrap-around spectrum copy rx_short_half needs
// (the uniform L = 256 specialisation); generic kernels use the warp path.
template <int N, int L, bool MIRROR = false, int ZV = 0>
FCW_DI void rx_short_one(const KParams& P, const Team& tm, const SymDev& sy, const float2* spec0,
                         const float2* spec1, float2* orow, float2* scr, const float2* stw, int gs, int gc) {
    if constexpr (L <= N) {
        if constexpr (L <= 32)
            rx_short_thread<N, L, ZV != 1>(P, tm, sy, spec0, spec1, orow, gs, gc);
        else if constexpr (L == 256 && MIRROR) {
            if (P.fused)
                rx_short_half<N, L, ZV>(P, tm, sy, spec0, spec1, orow, scr, stw, gs, gc);
            else
                rx_short_warp<N, L, ZV != 1>(P, tm, sy, spec0, spec1, orow, scr, stw, gs, gc);
        } else
            rx_short_warp<N, L, ZV != 1>(P, tm, sy, spec0, spec1, orow, scr, stw, gs, gc);
    }
}

template <int N, int LU, int ZV = 0>
FCW_DI void rx_short_all(const KParams& P, const Team& tm, const SymDev& sy, const float2* spec0,
                         const float2* spec1, float2* orow, float2* scr, const float2* stw) {
    if constexpr (ZV == 2 && LU == 16) {
        if (P.fused)
            rx_short_lanes16<N>(P, tm, sy, spec0, spec1, orow);
        else
            rx_short_one<N, LU>(P, tm, sy, spec0, spec1, orow, scr, stw, 0, P.M);
    } else if constexpr (ZV == 3 && use_team_short<N, LU>()) {
        if (P.fused)
            rx_short_team<N, LU, teams_per_cta<N>(), true>(P, tm, sy, spec0, spec1, orow, scr);
        else
            rx_short_team<N, LU, teams_per_cta<N>(), false>(P, tm, sy, spec0, spec1, orow, scr);
    } else if constexpr (use_team_short<N, LU>()) {
        if (2 * P.M > tm.nwarp)
            rx_short_one<N, LU>(P, tm, sy, spec0, spec1, orow, scr, stw, 0, P.M);
        else if (P.fused)
            rx_short_team<N, LU, teams_per_cta<N>(), true>(P, tm, sy, spec0, spec1, orow, scr);
        else
            rx_short_team<N, LU, teams_per_cta<N>(), false>(P, tm, sy, spec0, spec1, orow, scr);
    } else if constexpr (LU > 0) {
        rx_short_one<N, LU, LU == 256, ZV>(P, tm, sy, spec0, spec1, orow, scr, stw, 0, P.M);
    } else {
        for (int g = 0; g < P.n_groups; ++g) {
            const int gs = P.grp_start[g], gc = P.grp_count[g];
            switch (P.grp_L[g]) {
                case 4: rx_short_one<N, 4>(P, tm, sy, spec0, spec1, orow, scr, stw, gs, gc); break;
                case 8: rx_short_one<N, 8>(P, tm, sy, spec0, spec1, orow, scr, stw, gs, gc); break;
                case 16: rx_short_one<N, 16>(P, tm, sy, spec0, spec1, orow, scr, stw, gs, gc); break;
                case 32: rx_short_one<N, 32>(P, tm, sy, spec0, spec1, orow, scr, stw, gs, gc); break;
                case 64: rx_short_one<N, 64>(P, tm, sy, spec0, spec1, orow, scr, stw, gs, gc); break;
                case 128: rx_short_one<N, 128>(P, tm, sy, spec0, spec1, orow, scr, stw, gs, gc); break;
                case 256: rx_short_one<N, 256>(P, tm, sy, spec0, spec1, orow, scr, stw, gs, gc); break;
                case 512: rx_short_one<N, 512>(P, tm, sy, spec0, spec1, orow, scr, stw, gs, gc); break;
                case 1024: rx_short_one<N, 1024>(P, tm, sy, spec0, spec1, orow, scr, stw, gs, gc); break;
                default: break;
            }
        }
    }
}

// ------------------------------------------------------------------ kernels

template <int LU, int ZV = 0>
constexpr int min_blocks() {
    // ZV = 3 (team-only short path, few L >= 512 subbands: 4-8 points per
    // thread): two CTAs per SM at <= 128 registers
    if (ZV == 3) return 2;
    // L >= 512: the warp paths hold 16-32 points per lane; one CTA per SM with
    // up to 255 registers beats two spilling CTAs (config 2: 30 -> 38 Gsamples/s)
    if (LU >= 512) return 1;
    return (LU >= 64 || (LU > 0 && LU <= 16)) ? 2 : 1;
}


// Team-scope barrier: the CTA barrier for a single team, else named barrier
// 1 + g over the team's threads (bar.sync counts must be warp multiples).
template <int G>
FCW_DI void team_sync(int g, int nthr) {
    if constexpr (G == 1)
        __syncthreads();
    else
        asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(nthr) : "memory");
}

// ------------------------------------------------ narrowband long transforms
// ZV == 2: every subband's L-bin span lies in the 16 bins [k0, k0 + 16) (mod
// N) — config 1, one 12-subcarrier subband in N = 1024.  The N-point transform
// of a block then collapses to one 16-point transform per thread with input
// and output twiddles (the pruned IDFT_N of SURVEY §7 hard part 1e): no SMEM
// exchange passes.  Thread t holds x[t + T s], s < 16, T = N / 16.

// p[k] = u^k for k < 16, each at most three products deep.
FCW_DI void cpow16(float2 (&p)[16], float2 u) {
    p[0] = make_float2(1.f, 0.f);
    p[1] = u;
    p[2] = cmul(u, u);
    p[3] = cmul(p[2], u);
    p[4] = cmul(p[2], p[2]);
#pragma unroll
    for (int k = 5; k < 8; ++k) p[k] = cmul(p[4], p[k - 4]);
    p[8] = cmul(p[4], p[4]);
#pragma unroll
    for (int k = 9; k < 16; ++k) p[k] = cmul(p[8], p[k - 8]);
}

// TX: x_f[t + T s] = sum_k S_f[k0 + k] e^{+2 pi i (t + T s)(k0 + k) / N}
//   = E(t k0) w16^{s k0} IDFT16_s(S_f[k0 + k] E(t k)),  E(a) = e^{2 pi i a / N}.
template <int N>
FCW_DI void nb_long_inverse(float2 (&v)[2][16], const float2* spec0, const float2* spec1, const float2* tw,
                            int t, int k0) {
    constexpr int T = N / 16;
    float2 w[16], q[16];
    cpow16(w, tw_conj(tw, t));  // E(t)^k
#pragma unroll
    for (int f = 0; f < 2; ++f) {
        const float2* S = f ? spec1 : spec0;
#pragma unroll
        for (int k = 0; k < 16; ++k) v[f][k] = cmul(S[(k0 + k) & (N - 1)], w[k]);
        fft_reg<16, +1>(v[f]);
    }
    cpow16(q, tw_conj(tw, (T * k0) & (N - 1)));  // w16^{s k0}
    const float2 c = tw_conj(tw, (int)(((unsigned)t * (unsigned)k0) & (unsigned)(N - 1)));
#pragma unroll
    for (int s = 0; s < 16; ++s) {
        const float2 ps = cmul(q[s], c);
        v[0][s] = cmul(v[0][s], ps);
        v[1][s] = cmul(v[1][s], ps);
    }
}

// RX: Y_f[k0 + k] = sum_t W^{t(k0 + k)} DFT16_k(y_f[t + T s] W16^{s k0}),
// W = e^{-2 pi i / N}; the sum over the T threads goes through SMEM
// (red: 32 T float2, the team's spectrum region) in a fixed order.
template <int N, int G>
FCW_DI void nb_long_forward(float2 (&v)[2][16], float2* spec0, float2* spec1, float2* red, const float2* tw, int t,
                            int k0, int g, int TT) {
    constexpr int T = N / 16;
    static_assert(T >= 64 && T % 32 == 0, "narrowband reduction: T = N / 16 >= 64");
    float2 q[16], w[16];
    cpow16(q, __ldg(&tw[(T * k0) & (N - 1)]));  // W16^{s k0}
#pragma unroll
    for (int s = 1; s < 16; ++s) {
        v[0][s] = cmul(v[0][s], q[s]);
        v[1][s] = cmul(v[1][s], q[s]);
    }
    fft_reg<16, -1>(v[0]);
    fft_reg<16, -1>(v[1]);
    cpow16(w, __ldg(&tw[t]));  // W^{t k}
    const float2 c = __ldg(&tw[(int)(((unsigned)t * (unsigned)k0) & (unsigned)(N - 1))]);
    // partials thread-major, padded (conflict-free): red[t * 33 + p], p = 16 f + k
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const float2 pk = cmul(w[k], c);
        red[t * 33 + k] = cmul(v[0][k], pk);
        red[t * 33 + 16 + k] = cmul(v[1][k], pk);
    }
    team_sync<G>(g, TT);
    // warp w sums the partials of threads [32 w, 32 w + 32), lane = p
    constexpr int W = T / 32;
    const int lane = t & 31, wp = t >> 5;
    float2 a0 = zero2(), a1 = zero2(), a2 = zero2(), a3 = zero2();
    const float2* src = red + (32 * wp) * 33 + lane;
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
        a0 = cadd(a0, src[(j + 0) * 33]);
        a1 = cadd(a1, src[(j + 1) * 33]);
        a2 = cadd(a2, src[(j + 2) * 33]);
        a3 = cadd(a3, src[(j + 3) * 33]);
    }
    float2* accs = red + T * 33;  // W x 32 warp sums
    accs[wp * 32 + lane] = cadd(cadd(a0, a1), cadd(a2, a3));
    team_sync<G>(g, TT);
    if (wp == 0) {
        float2 y = accs[lane];
#pragma unroll
        for (int q = 1; q < W; ++q) y = cadd(y, accs[q * 32 + lane]);
        float2* S = lane < 16 ? spec0 : spec1;
        S[(k0 + (lane & 15)) & (N - 1)] = y;
    }
}

// Work distribution over the resident teams, two modes (chosen per launch):
//  * static: the launch's S*B (unit, symbol) pairs are split into one
//    contiguous balanced range per team, walked unit by unit (runs of at most
//    P.chunk symbols).  Few run starts (TX recomputes one symbol per start) and
//    +-1 symbol balance: best when each team has little work (many GPUs).
//  * dynamic: runs of P.chunk symbols are pulled from a global counter; the
//    next run's id is requested when a run starts, so the counter's round
//    trip is hidden.  Absorbs speed differences between CTAs: best at full
//    load.
template <int G, bool DYN>
struct RunSource {
    int pos, hi;  // static: this team's remaining range of S*B symbols
    int pending;  // dynamic: id of the next run (-1 before the first fetch)

    FCW_DI RunSource(const KParams& P, int g) : pos(0), hi(0), pending(-1) {
        if constexpr (!DYN) {
            const long long total = (long long)P.n_units * P.B;
            const long long nt = (long long)gridDim.x * P.teams;
            const long long t = (long long)blockIdx.x * P.teams + g;
            pos = (int)(total * t / nt);
            hi = (int)(total * (t + 1) / nt);
        }
    }

    // Static mode: the (unit, symbol) the NEXT run starts at, or false.
    FCW_DI bool peek(const KParams& P, int& unit, int& n0) const {
        if constexpr (DYN) {
            return false;
        } else {
            if (pos >= hi) return false;
            unit = pos / P.B;
            n0 = pos - unit * P.B;
            return true;
        }
    }

    // Next run (unit, [n0, n1)); false when the team is done.
    FCW_DI bool next(const KParams& P, int* s_item, int g, int gtid, int nthr, int& unit, int& n0, int& n1) {
        if constexpr (!DYN) {
            if (pos >= hi) return false;
            unit = pos / P.B;
            n0 = pos - unit * P.B;
            n1 = min(P.B, n0 + min(P.chunk, hi - pos));
            pos += n1 - n0;
            return true;
        }
        // every run executes at least one team barrier after the previous
        // read of *s_item, so this publish cannot race it
        if (gtid == 0) *s_item = pending >= 0 ? pending : atomicAdd(P.item_counter, 1);
        team_sync<G>(g, nthr);
        const int item = *s_item;
        if (item >= P.n_items) return false;
        if (gtid == 0) pending = atomicAdd(P.item_counter, 1);  // next run, in flight
        unit = item / P.nchunks;
        n0 = (item - unit * P.nchunks) * P.chunk;
        n1 = min(P.B, n0 + P.chunk);
        return true;
    }
};

// Shared layout of both kernels' SMEM: G teams x {spec0, spec1}, then one
// warp scratch per warp, the short twiddle table and the long two-level table.
struct Smem {
    float2 *spec0, *spec1, *scr, *stw;
    float2* ltw;  // two-level long-transform twiddles: W_N^i (64), W_N^(64 h) (N/64)
    int* s_item;  // this team's run-id slot (dynamic mode)
};

// Two-level long-transform twiddle table in SMEM for N >= 1024 (no global
// loads inside the long transform); smaller N read the plan table directly.
template <int N>
constexpr int long_twl() {
    return N >= 1024 ? 6 : 0;
}
template <int G>
FCW_DI Smem smem_layout(const KParams& P, int g) {
    extern __shared__ float4 smem_raw[];
    float2* sm = reinterpret_cast<float2*>(smem_raw);
    Smem s;
    s.spec0 = sm + (2 * g) * P.spec_stride;
    s.spec1 = s.spec0 + P.spec_stride;
    float2* rest = sm + 2 * G * P.spec_stride;
    s.scr = rest + (threadIdx.x >> 5) * P.scratch_stride;
    s.stw = rest + kWarps * P.scratch_stride;
    s.ltw = s.stw + P.stab_len;
    s.s_item = reinterpret_cast<int*>(s.ltw + kLtwLen + P.tw16_len) + g;
    return s;
}

template <int N, int LU, bool DYN, int ZV = 0>
__global__ void __launch_bounds__(kThreads, min_blocks<LU, ZV>()) tx_kernel(const KParams P) {
    constexpr int G = teams_per_cta<N>();
    constexpr int T = N / kPPT;                  // long-transform threads per team
    constexpr int TT = G == 1 ? kThreads : T;    // threads per team
    const int tid = threadIdx.x;
    const int g = tid / TT, gtid = tid - g * TT;
    const bool act = gtid < T;
    Team tm{gtid, TT, gtid >> 5, TT / 32};
    __shared__ unsigned tmem_slot;
    unsigned tmem_base = 0;
    if constexpr (tmem_tw<N, ZV>()) tmem_base = tmem_tables<N>(P, &tmem_slot, tm);
    const Smem S = smem_layout<G>(P, g);
    float2 *spec0 = S.spec0, *spec1 = S.spec1;
    // The block-1 tail that overlaps the next symbol lives in a per-team global
    // (L2-resident) buffer: written and read back by this team only.
    float2* carry = P.carry + ((long long)blockIdx.x * G + g) * (N / 2);
    for (int i = tid; i < P.stab_len; i += kThreads) S.stw[i] = __ldg(&P.tw[i * (N / P.stab_len)]);
    if constexpr (long_twl<N>() > 0)
        for (int i = tid; i < 64 + N / 64; i += kThreads) S.ltw[i] = __ldg(&P.tw[i < 64 ? i : 64 * (i - 64)]);
    // tw16[sel][m][t] = W_256^(m (t + 64 sel)) for the half-warp FFT_256
    for (int i = tid; i < P.tw16_len; i += kThreads) {
        const int sel = i >> 8, m = (i >> 4) & 15, t = i & 15;
        S.ltw[kLtwLen + i] = __ldg(&P.tw[((m * (t + 64 * sel)) & 255) * (N / 256)]);
    }
    __syncthreads();

    // this thread's range of the owner-grouped fix-up list (constant for the whole launch)
    constexpr bool kOwnerFix = ZV != 1 && ZV != 2;
    const int own_k0 = act && kOwnerFix ? __ldg(&P.own_start[gtid]) : 0;
    const int own_k1 = act && kOwnerFix ? __ldg(&P.own_start[gtid + 1]) : 0;

    RunSource<G, DYN> runs(P, g);
    int unit, n0, n1;
    while (runs.next(P, S.s_item, g, gtid, TT, unit, n0, n1)) {
        const float2* in_u = P.in + (long long)unit * P.in_stride;
        float2* out_u = P.out + (long long)unit * P.out_stride;
        const int nfirst = n0 > 0 ? n0 - 1 : 0;
        if (gtid == 0) {
            prefetch_l2(in_u + (long long)nfirst * P.row_len, 8LL * P.row_len);
            int un, nn;  // static mode: the next run's first row is on its way too
            if (runs.peek(P, un, nn))
                prefetch_l2(P.in + (long long)un * P.in_stride + (long long)(nn > 0 ? nn - 1 : 0) * P.row_len,
                            8LL * P.row_len);
        }

        for (int n = nfirst; n < n1; ++n) {
            const SymDev sy = P.sym[n];
            team_sync<G>(g, TT);  // previous symbol's transform no longer reads spec
            if (gtid == 0 && n + 1 < n1) {
                prefetch_l2(in_u + (long long)(n + 1) * P.row_len, 8LL * P.row_len);
            }
            if constexpr (kOwnerFix) {
                // bins no subband touches are zeroed up front (the short stage never writes them;
                // the barrier after it publishes them with the scattered bins)
                for (int k = gtid; k < P.n_zero; k += TT) {
                    const int q = __ldg(&P.zero_list[k]);
                    FCW_ASSERT(q >= 0 && q < P.spec_stride);
                    spec0[q] = zero2();
                    spec1[q] = zero2();
                }
            }
            if (!FCW_SKIP(P, 1)) {
                // time-domain input (continuous FC, ZV == 0 kernels only) stages within a symbol only
                const bool cross = ZV != 0 || !P.td;
                tx_short_all<N, LU, ZV>(P, tm, sy, in_u + (long long)n * P.row_len,
                                        n + 1 < n1 && cross ? in_u + (long long)(n + 1) * P.row_len : nullptr,
                                        n > nfirst && cross, spec0, spec1, S.scr, S.stw);
            }
            team_sync<G>(g, TT);
            if constexpr (!kOwnerFix) {
                // zero fill and secondary contributions (rank order) in phases of their own:
                // narrowband kernels, where every thread reads the 16 live bins, and the zv
                // kernels, where the phases measured faster (C5 TX 5.75 vs 5.85 ms)
                for (int k = gtid; k < P.n_zero; k += TT) {
                    const int q = __ldg(&P.zero_list[k]);
                    FCW_ASSERT(q >= 0 && q < P.spec_stride);
                    spec0[q] = zero2();
                    spec1[q] = zero2();
                }
                for (int l = 0; l < P.n_lvl; ++l) {
                    for (int k = P.lvl_start[l] + gtid; k < P.lvl_start[l + 1]; k += TT) {
                        const int q = __ldg(&P.fix_tgt[k]), e = N + __ldg(&P.fix_slot[k]);
                        FCW_ASSERT(q >= 0 && q < N && e < P.spec_stride);
                        spec0[q] = cadd(spec0[q], spec0[e]);
                        spec1[q] = cadd(spec1[q], spec1[e]);
                    }
                    team_sync<G>(g, TT);
                }
                if (P.n_lvl == 0) team_sync<G>(g, TT);
            } else if (act) {
                // secondary contributions of shared transition bins: the thread that loads bin q
                // below (q mod T) adds them itself, in rank order: no phase, no barrier
                for (int k = own_k0; k < own_k1; ++k) {
                    const int q = __ldg(&P.own_tgt[k]), e = N + __ldg(&P.own_slot[k]);
                    FCW_ASSERT(q >= 0 && q < N && (q & (T - 1)) == gtid && e < P.spec_stride);
                    spec0[q] = cadd(spec0[q], spec0[e]);
                    spec1[q] = cadd(spec1[q], spec1[e]);
                }
            }

            float2 cr[8];
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int u = gtid + T * m;
                cr[m] = (act && n > nfirst && u < sy.carry_len) ? carry[u] : zero2();
            }
            // zv plans: no subband touches the guard band [7N/16, 9N/16), i.e.
            // elements m = 7, 8 of every thread (T = N/16): known-zero inputs
            constexpr unsigned long long ZG = (ZV == 1 && N == 4096) ? 0x0180ull : 0ull;
            float2 v[2][kPPT];
            if constexpr (ZV == 2) {
                // narrowband plan: one 16-point transform per thread (no exchange)
                if (act) nb_long_inverse<N>(v, spec0, spec1, P.tw, gtid, P.nb_k0);
                team_sync<G>(g, TT);  // the spectra are read before the next symbol rewrites them
            } else {
                if (act) {
#pragma unroll
                    for (int m = 0; m < kPPT; ++m) {
                        if (!((ZG >> m) & 1ull)) {
                            v[0][m] = spec0[gtid + T * m];
                            v[1][m] = spec1[gtid + T * m];
                        }
                    }
                }
                float2* const bufs[2] = {spec0, spec1};
                if (!FCW_SKIP(P, 2))
                    team_fft<N, T, kPPT, +1, 2, true, tmem_tw_long<N, ZV>() ? kTwTmem : long_twl<N>(), ZG>(
                        v, bufs, long_twl<N>() ? S.ltw : P.tw, 1, gtid, act, G == 1 ? 0 : 1 + g, TT, tm.tm_a, tm.tm_c);
            }
            // every thread has read its carry before it is overwritten: the long
            // transform's exchange barriers already order that for N >= 512
            if (N < 512 || FCW_SKIP(P, 2)) team_sync<G>(g, TT);
            // symbol-wise overlap-add: block 0 at 0, block 1 at N/2, carry from n-1
            if (act) {
                const bool emit = n >= n0;
                float2* dst = out_u + sy.sigma;
#pragma unroll
                for (int mm = 0; mm < 24; ++mm) {
                    const int u = gtid + T * mm;
                    float2 val = zero2();
                    if (mm < 16) val = v[0][mm];
                    if (mm >= 8) val = cadd(val, v[1][mm - 8]);
                    if (mm < 8) val = cadd(val, cr[mm]);
                    // predicated single-instruction stores: the owned span goes to the waveform
                    // (streaming; an L2-side add under FCW_TX_ACCUMULATE), the rest to the carry
                    // (own_len = N + N_CP,n+1 >= N: the first 16 elements of a thread are always owned)
                    const bool own = mm < 16 || u < sy.own_len;
                    FCW_ASSERT(!(own && emit) || sy.sigma + u < P.Q);
                    FCW_ASSERT(own || u - sy.own_len < N / 2);
                    if (P.accumulate) red_add2_if(&dst[u], val, own && emit);
                    else stcs_if(&dst[u], val, own && emit);
                    if (mm >= 16) stg_if(&carry[own ? 0 : u - sy.own_len], val, !own);
                }
            }
        }
    }
    if constexpr (tmem_tw<N, ZV>()) tmem_release(tmem_base);
}

template <int N, int LU, bool DYN, int ZV = 0>
__global__ void __launch_bounds__(kThreads, min_blocks<LU, ZV>()) rx_kernel(const KParams P) {
    constexpr int G = teams_per_cta<N>();
    constexpr int T = N / kPPT;
    constexpr int TT = G == 1 ? kThreads : T;
    const int tid = threadIdx.x;
    const int g = tid / TT, gtid = tid - g * TT;
    const bool act = gtid < T;
    Team tm{gtid, TT, gtid >> 5, TT / 32};
    __shared__ unsigned tmem_slot;
    unsigned tmem_base = 0;
    if constexpr (tmem_tw<N, ZV>()) tmem_base = tmem_tables<N>(P, &tmem_slot, tm);
    const Smem S = smem_layout<G>(P, g);
    float2 *spec0 = S.spec0, *spec1 = S.spec1;
    for (int i = tid; i < P.stab_len; i += kThreads) S.stw[i] = __ldg(&P.tw[i * (N / P.stab_len)]);
    if constexpr (long_twl<N>() > 0)
        for (int i = tid; i < 64 + N / 64; i += kThreads) S.ltw[i] = __ldg(&P.tw[i < 64 ? i : 64 * (i - 64)]);
    // tw16[sel][m][t] = W_256^(m (t + 64 sel)) for the half-warp FFT_256
    for (int i = tid; i < P.tw16_len; i += kThreads) {
        const int sel = i >> 8, m = (i >> 4) & 15, t = i & 15;
        S.ltw[kLtwLen + i] = __ldg(&P.tw[((m * (t + 64 * sel)) & 255) * (N / 256)]);
    }
    __syncthreads();

    RunSource<G, DYN> runs(P, g);
    int unit, n0, n1;
    while (runs.next(P, S.s_item, g, gtid, TT, unit, n0, n1)) {
        const float2* in_u = P.in + (long long)unit * P.in_stride;
        float2* out_u = P.out + (long long)unit * P.out_stride;
        if (gtid == 0) {
            prefetch_l2(in_u + P.rx_base + P.sym[n0].sigma, 8LL * (3 * N / 2));
            int un, nn;  // static mode: the next run's first window is on its way too
            if (runs.peek(P, un, nn))
                prefetch_l2(P.in + (long long)un * P.in_stride + P.rx_base + P.sym[nn].sigma, 8LL * (3 * N / 2));
        }

        for (int n = n0; n < n1; ++n) {
            const SymDev sy = P.sym[n];
            if (gtid == 0 && n + 1 < n1) prefetch_l2(in_u + P.rx_base + P.sym[n + 1].sigma, 8LL * (3 * N / 2));
            float2 v[2][kPPT];
            bool bounded = false;  // continuous FC: zeros outside [0, wave_len) (rx_continuous pads)
            if constexpr (ZV == 0 || ZV == 3) bounded = P.td != nullptr;
            if (act && bounded) {
                const long long j0 = P.rx_base + sy.sigma + gtid;
#pragma unroll
                for (int mm = 0; mm < 24; ++mm) {
                    const long long j = j0 + T * mm;
                    const float2 val = (j >= 0 && j < P.wave_len) ? ld_stream(in_u + j) : zero2();
                    if (mm < 16) v[0][mm] = val;
                    if (mm >= 8) v[1][mm - 8] = val;
                }
            } else if (act) {
                // rx_segment (fc_sync.cpp:145-156): y0 = w[start, +N), y1 = w[start + N/2, +N)
                FCW_ASSERT(P.rx_base + sy.sigma >= 0 && P.rx_base + sy.sigma + 3 * N / 2 <= P.wave_len);
                const float2* src = in_u + P.rx_base + sy.sigma + gtid;
#pragma unroll
                for (int mm = 0; mm < 24; ++mm) {
                    const float2 val = ld_stream(&src[T * mm]);  // read-only, no L1 allocation
                    if (mm < 16) v[0][mm] = val;
                    if (mm >= 8) v[1][mm - 8] = val;
                }
            }
            team_sync<G>(g, TT);  // previous symbol's subband stage no longer reads spec
            if constexpr (ZV == 2) {
                // narrowband plan: 16-point transforms per thread + a fixed-order sum
                // over the team; only bins [k0, k0 + 16) are produced
                nb_long_forward<N, G>(v, spec0, spec1, spec0, P.tw, gtid, P.nb_k0, g, TT);
            } else {
            {
                float2* const bufs[2] = {spec0, spec1};
                if (!FCW_SKIP(P, 2))
                    team_fft<N, T, kPPT, -1, 2, true, tmem_tw_long<N, ZV>() ? kTwTmem : long_twl<N>()>(
                        v, bufs, long_twl<N>() ? S.ltw : P.tw, 1, gtid, act, G == 1 ? 0 : 1 + g, TT, tm.tm_a, tm.tm_c);
            }
            team_sync<G>(g, TT);
            if (act) {
#pragma unroll
                for (int m = 0; m < kPPT; ++m) {
                    spec0[gtid + T * m] = v[0][m];
                    spec1[gtid + T * m] = v[1][m];
                    if constexpr (LU == 256) {
                        // wrap-around copy of bins [0, L) at [N, N + L) (rx_short_half)
                        if (T * m < LU && gtid + T * m < LU) {
                            spec0[N + gtid + T * m] = v[0][m];
                            spec1[N + gtid + T * m] = v[1][m];
                        }
                    }
                }
            }
            }
            team_sync<G>(g, TT);
            if (!FCW_SKIP(P, 1))
                rx_short_all<N, LU, ZV>(P, tm, sy, spec0, spec1, out_u + (long long)n * P.row_len, S.scr, S.stw);
        }
    }
    if constexpr (tmem_tw<N, ZV>()) tmem_release(tmem_base);
}

// Dispatch tables filled by the per-N instantiation units.
using KernelFn = void (*)(KParams);
struct KernelPair {
    KernelFn tx, rx;        // static balanced ranges
    KernelFn tx_d, rx_d;    // dynamic runs
};

}  // namespace fcw
