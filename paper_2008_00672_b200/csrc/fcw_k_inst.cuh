// Instantiation helpers: each fcw_k_*.cu unit instantiates the kernels of one
// long-transform size N and a few short sizes L, so nvcc runs them in parallel.
#pragma once

#include "fcw_device.cuh"

// kernels_n<N>_l<L>(): the four kernels (static / dynamic schedule, TX / RX)
// specialised for a uniform short size L (0 = the generic mixed-L kernels).
#define FCW_KERNELS_NL(NN, LL)                                                                  \
    KernelPair kernels_n##NN##_l##LL() {                                                        \
        return KernelPair{tx_kernel<NN, LL, false>, rx_kernel<NN, LL, false>, tx_kernel<NN, LL, true>, \
                          rx_kernel<NN, LL, true>};                                             \
    }

// ... and the variant whose subbands leave DFT bins t + 16m, m in [5, 10],
// inactive and outside the window (ZV = 1, L = 256: see tx_short_half).
#define FCW_KERNELS_NLZ(NN, LL)                                                                   \
    KernelPair kernels_n##NN##_l##LL##z() {                                                       \
        return KernelPair{tx_kernel<NN, LL, false, 1>, rx_kernel<NN, LL, false, 1>,              \
                          tx_kernel<NN, LL, true, 1>, rx_kernel<NN, LL, true, 1>};               \
    }

// ... and the narrowband variant (ZV = 2: every subband span inside 16 bins).
#define FCW_KERNELS_NLN(NN, LL)                                                                   \
    KernelPair kernels_n##NN##_l##LL##n() {                                                       \
        return KernelPair{tx_kernel<NN, LL, false, 2>, rx_kernel<NN, LL, false, 2>,              \
                          tx_kernel<NN, LL, true, 2>, rx_kernel<NN, LL, true, 2>};               \
    }

// ... and the team-only variant (ZV = 3: uniform L >= 512 with at most one
// subband per two warps of a team, e.g. config 3's banks): the whole team
// transforms each subband at 4-8 points per thread, two CTAs per SM.
#define FCW_KERNELS_NLT(NN, LL)                                                                   \
    KernelPair kernels_n##NN##_l##LL##t() {                                                       \
        return KernelPair{tx_kernel<NN, LL, false, 3>, rx_kernel<NN, LL, false, 3>,              \
                          tx_kernel<NN, LL, true, 3>, rx_kernel<NN, LL, true, 3>};               \
    }
