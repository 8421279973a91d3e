// Instantiation helpers: each fcw_k_*.cu unit instantiates the kernels of a
// few long-transform sizes so nvcc runs them in parallel.
#pragma once

#include "fcw_device.cuh"

#define FCW_SPEC(NN, LL) \
    case LL:             \
        return KernelPair{tx_kernel<NN, LL, false>, rx_kernel<NN, LL, false>, tx_kernel<NN, LL, true>, \
                          rx_kernel<NN, LL, true>};

// Generic (mixed-L) kernel plus uniform-L specialisations for the common sizes.
#define FCW_KERNELS_FULL(NN)                                                   \
    KernelPair kernels_n##NN(int LU) {                                         \
        switch (LU) {                                                          \
            FCW_SPEC(NN, 16)                                                   \
            FCW_SPEC(NN, 32)                                                   \
            FCW_SPEC(NN, 64)                                                   \
            FCW_SPEC(NN, 128)                                                  \
            FCW_SPEC(NN, 256)                                                  \
            FCW_SPEC(NN, 512)                                                  \
            FCW_SPEC(NN, 1024)                                                 \
            default:                                                           \
                return KernelPair{tx_kernel<NN, 0, false>, rx_kernel<NN, 0, false>, tx_kernel<NN, 0, true>, \
                                  rx_kernel<NN, 0, true>};                     \
        }                                                                      \
    }

#define FCW_KERNELS_GENERIC(NN) \
    KernelPair kernels_n##NN(int) {                                                                  \
        return KernelPair{tx_kernel<NN, 0, false>, rx_kernel<NN, 0, false>, tx_kernel<NN, 0, true>, \
                          rx_kernel<NN, 0, true>};                                                  \
    }
