// Kernel instantiations for N = 2048: uniform-L specialisations L = 16, 32, 64.
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NL(2048, 16)
FCW_KERNELS_NL(2048, 32)
FCW_KERNELS_NL(2048, 64)
}  // namespace fcw
