// Kernel instantiations for N = 4096: uniform-L specialisations L = 16, 32, 64.
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NL(4096, 16)
FCW_KERNELS_NL(4096, 32)
FCW_KERNELS_NL(4096, 64)
}  // namespace fcw
