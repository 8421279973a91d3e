// Kernel instantiations for N = 1024: uniform-L specialisations L = 16, 32, 64.
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NL(1024, 16)
FCW_KERNELS_NL(1024, 32)
FCW_KERNELS_NL(1024, 64)
}  // namespace fcw
