// Kernel instantiations for N = 1024: uniform-L specialisations L = 128, 256.
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NL(1024, 128)
FCW_KERNELS_NL(1024, 256)
}  // namespace fcw
