// Kernel instantiations for N = 2048: uniform-L specialisations L = 128, 256.
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NL(2048, 128)
FCW_KERNELS_NL(2048, 256)
}  // namespace fcw
