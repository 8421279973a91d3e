// Kernel instantiations for N = 4096: uniform-L specialisations L = 128, 256.
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NL(4096, 128)
FCW_KERNELS_NL(4096, 256)
}  // namespace fcw
