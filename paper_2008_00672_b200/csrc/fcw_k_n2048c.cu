// Kernel instantiations for N = 2048: uniform-L specialisations L = 512, 1024.
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NL(2048, 512)
FCW_KERNELS_NL(2048, 1024)
}  // namespace fcw
