// Kernel instantiations for N = 4096, L = 256 with the zero-bin variant (ZV = 1).
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NLZ(4096, 256)
}  // namespace fcw
