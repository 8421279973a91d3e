// Kernel instantiations for N = 2048: uniform-L specialisations L = 128, 256.
// N = 2048 kernels keep every complex helper packed (config 2: 43.3 vs 42.1 Gsamples/s
// with scalar products / fused steps; see FCW_PK_* in fcw_fft.cuh).
#define FCW_PK_MUL 1
#define FCW_PK_FMA 1
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NL(2048, 128)
FCW_KERNELS_NL(2048, 256)
}  // namespace fcw
