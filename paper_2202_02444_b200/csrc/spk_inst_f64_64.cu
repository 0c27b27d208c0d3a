// Instantiates the fused bound / eval kernels for precision double, MMAX 64.
#include "spk_kernels.cuh"
namespace spk {
SPK_DEFINE_DISPATCH(double, 64)
}  // namespace spk
