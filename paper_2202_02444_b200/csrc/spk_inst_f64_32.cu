// Instantiates the fused bound / eval kernels for precision double, MMAX 32.
#include "spk_kernels.cuh"
namespace spk {
SPK_DEFINE_DISPATCH(double, 32)
}  // namespace spk
