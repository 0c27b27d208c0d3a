// Instantiates the fused bound / eval kernels for precision double, MMAX 256.
#include "spk_kernels.cuh"
namespace spk {
SPK_DEFINE_DISPATCH(double, 256)
}  // namespace spk
