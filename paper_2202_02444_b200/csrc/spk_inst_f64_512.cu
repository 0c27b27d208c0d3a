// Instantiates the fused bound / eval kernels for precision double, MMAX 512.
#include "spk_kernels.cuh"
namespace spk {
SPK_DEFINE_DISPATCH(double, 512)
}  // namespace spk
