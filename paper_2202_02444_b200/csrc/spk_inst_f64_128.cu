// Instantiates the fused bound / eval kernels for precision double, MMAX 128.
#include "spk_kernels.cuh"
namespace spk {
SPK_DEFINE_DISPATCH(double, 128)
}  // namespace spk
