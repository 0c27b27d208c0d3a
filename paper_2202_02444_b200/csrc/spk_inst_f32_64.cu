// Instantiates the fused bound / eval kernels for precision float, MMAX 64.
#include "spk_kernels.cuh"
namespace spk {
SPK_DEFINE_DISPATCH(float, 64)
}  // namespace spk
