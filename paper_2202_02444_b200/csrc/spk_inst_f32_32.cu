// Instantiates the fused bound / eval kernels for precision float, MMAX 32.
#include "spk_kernels.cuh"
namespace spk {
SPK_DEFINE_DISPATCH(float, 32)
}  // namespace spk
