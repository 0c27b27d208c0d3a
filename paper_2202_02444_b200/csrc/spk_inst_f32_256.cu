// Instantiates the fused bound / eval kernels for precision float, MMAX 256.
#include "spk_kernels.cuh"
namespace spk {
SPK_DEFINE_DISPATCH(float, 256)
}  // namespace spk
