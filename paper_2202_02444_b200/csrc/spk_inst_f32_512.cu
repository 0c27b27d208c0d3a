// Instantiates the fused bound / eval kernels for precision float, MMAX 512.
#include "spk_kernels.cuh"
namespace spk {
SPK_DEFINE_DISPATCH(float, 512)
}  // namespace spk
