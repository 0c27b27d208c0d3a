// Instantiates the fused bound / eval kernels for precision float, MMAX 128.
#include "spk_kernels.cuh"
namespace spk {
SPK_DEFINE_DISPATCH(float, 128)
}  // namespace spk
