// Instantiates the fused range-marching round kernels for precision float.
#include "spk_march_pass.cuh"
namespace spk {
SPK_DEFINE_MARCH_DISPATCH(float)
}  // namespace spk
