// Instantiates the fused range-marching round kernels for precision double.
#include "spk_march_pass.cuh"
namespace spk {
SPK_DEFINE_MARCH_DISPATCH(double)
}  // namespace spk
