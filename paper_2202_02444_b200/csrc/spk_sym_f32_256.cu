// Instantiates the symbol-carrying kernels for precision float, MMAX 256.
#include "spk_symbolic.cuh"
namespace spk {
SPK_DEFINE_SYM_DISPATCH(float, 256, 16)
}  // namespace spk
