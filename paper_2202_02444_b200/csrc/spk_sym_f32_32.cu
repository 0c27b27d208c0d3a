// Instantiates the symbol-carrying kernels for precision float, MMAX 32.
#include "spk_symbolic.cuh"
namespace spk {
SPK_DEFINE_SYM_DISPATCH(float, 32, 32)
}  // namespace spk
