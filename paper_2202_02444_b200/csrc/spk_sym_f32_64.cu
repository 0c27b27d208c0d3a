// Instantiates the symbol-carrying kernels for precision float, MMAX 64.
#include "spk_symbolic.cuh"
namespace spk {
SPK_DEFINE_SYM_DISPATCH(float, 64, 32)
}  // namespace spk
