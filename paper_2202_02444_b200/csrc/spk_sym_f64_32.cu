// Instantiates the symbol-carrying kernels for precision double, MMAX 32.
#include "spk_symbolic.cuh"
namespace spk {
SPK_DEFINE_SYM_DISPATCH(double, 32, 32)
}  // namespace spk
