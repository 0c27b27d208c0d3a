// Instantiates the symbol-carrying kernels for precision double, MMAX 64.
#include "spk_symbolic.cuh"
namespace spk {
SPK_DEFINE_SYM_DISPATCH(double, 64, 32)
}  // namespace spk
