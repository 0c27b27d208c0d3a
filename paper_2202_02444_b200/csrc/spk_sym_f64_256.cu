// Instantiates the symbol-carrying kernels for precision double, MMAX 256.
#include "spk_symbolic.cuh"
namespace spk {
SPK_DEFINE_SYM_DISPATCH(double, 256, 16)
}  // namespace spk
