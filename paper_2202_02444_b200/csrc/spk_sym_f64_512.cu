// Instantiates the symbol-carrying kernels for precision double, MMAX 512.
#include "spk_symbolic.cuh"
namespace spk {
SPK_DEFINE_SYM_DISPATCH(double, 512, 16)
}  // namespace spk
