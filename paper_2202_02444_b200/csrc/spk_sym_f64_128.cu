// Instantiates the symbol-carrying kernels for precision double, MMAX 128.
#include "spk_symbolic.cuh"
namespace spk {
SPK_DEFINE_SYM_DISPATCH(double, 128, 16)
}  // namespace spk
