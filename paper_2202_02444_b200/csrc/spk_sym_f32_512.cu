// Instantiates the symbol-carrying kernels for precision float, MMAX 512.
#include "spk_symbolic.cuh"
namespace spk {
SPK_DEFINE_SYM_DISPATCH(float, 512, 16)
}  // namespace spk
