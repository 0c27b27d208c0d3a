// Instantiates the symbol-carrying kernels for precision float, MMAX 128.
#include "spk_symbolic.cuh"
namespace spk {
SPK_DEFINE_SYM_DISPATCH(float, 128, 16)
}  // namespace spk
