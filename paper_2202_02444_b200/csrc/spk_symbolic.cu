// Symbol-carrying policies (affine-truncate, affine-full).  Placeholder
// until the K3 truncate kernel lands: reports an unsupported shape.
#include "spk_kernels.cuh"
#include "spk_abi_internal.h"

namespace spk {

int launch_symbolic(const spk_net*, int, int, int, long long, int, const double*, const double*, double*,
                    double*, int8_t*, cudaStream_t) {
  return fail(SPK_ERR_UNSUPPORTED_SHAPE, "affine-truncate / affine-full kernels not built yet");
}
int launch_symbolic_aabb(const spk_net*, int, int, int, long long, const double*, const double*, double*,
                         double*, int8_t*, cudaStream_t) {
  return fail(SPK_ERR_UNSUPPORTED_SHAPE, "affine-truncate / affine-full kernels not built yet");
}

}  // namespace spk
