// kernels_tile.cu -- Cartesian constant-coefficient 3D tile kernel (placeholder until written).
#include "internal.h"

namespace mf {

bool cart_tile_supported(const Geo &) { return false; }

cudaError_t launch_apply_cart_tile(const Geo &, const Tables &, const double *, double *, cudaStream_t,
                                   int64_t *) {
  return cudaErrorNotSupported;
}

}  // namespace mf
