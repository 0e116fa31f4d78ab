// placeholder until the backward kernels land
#include <cuda_runtime.h>
#include "ffa_common.cuh"
namespace magi {
cudaError_t launch_ffa_bwd(const FwdTile*, const FwdItem*, int, const BwdTile*, const BwdItem*, int,
                           int, int, int, int, int, float, const void*, const void*, const void*,
                           const float*, const float*, const void*, void*, void*, void*, int, int,
                           cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace magi
