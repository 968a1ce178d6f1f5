// Tensor-core conv instantiations: K width 256, dgrad (W read MN-major).
#include "conv_tc_dispatch.cuh"

namespace vp {
int conv_tc_k256_d(int64_t nd, const FwdParams& p, void* part, cudaStream_t st) {
  return conv_tc_nd<256, true>(nd, p, part, st);
}
}  // namespace vp
