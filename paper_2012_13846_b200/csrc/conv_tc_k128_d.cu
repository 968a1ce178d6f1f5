// Tensor-core conv instantiations: K width 128, dgrad (W read MN-major).
#include "conv_tc_dispatch.cuh"

namespace vp {
int conv_tc_k128_d(int64_t nd, const FwdParams& p, void* part, cudaStream_t st) {
  return conv_tc_nd<128, true>(nd, p, part, st);
}
}  // namespace vp
