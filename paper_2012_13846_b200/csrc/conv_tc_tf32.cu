// Tensor-core conv instantiations for fp32 features with tf32 math
// (kind::tf32, MODE 2): K widths in 2-byte units 32..256 (C_in 16..128 fp32).
#include "conv_tc_dispatch.cuh"

namespace vp {
int conv_tc_tf32(int64_t kd, int64_t nd, const FwdParams& p, void* part, cudaStream_t st) {
  return conv_mode<false, 2>(kd, nd, p, part, st);
}
}  // namespace vp
