// Tensor-core conv instantiations for bf16 widths that are multiples of 8
// but not tile widths (MODE 1: padded to 32/64/128/256, runtime strides).
#include "conv_tc_dispatch.cuh"

namespace vp {
int conv_tc_pad_fwd(int64_t kd, int64_t nd, const FwdParams& p, void* part, cudaStream_t st) {
  return conv_mode<false, 1>(kd, nd, p, part, st);
}
int conv_tc_pad_dgrad(int64_t kd, int64_t nd, const FwdParams& p, void* part, cudaStream_t st) {
  return conv_mode<true, 1>(kd, nd, p, part, st);
}
}  // namespace vp
