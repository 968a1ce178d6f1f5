// Model glue for the SparseResNet training step: batch norm over rows,
// ReLU, residual add, global average pool per batch index, linear + softmax
// cross entropy, SGD with momentum.  No reference implementation exists
// (SPEC.md:185 lists BN/pool/activation math as a non-goal), so parity is
// self-defined against oracle/voxpipe_oracle.py.  Every reduction runs in a
// fixed order (per-block partials, then an ordered sum) -> deterministic.
#include "common.cuh"

namespace vp {

constexpr int kRowsPerBlock = 512;
constexpr int kGlueThreads = 256;

// Per-block per-channel partial sums. Thread layout: channel c = tid % C_eff,
// row lane r = tid / C_eff (C_eff = min(C, 256); channels beyond loop).
__global__ void __launch_bounds__(kGlueThreads)
bn_partial_kernel(const void* __restrict__ x, int dtype, const int32_t* n_dev, int64_t cap, int C,
                  const void* __restrict__ gy, const void* __restrict__ gy2, int gy_dtype,
                  const void* __restrict__ y, int y_dtype, int relu, const float* __restrict__ mean,
                  const float* __restrict__ rstd, float* __restrict__ part /*[blocks][2][C]*/) {
  __shared__ float s_a[kGlueThreads], s_b[kGlueThreads];
  const int n = load_count(n_dev, cap);
  const int64_t r0 = (int64_t)blockIdx.x * kRowsPerBlock;
  const int64_t r1 = (r0 + kRowsPerBlock < (int64_t)n) ? r0 + kRowsPerBlock : (int64_t)n;
  const int ceff = C < kGlueThreads ? C : kGlueThreads;
  const int lanes = kGlueThreads / ceff;
  const int tc = threadIdx.x % ceff, tr = threadIdx.x / ceff;
  for (int c0 = 0; c0 < C; c0 += ceff) {
    const int c = c0 + tc;
    float a = 0.f, b = 0.f;
    if (tr < lanes && c < C) {
      if (gy == nullptr) {  // stats: sum x, sum x^2
        for (int64_t r = r0 + tr; r < r1; r += lanes) {
          float v = ldf(x, dtype, r * C + c);
          a += v;
          b += v * v;
        }
      } else {  // backward: sum gy', sum gy' * xhat
        const float mu = mean[c], rs = rstd[c];
        for (int64_t r = r0 + tr; r < r1; r += lanes) {
          float g = ldf(gy, gy_dtype, r * C + c);
          if (gy2) g += ldf(gy2, gy_dtype, r * C + c);
          if (relu && ldf(y, y_dtype, r * C + c) <= 0.f) g = 0.f;
          float xh = (ldf(x, dtype, r * C + c) - mu) * rs;
          a += g;
          b += g * xh;
        }
      }
    }
    s_a[threadIdx.x] = a;
    s_b[threadIdx.x] = b;
    __syncthreads();
    if (tr == 0 && c < C) {
      float sa = 0.f, sb = 0.f;
      for (int l = 0; l < lanes; ++l) {
        sa += s_a[l * ceff + tc];
        sb += s_b[l * ceff + tc];
      }
      part[((int64_t)blockIdx.x * 2) * C + c] = sa;
      part[((int64_t)blockIdx.x * 2 + 1) * C + c] = sb;
    }
    __syncthreads();
  }
}

// Ordered sum over the blocks' partials (f64); block per channel chunk.
__global__ void bn_finalize_kernel(const float* __restrict__ part, int nblocks_cap, const int32_t* n_dev,
                                   int64_t cap, int C, float eps, float* out_a, float* out_b, int mode) {
  const int n = load_count(n_dev, cap);
  const int nb = (int)((n + kRowsPerBlock - 1) / kRowsPerBlock);
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    double sa = 0.0, sb = 0.0;
    for (int b = 0; b < nb; ++b) {
      sa += part[((int64_t)b * 2) * C + c];
      sb += part[((int64_t)b * 2 + 1) * C + c];
    }
    if (mode == 0) {  // mean, rstd (biased variance, as in training-mode BN)
      double mu = n > 0 ? sa / n : 0.0;
      double var = n > 0 ? sb / n - mu * mu : 0.0;
      if (var < 0) var = 0;
      out_a[c] = (float)mu;
      out_b[c] = (float)(1.0 / sqrt(var + (double)eps));
    } else {  // gbeta, ggamma
      out_a[c] = (float)sb;  // ggamma = sum gy' xhat
      out_b[c] = (float)sa;  // gbeta  = sum gy'
    }
  }
}

__global__ void bn_apply_kernel(const void* __restrict__ x, int dtype, const int32_t* n_dev, int64_t cap, int C,
                                const float* __restrict__ mean, const float* __restrict__ rstd,
                                const float* __restrict__ gamma, const float* __restrict__ beta,
                                const void* __restrict__ res, int res_dtype, int relu, void* __restrict__ y,
                                int y_dtype) {
  const int n = load_count(n_dev, cap);
  const int64_t total = (int64_t)n * C;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % C);
    float v = (ldf(x, dtype, e) - mean[c]) * rstd[c] * gamma[c] + beta[c];
    if (res) v += ldf(res, res_dtype, e);
    if (relu) v = fmaxf(v, 0.f);
    stf(y, y_dtype, e, v);
  }
}

__global__ void bn_backward_apply_kernel(const void* __restrict__ gy, const void* __restrict__ gy2, int gy_dtype, const void* __restrict__ y,
                                         int y_dtype, const void* __restrict__ x, int x_dtype, const int32_t* n_dev,
                                         int64_t cap, int C, const float* __restrict__ mean,
                                         const float* __restrict__ rstd, const float* __restrict__ gamma,
                                         int relu, const float* __restrict__ ggamma, const float* __restrict__ gbeta,
                                         void* __restrict__ gx, int gx_dtype, void* __restrict__ gres) {
  const int n = load_count(n_dev, cap);
  const int64_t total = (int64_t)n * C;
  const float inv_n = n > 0 ? 1.f / (float)n : 0.f;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % C);
    float g = ldf(gy, gy_dtype, e);
    if (gy2) g += ldf(gy2, gy_dtype, e);
    if (relu && ldf(y, y_dtype, e) <= 0.f) g = 0.f;
    const float xh = (ldf(x, x_dtype, e) - mean[c]) * rstd[c];
    const float v = gamma[c] * rstd[c] * (g - inv_n * gbeta[c] - xh * inv_n * ggamma[c]);
    stf(gx, gx_dtype, e, v);
    if (gres) stf(gres, gx_dtype, e, g);
  }
}

// ------------------------------------------------------------------ pooling
__global__ void batch_count_kernel(const int4* __restrict__ coords, const int32_t* n_dev, int64_t cap, int B,
                                   int32_t* counts) {
  const int n = load_count(n_dev, cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int b = coords[i].x;
    if (b >= 0 && b < B) atomicAdd(&counts[b], 1);
  }
}
__global__ void batch_starts_kernel(const int32_t* counts, int B, int32_t* starts) {
  __shared__ int s_warp[1024 / 32 + 1];
  __shared__ int s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < B; base += 1024) {
    int i = base + threadIdx.x, tot;
    int v = i < B ? counts[i] : 0;
    int e = block_exclusive_scan<1024>(v, s_warp, &tot);
    if (i < B) starts[i] = s_carry + e;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += tot;
    __syncthreads();
  }
}
// rows are batch-contiguous (voxelize+batch order, preserved by first-seen
// downsampling): segment b = [starts[b], starts[b]+counts[b]).
__global__ void pool_kernel(const void* __restrict__ x, int dtype, int C, int B, const int32_t* counts,
                            const int32_t* starts, float* out) {
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    const int s = starts[b], cnt = counts[b];
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
      float acc = 0.f;
      for (int r = 0; r < cnt; ++r) acc += ldf(x, dtype, (int64_t)(s + r) * C + c);
      out[(int64_t)b * C + c] = cnt > 0 ? acc / (float)cnt : 0.f;
    }
  }
}
__global__ void pool_backward_kernel(const float* __restrict__ gout, const int4* __restrict__ coords,
                                     const int32_t* __restrict__ counts, const int32_t* n_dev, int64_t cap, int C,
                                     void* gx, int gx_dtype) {
  const int n = load_count(n_dev, cap);
  const int64_t total = (int64_t)n * C;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / C;
    const int c = (int)(e - r * C);
    const int b = coords[r].x;
    stf(gx, gx_dtype, e, gout[(int64_t)b * C + c] / (float)counts[b]);
  }
}

// ------------------------------------------------------------------ linear + xent
// kernel 1: one block per sample: logits, softmax, per-sample loss,
// g_logits = (p - onehot)/B, g_pooled = g_logits @ W.
__global__ void xent_sample_kernel(const float* __restrict__ pooled, int B, int C, const float* __restrict__ w,
                                   const float* __restrict__ bias, int classes, const int32_t* __restrict__ labels,
                                   float* logits, float* g_logits, float* loss_b, float* g_pooled) {
  extern __shared__ float sm[];
  float* s_logit = sm;  // classes
  __shared__ float s_max, s_sum;
  const int b = blockIdx.x;
  for (int j = threadIdx.x; j < classes; j += blockDim.x) {
    float acc = bias[j];
    for (int c = 0; c < C; ++c) acc += w[(int64_t)j * C + c] * pooled[(int64_t)b * C + c];
    s_logit[j] = acc;
    logits[(int64_t)b * classes + j] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = -INFINITY;
    for (int j = 0; j < classes; ++j) m = fmaxf(m, s_logit[j]);
    float s = 0.f;
    for (int j = 0; j < classes; ++j) s += expf(s_logit[j] - m);
    s_max = m;
    s_sum = s;
    const int lab = labels[b];
    loss_b[b] = -(s_logit[lab] - m - logf(s));
  }
  __syncthreads();
  const int lab = labels[b];
  for (int j = threadIdx.x; j < classes; j += blockDim.x) {
    float p = expf(s_logit[j] - s_max) / s_sum;
    g_logits[(int64_t)b * classes + j] = (p - (j == lab ? 1.f : 0.f)) / (float)B;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float acc = 0.f;
    for (int j = 0; j < classes; ++j) acc += g_logits[(int64_t)b * classes + j] * w[(int64_t)j * C + c];
    g_pooled[(int64_t)b * C + c] = acc;
  }
}
// kernel 2: fc grads and the mean loss, summed over samples in order.
__global__ void xent_reduce_kernel(const float* __restrict__ pooled, int B, int C, int classes,
                                   const float* __restrict__ g_logits, const float* __restrict__ loss_b,
                                   float* g_w, float* g_b, float* loss) {
  const int64_t total = (int64_t)classes * (C + 1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / (C + 1));
    const int c = (int)(e - (int64_t)j * (C + 1));
    float acc = 0.f;
    if (c < C) {
      for (int b = 0; b < B; ++b) acc += g_logits[(int64_t)b * classes + j] * pooled[(int64_t)b * C + c];
      g_w[(int64_t)j * C + c] = acc;
    } else {
      for (int b = 0; b < B; ++b) acc += g_logits[(int64_t)b * classes + j];
      g_b[j] = acc;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    float s = 0.f;
    for (int b = 0; b < B; ++b) s += loss_b[b];
    *loss = s / (float)B;
  }
}

__global__ void sgd_kernel(float* __restrict__ p, float* __restrict__ m, const float* __restrict__ g, int64_t n,
                           float lr, float mom, __nv_bfloat16* __restrict__ pb, int64_t nb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float mi = mom * m[i] + g[i];
    float pi = p[i] - lr * mi;
    m[i] = mi;
    p[i] = pi;
    if (pb && i < nb) pb[i] = __float2bfloat16_rn(pi);
  }
}

static int grid_for(int64_t total) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), kNumSMs * 16)); }

}  // namespace vp

using namespace vp;

extern "C" {

size_t vp_bn_stats_ws_bytes(int64_t cap_n, int64_t C) {
  return align_up((size_t)std::max<int64_t>(1, ceil_div(cap_n, kRowsPerBlock)) * 2 * C * 4, 256);
}

int vp_bn_stats(const void* x, int32_t xd, const int32_t* n_dev, int64_t cap, int64_t C, float eps, float* mean,
                float* rstd, void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(ws_bytes >= vp_bn_stats_ws_bytes(cap, C), VP_EVALIDATION, "bn_stats: workspace too small");
  const int nb = (int)std::max<int64_t>(1, ceil_div(cap, kRowsPerBlock));
  bn_partial_kernel<<<nb, kGlueThreads, 0, st>>>(x, xd, n_dev, cap, (int)C, nullptr, nullptr, 0, nullptr, 0, 0,
                                                  nullptr, nullptr, (float*)ws);
  VP_CHECK_LAUNCH("bn_partial");
  bn_finalize_kernel<<<(int)ceil_div(C, 128), 128, 0, st>>>((const float*)ws, nb, n_dev, cap, (int)C, eps, mean,
                                                            rstd, 0);
  VP_CHECK_LAUNCH("bn_finalize");
  return VP_OK;
}

int vp_bn_apply(const void* x, int32_t xd, const int32_t* n_dev, int64_t cap, int64_t C, const float* mean,
                const float* rstd, const float* gamma, const float* beta, const void* res, int32_t rd, int32_t relu,
                void* y, int32_t yd, vp_stream_t stream) {
  if (cap <= 0) return VP_OK;
  bn_apply_kernel<<<grid_for(cap * C), 256, 0, (cudaStream_t)stream>>>(x, xd, n_dev, cap, (int)C, mean, rstd, gamma,
                                                                      beta, res, rd, relu, y, yd);
  VP_CHECK_LAUNCH("bn_apply");
  return VP_OK;
}

size_t vp_bn_backward_ws_bytes(int64_t cap_n, int64_t C) { return vp_bn_stats_ws_bytes(cap_n, C); }

int vp_bn_backward(const void* gy, const void* gy2, int32_t gyd, const void* y, int32_t yd, const void* x, int32_t xd,
                   const int32_t* n_dev, int64_t cap, int64_t C, const float* mean, const float* rstd,
                   const float* gamma, int32_t relu, void* gx, int32_t gxd, void* gres, float* ggamma, float* gbeta,
                   void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(ws_bytes >= vp_bn_backward_ws_bytes(cap, C), VP_EVALIDATION, "bn_backward: workspace too small");
  const int nb = (int)std::max<int64_t>(1, ceil_div(cap, kRowsPerBlock));
  bn_partial_kernel<<<nb, kGlueThreads, 0, st>>>(x, xd, n_dev, cap, (int)C, gy, gy2, gyd, y, yd, relu, mean, rstd,
                                                  (float*)ws);
  VP_CHECK_LAUNCH("bn_bwd_partial");
  bn_finalize_kernel<<<(int)ceil_div(C, 128), 128, 0, st>>>((const float*)ws, nb, n_dev, cap, (int)C, 0.f, ggamma,
                                                            gbeta, 1);
  VP_CHECK_LAUNCH("bn_bwd_finalize");
  if (cap > 0) {
    bn_backward_apply_kernel<<<grid_for(cap * C), 256, 0, st>>>(gy, gy2, gyd, y, yd, x, xd, n_dev, cap, (int)C, mean, rstd,
                                                                gamma, relu, ggamma, gbeta, gx, gxd, gres);
    VP_CHECK_LAUNCH("bn_bwd_apply");
  }
  return VP_OK;
}

size_t vp_global_pool_ws_bytes(int32_t B) { return align_up((size_t)B * 4, 256); }

int vp_global_pool(const void* x, int32_t xd, const int32_t* coords, const int32_t* n_dev, int64_t cap, int64_t C,
                   int32_t B, float* out, int32_t* counts, void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(ws_bytes >= vp_global_pool_ws_bytes(B), VP_EVALIDATION, "global_pool: workspace too small");
  int32_t* starts = (int32_t*)ws;
  cudaMemsetAsync(counts, 0, sizeof(int32_t) * B, st);
  if (cap > 0) {
    batch_count_kernel<<<grid_for(cap), 256, 0, st>>>((const int4*)coords, n_dev, cap, B, counts);
    VP_CHECK_LAUNCH("batch_count");
  }
  batch_starts_kernel<<<1, 1024, 0, st>>>(counts, B, starts);
  VP_CHECK_LAUNCH("batch_starts");
  pool_kernel<<<std::min(B, kNumSMs * 4), C < 256 ? (int)C : 256, 0, st>>>(x, xd, (int)C, B, counts, starts, out);
  VP_CHECK_LAUNCH("pool");
  return VP_OK;
}

int vp_global_pool_backward(const float* gout, const int32_t* coords, const int32_t* counts, const int32_t* n_dev,
                            int64_t cap, int64_t C, void* gx, int32_t gxd, vp_stream_t stream) {
  if (cap <= 0) return VP_OK;
  pool_backward_kernel<<<grid_for(cap * C), 256, 0, (cudaStream_t)stream>>>(gout, (const int4*)coords, counts, n_dev,
                                                                           cap, (int)C, gx, gxd);
  VP_CHECK_LAUNCH("pool_backward");
  return VP_OK;
}

size_t vp_linear_xent_ws_bytes(int32_t B, int32_t classes) { return align_up((size_t)B * (classes + 1) * 4, 256); }

int vp_linear_xent(const float* pooled, int32_t B, int32_t C, const float* w, const float* b, int32_t classes,
                   const int32_t* labels, float* logits, float* loss, float* g_pooled, float* g_w, float* g_b,
                   void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(ws_bytes >= vp_linear_xent_ws_bytes(B, classes), VP_EVALIDATION, "linear_xent: workspace too small");
  float* g_logits = (float*)ws;
  float* loss_b = g_logits + (size_t)B * classes;
  xent_sample_kernel<<<B, 128, classes * sizeof(float), st>>>(pooled, B, C, w, b, classes, labels, logits, g_logits,
                                                             loss_b, g_pooled);
  VP_CHECK_LAUNCH("xent_sample");
  xent_reduce_kernel<<<grid_for((int64_t)classes * (C + 1)), 256, 0, st>>>(pooled, B, C, classes, g_logits, loss_b,
                                                                          g_w, g_b, loss);
  VP_CHECK_LAUNCH("xent_reduce");
  return VP_OK;
}

int vp_sgd_momentum(float* p, float* m, const float* g, int64_t n, float lr, float momentum, void* pb, int64_t nb,
                    vp_stream_t stream) {
  if (n <= 0) return VP_OK;
  sgd_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(p, m, g, n, lr, momentum, (__nv_bfloat16*)pb, nb);
  VP_CHECK_LAUNCH("sgd");
  return VP_OK;
}

}  // extern "C"
