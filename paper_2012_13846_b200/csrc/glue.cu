// Model glue for the SparseResNet training step: batch norm over rows,
// ReLU, residual add, global average pool per batch index, linear + softmax
// cross entropy, SGD with momentum.  No reference implementation exists
// (SPEC.md:185 lists BN/pool/activation math as a non-goal), so parity is
// self-defined against oracle/voxpipe_oracle.py.  Every reduction runs in a
// fixed order (per-block partials, then an ordered sum) -> deterministic.
#include <cstdlib>
#include <initializer_list>

#include "bn_epi.cuh"
#include "common.cuh"

namespace vp {

constexpr int kGlueThreads = 256;

// 8-wide (16 B for bf16) vector access; VEC == 1 is the scalar fallback for
// channel counts that are not a multiple of 8.  DT >= 0 fixes the dtype at
// compile time: with no dtype branch between them the compiler keeps every
// load of an unrolled row batch in flight (a runtime switch serialised them).
template <int VEC, int DT = -1>
__device__ __forceinline__ void ldv(const void* p, int dtype_rt, int64_t i, float* v) {
  const int dtype = DT >= 0 ? DT : dtype_rt;
  if (VEC == 8 && dtype == VP_BF16) {
    uint4 raw = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p) + i);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float2 f = __bfloat1622float2(h[q]);
      v[2 * q] = f.x;
      v[2 * q + 1] = f.y;
    }
  } else if (VEC == 8 && dtype == VP_F32) {
    const float4* f = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p) + i);
    float4 a = f[0], b = f[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int q = 0; q < VEC; ++q) v[q] = ldf(p, dtype, i + q);
  }
}
template <int VEC, int DT = -1>
__device__ __forceinline__ void stv(void* p, int dtype_rt, int64_t i, const float* v) {
  const int dtype = DT >= 0 ? DT : dtype_rt;
  if (VEC == 8 && dtype == VP_BF16) {
    uint4 raw;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
    for (int q = 0; q < 4; ++q) h[q] = __floats2bfloat162_rn(v[2 * q], v[2 * q + 1]);
    *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p) + i) = raw;
  } else if (VEC == 8 && dtype == VP_F32) {
    float4* f = reinterpret_cast<float4*>(reinterpret_cast<float*>(p) + i);
    f[0] = make_float4(v[0], v[1], v[2], v[3]);
    f[1] = make_float4(v[4], v[5], v[6], v[7]);
  } else {
#pragma unroll
    for (int q = 0; q < VEC; ++q) stf(p, dtype, i + q, v[q]);
  }
}

// Raw row vectors: a batch of loads is issued into these before any of it is
// converted (bf16 rows stay packed: 4 registers per 8 channels), so deep
// batches fit in registers.  Generic dtypes convert at load.
template <int VEC, int DT>
struct RawVec {
  float v[VEC];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int q = 0; q < VEC; ++q) v[q] = 0.f;
  }
  __device__ __forceinline__ void load(const void* p, int dt, int64_t i) { ldv<VEC, DT>(p, dt, i, v); }
  __device__ __forceinline__ void get(float* o) const {
#pragma unroll
    for (int q = 0; q < VEC; ++q) o[q] = v[q];
  }
};
template <>
struct RawVec<8, VP_BF16> {
  uint4 r;
  __device__ __forceinline__ void zero() { r = make_uint4(0u, 0u, 0u, 0u); }
  __device__ __forceinline__ void load(const void* p, int, int64_t i) {
    r = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p) + i);
  }
  __device__ __forceinline__ void get(float* o) const {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __bfloat1622float2(h[q]);
      o[2 * q] = f.x;
      o[2 * q + 1] = f.y;
    }
  }
};
// rows per batch: deeper for the packed bf16 rows
template <int VEC, int DT>
struct BnDepth {
  static constexpr int stats = (VEC == 8 && DT == VP_BF16) ? 8 : 4;
  static constexpr int bwd = (VEC == 8 && DT == VP_BF16) ? 4 : 2;
  static constexpr int apply = (VEC == 8 && DT == VP_BF16) ? 4 : 2;
};

// Fused BN (one cooperative launch): after the statistics, every block waits
// for the last block's result (epoch flag) and applies the normalisation to
// its rows.  mode 0 = statistics only, 1 = forward apply, 2 = backward apply.
struct BnFuse {
  int mode;
  int* epoch;
  const float* gamma;
  const float* beta;
  const void* res;
  int res_dtype;
  int relu;
  void* out;
  int out_dtype;
  void* gres;
};

template <int VEC, int DT>
__device__ __forceinline__ void bn_apply_rows(const void* __restrict__ x, int dtype, int n, int C,
                                              const float* __restrict__ mean, const float* __restrict__ rstd,
                                              const float* __restrict__ gamma, const float* __restrict__ beta,
                                              const void* __restrict__ res, int res_dtype, int relu,
                                              void* __restrict__ y, int y_dtype, int blk, int nblk);
template <int VEC, int DT>
__device__ __forceinline__ void bn_backward_apply_rows(
    const void* __restrict__ gy, const void* __restrict__ gy2, int gy_dtype, const void* __restrict__ y, int y_dtype,
    const void* __restrict__ x, int x_dtype, int n, int C, const float* __restrict__ mean,
    const float* __restrict__ rstd, const float* __restrict__ gamma, int relu, const float* __restrict__ ggamma,
    const float* __restrict__ gbeta, void* __restrict__ gx, int gx_dtype, void* __restrict__ gres, int blk, int nblk);

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int VEC, int DT>
__device__ __forceinline__ void bn_fused_apply(const void* x, int dtype, int n, int C, const void* gy, const void* gy2,
                                               int gy_dtype, const void* y, int y_dtype, int relu, const float* mean,
                                               const float* rstd, const float* out_a, const float* out_b,
                                               const BnFuse& F) {
  if (F.mode == 1)  // forward: out_a/out_b = mean/rstd just computed
    bn_apply_rows<VEC, DT>(x, dtype, n, C, out_a, out_b, F.gamma, F.beta, F.res, F.res_dtype, F.relu, F.out, F.out_dtype,
                       blockIdx.x, gridDim.x);
  else  // backward: out_a/out_b = ggamma/gbeta
    bn_backward_apply_rows<VEC, DT>(gy, gy2, gy_dtype, y, y_dtype, x, dtype, n, C, mean, rstd, F.gamma, relu, out_a,
                                out_b, F.out, F.out_dtype, F.gres, blockIdx.x, gridDim.x);
}

// Reduce the per-block partials [nb][2][C] in a fixed order (same result in
// every block that calls it) and write (mean, rstd) for stats (gy == null in
// the producer) or (ggamma, gbeta) = (sum g*xhat, sum g) to out_a / out_b.
// Called by all threads of a block; ends with a __syncthreads.
__device__ __noinline__ void bn_finalize(const float* __restrict__ part, int nb, int C, int n, bool stats, float eps,
                                         float* __restrict__ out_a, float* __restrict__ out_b) {
  __shared__ double d_a[4 * kGlueThreads], d_b[4 * kGlueThreads];  // [G][cc][4]
  // channel quads (4 channels as one float4 of a and one of b) when C % 4 == 0,
  // else single channels; the G thread groups stride over the blocks with 4
  // block rows (8 loads) in flight, then the groups are summed in order
  const int W = (C % 4 == 0) ? 4 : 1;
  const int units = C / W;
  for (int u0 = 0; u0 < units; u0 += kGlueThreads) {
    const int cc = min(units - u0, kGlueThreads);
    const int G = kGlueThreads / cc;  // block groups per unit
    const int uu = u0 + threadIdx.x % cc, g = threadIdx.x / cc;
    double a4[4] = {0.0, 0.0, 0.0, 0.0}, b4[4] = {0.0, 0.0, 0.0, 0.0};
    if (g < G) {
      if (W == 4) {
        for (int b0 = g; b0 < nb; b0 += 4 * G) {
          float4 ta[4], tb[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int b = b0 + q * G;
            ta[q] = tb[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (b < nb) {
              ta[q] = __ldcg(reinterpret_cast<const float4*>(part + ((int64_t)b * 2) * C) + uu);
              tb[q] = __ldcg(reinterpret_cast<const float4*>(part + ((int64_t)b * 2 + 1) * C) + uu);
            }
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            a4[0] += ta[q].x; a4[1] += ta[q].y; a4[2] += ta[q].z; a4[3] += ta[q].w;
            b4[0] += tb[q].x; b4[1] += tb[q].y; b4[2] += tb[q].z; b4[3] += tb[q].w;
          }
        }
      } else {
        for (int b0 = g; b0 < nb; b0 += 4 * G) {
          float ta[4], tb[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int b = b0 + q * G;
            ta[q] = b < nb ? __ldcg(part + ((int64_t)b * 2) * C + uu) : 0.f;
            tb[q] = b < nb ? __ldcg(part + ((int64_t)b * 2 + 1) * C + uu) : 0.f;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            a4[0] += ta[q];
            b4[0] += tb[q];
          }
        }
      }
    }
    __syncthreads();
    if (g < G) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        d_a[(g * cc + threadIdx.x % cc) * 4 + k] = a4[k];
        d_b[(g * cc + threadIdx.x % cc) * 4 + k] = b4[k];
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < cc * W; e += kGlueThreads) {
      const int i = e / W, k = e % W;
      double sa = 0.0, sb = 0.0;
      for (int gg = 0; gg < G; ++gg) {
        sa += d_a[(gg * cc + i) * 4 + k];
        sb += d_b[(gg * cc + i) * 4 + k];
      }
      const int ch = (u0 + i) * W + k;
      if (stats) {  // mean, rstd (biased variance, training-mode BN)
        const double mu = n > 0 ? sa / n : 0.0;
        double var = n > 0 ? sb / n - mu * mu : 0.0;
        if (var < 0) var = 0;
        out_a[ch] = (float)mu;
        out_b[ch] = (float)(1.0 / sqrt(var + (double)eps));
      } else {  // ggamma = sum g*xhat, gbeta = sum g
        out_a[ch] = (float)sb;
        out_b[ch] = (float)sa;
      }
    }
    __syncthreads();
  }
}

// Per-block per-channel partial sums over `rpb` rows.  Thread layout: tpr =
// C/VEC threads cover one row (VEC channels each), lanes = 256/tpr rows in
// flight.  stats mode (gy == null): (sum x, sum x^2); backward mode:
// (sum g, sum g*xhat) with g = (gy [+ gy2]) masked by (y > 0) when relu.
template <int VEC, int DT>
__global__ void __launch_bounds__(kGlueThreads)
bn_partial_kernel(const void* __restrict__ x, int dtype, const int32_t* n_dev, int64_t cap, int C,
                  const void* __restrict__ gy, const void* __restrict__ gy2, int gy_dtype,
                  const void* __restrict__ y, int y_dtype, int relu, const float* __restrict__ mean,
                  const float* __restrict__ rstd, float* __restrict__ part /*[blocks][2][C]*/,
                  int* __restrict__ ticket, float eps, float* __restrict__ out_a, float* __restrict__ out_b,
                  const BnFuse F) {
  ::vp::pdl_begin();
  __shared__ float s_a[kGlueThreads * VEC], s_b[kGlueThreads * VEC];
  const int n = load_count(n_dev, cap);
  const int e0 = F.mode ? ld_acquire(F.epoch) : 0;  // before arriving: the last block bumps it
  const int tpr = C / VEC;
  const int lanes = kGlueThreads / tpr;
  const int cv = threadIdx.x % tpr, lr = threadIdx.x / tpr;
  const int c0 = cv * VEC;
  float a[VEC], b[VEC], mu[VEC], rs[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q) a[q] = b[q] = 0.f;
  const int64_t stride = (int64_t)gridDim.x * lanes;
  if (lr < lanes) {
    if (gy == nullptr) {
      // block b owns row groups b, b+G, b+2G, ... (G = gridDim.x, fixed per
      // capacity) -> balanced for any live n, fixed summation order.  Rows
      // are loaded in batches of 4 (all loads issued before the first add).
      constexpr int U = BnDepth<VEC, DT>::stats;
      for (int64_t r0 = (int64_t)blockIdx.x * lanes + lr; r0 < n; r0 += U * stride) {
        RawVec<VEC, DT> rv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t r = r0 + u * stride;
          rv[u].zero();
          if (r < n) rv[u].load(x, dtype, r * C + c0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float v[VEC];
          rv[u].get(v);
#pragma unroll
          for (int q = 0; q < VEC; ++q) {
            a[q] += v[q];
            b[q] += v[q] * v[q];
          }
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        mu[q] = mean[c0 + q];
        rs[q] = rstd[c0 + q];
      }
      constexpr int U = BnDepth<VEC, DT>::bwd;
      for (int64_t r0 = (int64_t)blockIdx.x * lanes + lr; r0 < n; r0 += U * stride) {
        RawVec<VEC, DT> rg[U], rg2[U], ry[U], rx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t r = r0 + u * stride;
          rg[u].zero();
          rg2[u].zero();
          ry[u].zero();
          rx[u].zero();
          if (r < n) {
            rg[u].load(gy, gy_dtype, r * C + c0);
            if (gy2) rg2[u].load(gy2, gy_dtype, r * C + c0);
            if (relu) ry[u].load(y, y_dtype, r * C + c0);
            rx[u].load(x, dtype, r * C + c0);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float g[VEC], g2[VEC], yy[VEC], xv[VEC];
          rg[u].get(g);
          rg2[u].get(g2);
          ry[u].get(yy);
          rx[u].get(xv);
#pragma unroll
          for (int q = 0; q < VEC; ++q) {
            const float gs = gy2 ? g[q] + g2[q] : g[q];
            const float gq = (relu && yy[q] <= 0.f) ? 0.f : gs;
            a[q] += gq;
            b[q] += gq * (xv[q] - mu[q]) * rs[q];
          }
        }
      }
    }
  }
  if (tpr <= 32 && 32 % tpr == 0) {
    // whole rows per warp: fixed xor tree over the warp's rows, then the 8
    // warps' sums in order (all threads busy instead of C serial sums)
#pragma unroll
    for (int q = 0; q < VEC; ++q)
      for (int m = tpr; m < 32; m <<= 1) {
        a[q] += __shfl_xor_sync(0xffffffffu, a[q], m);
        b[q] += __shfl_xor_sync(0xffffffffu, b[q], m);
      }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane < tpr) {
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        s_a[warp * C + lane * VEC + q] = a[q];
        s_b[warp * C + lane * VEC + q] = b[q];
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < C; e += kGlueThreads) {
      float sa = 0.f, sb = 0.f;
#pragma unroll
      for (int w2 = 0; w2 < kGlueThreads / 32; ++w2) {
        sa += s_a[w2 * C + e];
        sb += s_b[w2 * C + e];
      }
      part[((int64_t)blockIdx.x * 2) * C + e] = sa;
      part[((int64_t)blockIdx.x * 2 + 1) * C + e] = sb;
    }
  } else {
#pragma unroll
  for (int q = 0; q < VEC; ++q) {
    s_a[threadIdx.x * VEC + q] = a[q];
    s_b[threadIdx.x * VEC + q] = b[q];
  }
  __syncthreads();
  // fixed-order reduction over the row lanes: thread (cv, q) sums lanes 0..lanes-1
  for (int e = threadIdx.x; e < C; e += kGlueThreads) {
    const int ecv = e / VEC, q = e % VEC;
    float sa = 0.f, sb = 0.f;
    for (int l = 0; l < lanes; ++l) {
      sa += s_a[(l * tpr + ecv) * VEC + q];
      sb += s_b[(l * tpr + ecv) * VEC + q];
    }
    part[((int64_t)blockIdx.x * 2) * C + e] = sa;
    part[((int64_t)blockIdx.x * 2 + 1) * C + e] = sb;
  }
  }
  // ticket == null: the consumer kernel reduces the partials (bn_finalize in
  // every one of its blocks) -> no fence / ticket / serial tail here.
  if (ticket == nullptr) return;
  // The LAST block to finish reduces every block's partials in block order
  // (fixed order -> deterministic) and writes the statistics: one launch
  // instead of partial + finalize.
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  // atomicInc wraps to 0 after the last block: the ticket re-arms itself
  // (and a stale value recovers after one launch)
  if (threadIdx.x == 0) s_last = atomicInc(reinterpret_cast<unsigned int*>(ticket), gridDim.x - 1) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) {
    if (!F.mode) return;
    // cooperative launch: every block is resident, so waiting is safe
    if (threadIdx.x == 0)
      while (ld_acquire(F.epoch) == e0) __nanosleep(32);
    __syncthreads();
    bn_fused_apply<VEC, DT>(x, dtype, n, C, gy, gy2, gy_dtype, y, y_dtype, relu, mean, rstd, out_a, out_b, F);
    return;
  }
  __threadfence();
  bn_finalize(part, gridDim.x, C, n, gy == nullptr, eps, out_a, out_b);
  if (F.mode) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release(F.epoch, e0 + 1);
    bn_fused_apply<VEC, DT>(x, dtype, n, C, gy, gy2, gy_dtype, y, y_dtype, relu, mean, rstd, out_a, out_b, F);
  }
}

template <int VEC, int DT>
__device__ __forceinline__ void bn_apply_rows(const void* __restrict__ x, int dtype, int n, int C,
                                              const float* __restrict__ mean, const float* __restrict__ rstd,
                                              const float* __restrict__ gamma, const float* __restrict__ beta,
                                              const void* __restrict__ res, int res_dtype, int relu,
                                              void* __restrict__ y, int y_dtype, int blk, int nblk) {
  const int tpr = C / VEC, lanes = kGlueThreads / tpr;
  const int cv = threadIdx.x % tpr, lr = threadIdx.x / tpr;
  if (lr >= lanes) return;
  const int c0 = cv * VEC;
  float sc[VEC], sh[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q) {
    sc[q] = rstd[c0 + q] * gamma[c0 + q];
    sh[q] = beta[c0 + q] - mean[c0 + q] * sc[q];
  }
  const int64_t stride = (int64_t)nblk * lanes;
  constexpr int U = BnDepth<VEC, DT>::apply;
  for (int64_t r0 = (int64_t)blk * lanes + lr; r0 < n; r0 += U * stride) {
    RawVec<VEC, DT> rx[U], rr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u * stride;
      rx[u].zero();
      rr[u].zero();
      if (r < n) {
        rx[u].load(x, dtype, r * C + c0);
        if (res) rr[u].load(res, res_dtype, r * C + c0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u * stride;
      if (r >= n) break;
      float v[VEC], rv[VEC];
      rx[u].get(v);
      rr[u].get(rv);
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        float o = v[q] * sc[q] + sh[q];
        if (res) o += rv[q];
        v[q] = relu ? fmaxf(o, 0.f) : o;
      }
      stv<VEC, DT>(y, y_dtype, r * C + c0, v);
    }
  }
}

// part != null: (mean, rstd) are first reduced from the statistics kernel's
// per-block partials by every block (bn_finalize into shared memory); block 0
// also stores them to mean / rstd for the backward pass.
template <int VEC, int DT>
__global__ void __launch_bounds__(kGlueThreads)
bn_apply_kernel(const void* __restrict__ x, int dtype, const int32_t* n_dev, int64_t cap, int C,
                const float* __restrict__ mean, const float* __restrict__ rstd, const float* __restrict__ gamma,
                const float* __restrict__ beta, const void* __restrict__ res, int res_dtype, int relu,
                void* __restrict__ y, int y_dtype, const float* __restrict__ part, int nb, float eps,
                float* __restrict__ mean_out, float* __restrict__ rstd_out, const int* __restrict__ nb_dev) {
  extern __shared__ float s_stat[];
  ::vp::pdl_begin();
  const int n = load_count(n_dev, cap);
  if (part) {
    if (nb_dev) nb = *nb_dev;  // written by the producer (bn_epi.cuh)
    bn_finalize(part, nb, C, n, true, eps, s_stat, s_stat + C);
    if (blockIdx.x == 0)
      for (int c = threadIdx.x; c < C; c += kGlueThreads) {
        mean_out[c] = s_stat[c];
        rstd_out[c] = s_stat[C + c];
      }
    mean = s_stat;
    rstd = s_stat + C;
  }
  bn_apply_rows<VEC, DT>(x, dtype, n, C, mean, rstd, gamma, beta, res, res_dtype, relu, y, y_dtype,
                     blockIdx.x, gridDim.x);
}

template <int VEC, int DT>
__device__ __forceinline__ void bn_backward_apply_rows(
    const void* __restrict__ gy, const void* __restrict__ gy2, int gy_dtype, const void* __restrict__ y, int y_dtype,
    const void* __restrict__ x, int x_dtype, int n, int C, const float* __restrict__ mean,
    const float* __restrict__ rstd, const float* __restrict__ gamma, int relu, const float* __restrict__ ggamma,
    const float* __restrict__ gbeta, void* __restrict__ gx, int gx_dtype, void* __restrict__ gres, int blk, int nblk) {
  const int tpr = C / VEC, lanes = kGlueThreads / tpr;
  const int cv = threadIdx.x % tpr, lr = threadIdx.x / tpr;
  if (lr >= lanes) return;
  const int c0 = cv * VEC;
  const float inv_n = n > 0 ? 1.f / (float)n : 0.f;
  float k1[VEC], k2[VEC], k3[VEC], mu[VEC], rs[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q) {
    const int c = c0 + q;
    mu[q] = mean[c];
    rs[q] = rstd[c];
    k1[q] = gamma[c] * rs[q];         // gx = k1*(g - gbeta/n - xhat*ggamma/n)
    k2[q] = inv_n * gbeta[c];
    k3[q] = inv_n * ggamma[c];
  }
  const int64_t stride = (int64_t)nblk * lanes;
  constexpr int U = BnDepth<VEC, DT>::apply;
  for (int64_t r0 = (int64_t)blk * lanes + lr; r0 < n; r0 += U * stride) {
    RawVec<VEC, DT> rg[U], rg2[U], ry[U], rx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u * stride;
      rg[u].zero();
      rg2[u].zero();
      ry[u].zero();
      rx[u].zero();
      if (r < n) {
        rg[u].load(gy, gy_dtype, r * C + c0);
        if (gy2) rg2[u].load(gy2, gy_dtype, r * C + c0);
        if (relu) ry[u].load(y, y_dtype, r * C + c0);
        rx[u].load(x, x_dtype, r * C + c0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u * stride;
      if (r >= n) break;
      float g[VEC], g2[VEC], yy[VEC], xv[VEC];
      rg[u].get(g);
      rg2[u].get(g2);
      ry[u].get(yy);
      rx[u].get(xv);
#pragma unroll
      for (int q = 0; q < VEC; ++q) {
        if (gy2) g[q] += g2[q];
        if (relu && yy[q] <= 0.f) g[q] = 0.f;
        const float xh = (xv[q] - mu[q]) * rs[q];
        xv[q] = k1[q] * (g[q] - k2[q] - xh * k3[q]);
      }
      stv<VEC, DT>(gx, gx_dtype, r * C + c0, xv);
      if (gres) stv<VEC, DT>(gres, gx_dtype, r * C + c0, g);
    }
  }
}

// part != null: (ggamma, gbeta) reduced from the partials by every block
// (block 0 stores them to ggamma_out / gbeta_out), as in bn_apply_kernel.
template <int VEC, int DT>
__global__ void __launch_bounds__(kGlueThreads)
bn_backward_apply_kernel(const void* __restrict__ gy, const void* __restrict__ gy2, int gy_dtype,
                         const void* __restrict__ y, int y_dtype, const void* __restrict__ x, int x_dtype,
                         const int32_t* n_dev, int64_t cap, int C, const float* __restrict__ mean,
                         const float* __restrict__ rstd, const float* __restrict__ gamma, int relu,
                         const float* __restrict__ ggamma, const float* __restrict__ gbeta, void* __restrict__ gx,
                         int gx_dtype, void* __restrict__ gres, const float* __restrict__ part, int nb,
                         float* __restrict__ ggamma_out, float* __restrict__ gbeta_out, const int* __restrict__ nb_dev) {
  extern __shared__ float s_stat[];
  ::vp::pdl_begin();
  const int n = load_count(n_dev, cap);
  if (part) {
    if (nb_dev) {
      // producer partials (bn_epi.cuh): [0] = sum g, [1] = sum g*(x - mean);
      // ggamma = rstd * [1]
      nb = *nb_dev;
      bn_finalize(part, nb, C, n, false, 0.f, s_stat, s_stat + C);
      for (int c = threadIdx.x; c < C; c += kGlueThreads) s_stat[c] *= rstd[c];
      __syncthreads();
    } else {
      bn_finalize(part, nb, C, n, false, 0.f, s_stat, s_stat + C);
    }
    if (blockIdx.x == 0)
      for (int c = threadIdx.x; c < C; c += kGlueThreads) {
        ggamma_out[c] = s_stat[c];
        gbeta_out[c] = s_stat[C + c];
      }
    ggamma = s_stat;
    gbeta = s_stat + C;
  }
  bn_backward_apply_rows<VEC, DT>(gy, gy2, gy_dtype, y, y_dtype, x, x_dtype, n, C, mean, rstd, gamma,
                              relu, ggamma, gbeta, gx, gx_dtype, gres, blockIdx.x, gridDim.x);
}

// number of partial blocks: ~16 row passes of 8 elements per thread, at most
// one block per SM -> the partial phase is short and the last block reduces
// few partials per channel (the element count, not the capacity, would be
// ideal, but it lives on the device; the capacity bounds it)
static int bn_passes() {  // row passes per thread in the partial phase (VP_BN_PASSES overrides, for tuning)
  static const int v = getenv("VP_BN_PASSES") ? std::max(1, atoi(getenv("VP_BN_PASSES"))) : 24;
  return v;
}
static int bn_bwd_passes() {  // the backward partials read 3-4 tensors: own pass count (VP_BN_BWD_PASSES)
  static const int v = getenv("VP_BN_BWD_PASSES") ? std::max(1, atoi(getenv("VP_BN_BWD_PASSES"))) : bn_passes();
  return v;
}
static int bn_partial_blocks(int64_t cap, int64_t C, bool bwd = false) {
  const int64_t elems = std::max<int64_t>(cap, 1) * C;
  const int passes = bwd ? bn_bwd_passes() : bn_passes();
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(elems, (int64_t)kGlueThreads * 8 * passes), kNumSMs));
}
// partial rows reserved in the (shared forward/backward) workspace
static int bn_partial_slots(int64_t cap, int64_t C) {
  return std::max(bn_partial_blocks(cap, C, false), bn_partial_blocks(cap, C, true));
}

static bool bn_shape_ok(int64_t C) { return (C % 8 == 0 && C / 8 <= kGlueThreads) || C <= kGlueThreads; }

static int bn_apply_per_sm() {  // apply blocks per SM (VP_BN_APPLY_PER_SM overrides, for tuning)
  static const int v = getenv("VP_BN_APPLY_PER_SM") ? std::max(1, atoi(getenv("VP_BN_APPLY_PER_SM"))) : 1;
  return v;
}
static int bn_grid_rows(int64_t cap, int64_t C) {
  const int vec = (C % 8 == 0) ? 8 : 1;
  const int lanes = std::max<int>(1, kGlueThreads / (int)(C / vec));
  return (int)std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(std::max<int64_t>(cap, 1), lanes), (int64_t)kNumSMs * bn_apply_per_sm()));
}

// ------------------------------------------------------------------ pooling
__global__ void batch_count_kernel(const int4* __restrict__ coords, const int32_t* n_dev, int64_t cap, int B,
                                   int32_t* counts) {
  ::vp::pdl_begin();
  const int n = load_count(n_dev, cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int b = coords[i].x;
    if (b >= 0 && b < B) atomicAdd(&counts[b], 1);
  }
}
__global__ void batch_starts_kernel(const int32_t* counts, int B, int32_t* starts) {
  ::vp::pdl_begin();
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
template <int DT>  // x dtype at compile time (-1: runtime) so the row loads batch
__global__ void pool_kernel(const void* __restrict__ x, int dtype, int C, int B, const int32_t* counts,
                            const int32_t* starts, float* out) {
  ::vp::pdl_begin();
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    const int s = starts[b], cnt = counts[b];
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
      float acc = 0.f;
#pragma unroll 8
      for (int r = 0; r < cnt; ++r) {
        const int64_t i = (int64_t)(s + r) * C + c;
        acc += DT == VP_BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(x)[i])
               : DT == VP_F32 ? reinterpret_cast<const float*>(x)[i]
                              : ldf(x, dtype, i);
      }
      out[(int64_t)b * C + c] = cnt > 0 ? acc / (float)cnt : 0.f;
    }
  }
}
__global__ void pool_backward_kernel(const float* __restrict__ gout, const int4* __restrict__ coords,
                                     const int32_t* __restrict__ counts, const int32_t* n_dev, int64_t cap, int C,
                                     void* gx, int gx_dtype) {
  ::vp::pdl_begin();
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
  ::vp::pdl_begin();
  extern __shared__ float sm[];
  float* s_logit = sm;            // classes
  float* s_g = sm + classes;      // classes: this sample's g_logits
  float* s_x = sm + 2 * classes;  // C: this sample's pooled row
  __shared__ float s_max, s_sum;
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int c = threadIdx.x; c < C; c += blockDim.x) s_x[c] = pooled[(int64_t)b * C + c];
  __syncthreads();
  // logits: a warp per class, lanes stride the channels (coalesced W row),
  // fixed xor tree -> deterministic
  for (int j = warp; j < classes; j += nw) {
    float acc = 0.f;
#pragma unroll 4
    for (int c = lane; c < C; c += 32) acc += w[(int64_t)j * C + c] * s_x[c];
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if (lane == 0) {
      const float v = acc + bias[j];
      s_logit[j] = v;
      logits[(int64_t)b * classes + j] = v;
    }
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
    const float p = expf(s_logit[j] - s_max) / s_sum;
    const float gj = (p - (j == lab ? 1.f : 0.f)) / (float)B;
    s_g[j] = gj;
    g_logits[(int64_t)b * classes + j] = gj;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float acc = 0.f;
#pragma unroll 8
    for (int j = 0; j < classes; ++j) acc += s_g[j] * w[(int64_t)j * C + c];
    g_pooled[(int64_t)b * C + c] = acc;
  }
}
// kernel 2: fc grads and the mean loss, summed over samples in order.
__global__ void xent_reduce_kernel(const float* __restrict__ pooled, int B, int C, int classes,
                                   const float* __restrict__ g_logits, const float* __restrict__ loss_b,
                                   float* g_w, float* g_b, float* loss) {
  ::vp::pdl_begin();
  const int64_t total = (int64_t)classes * (C + 1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / (C + 1));
    const int c = (int)(e - (int64_t)j * (C + 1));
    float acc = 0.f;
    if (c < C) {
#pragma unroll 8
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

// ------------------------------------------------------------------ fused head
// The classifier head of the training step in two launches: head_kernel runs
// one block per cloud (rows [starts[b], starts[b] + counts[b]), batch-
// contiguous): mean pool -> logits (warp per class, fixed xor tree) ->
// softmax / loss -> g_logits = (p - onehot) / B -> g_pooled = g_logits W ->
// the gradient of every row of the cloud, g = g_pooled / count, masked by
// the last BN's ReLU (act > 0) and stored rounded (gm) with that BN's
// backward statistics per cloud (sum gm, sum gm (pre - mean): bn_epi.cuh
// partial row b); head_reduce_kernel (one block) sums the fc gradients and
// the loss over clouds in order and finalizes the BN statistics.  The
// arithmetic of pool + xent + pool_backward + the unfused BN statistics
// pass; the pool, pooled-gradient and statistics sums run in G thread
// groups whose partials are added in group order (deterministic).
constexpr int kHeadThreads = 1024;

struct HeadBn {
  const void* act;    // last BN output (ReLU mask source), nullable
  const void* pre;    // last BN input (conv output), nullable = no statistics
  const float* mean;
  void* gm;           // [n, C] row gradients (masked)
  float* part;        // bn_epi partial rows (B of them)
  int* nb;
};

// G = blockDim / C thread groups per channel (4 at C = 256 with 1024
// threads) split the rows of the pool, the classes of the pooled gradient and
// the rows of the backward pass; the groups' partials are summed in group
// order (deterministic)
template <int DT>
__global__ void __launch_bounds__(kHeadThreads)
head_kernel(const void* __restrict__ a, int dtype, const int32_t* __restrict__ seg, int B, int C,
            const float* __restrict__ w, const float* __restrict__ bias, int classes, const int32_t* __restrict__ labels,
            float* __restrict__ pooled, float* __restrict__ logits, float* __restrict__ g_logits,
            float* __restrict__ loss_b, float* __restrict__ g_pooled, const HeadBn hb) {
  ::vp::pdl_begin();
  extern __shared__ float sm[];
  const bool grouped = C <= (int)blockDim.x;
  const int G = grouped ? (int)blockDim.x / C : 1;
  float* s_x = sm;                 // C: pooled row
  float* s_gp = sm + C;            // C: g_pooled row
  float* s_logit = sm + 2 * C;     // classes
  float* s_g = s_logit + classes;  // classes
  float* s_r1 = s_g + classes;     // [G][C] group partials
  float* s_r2 = s_r1 + G * C;      // [G][C]
  __shared__ float s_max, s_sum;
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int grp = grouped ? (int)threadIdx.x / C : 0;
  const int cstart = grouped ? (int)threadIdx.x % C : (int)threadIdx.x, cstride = grouped ? C : (int)blockDim.x;
  const bool in_grp = grp < G;
  const int cnt = seg[b], st = seg[B + b];
  if (b == 0 && threadIdx.x == 0 && hb.nb) *hb.nb = B;
  auto ld = [&](const void* p, int64_t i) -> float {
    return DT == VP_BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i])
           : DT == VP_F32 ? reinterpret_cast<const float*>(p)[i] : ldf(p, dtype, i);
  };
  constexpr int U = 8;  // rows per batch: every load of a batch issued before any use
  if (in_grp)
    for (int c = cstart; c < C; c += cstride) {
      float acc = 0.f;
      for (int r0 = grp; r0 < cnt; r0 += U * G) {
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int r = r0 + u * G;
          v[u] = r < cnt ? ld(a, (int64_t)(st + r) * C + c) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
      }
      s_r1[grp * C + c] = acc;
    }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float acc = 0.f;
    for (int q = 0; q < G; ++q) acc += s_r1[q * C + c];
    const float v = cnt > 0 ? acc / (float)cnt : 0.f;
    s_x[c] = v;
    pooled[(int64_t)b * C + c] = v;
  }
  __syncthreads();
  for (int j = warp; j < classes; j += nw) {
    float acc = 0.f;
#pragma unroll 4
    for (int c = lane; c < C; c += 32) acc += w[(int64_t)j * C + c] * s_x[c];
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if (lane == 0) {
      const float v = acc + bias[j];
      s_logit[j] = v;
      logits[(int64_t)b * classes + j] = v;
    }
  }
  __syncthreads();
  const int lab = labels[b];
  if (threadIdx.x == 0) {
    float m = -INFINITY;
    for (int j = 0; j < classes; ++j) m = fmaxf(m, s_logit[j]);
    float sum = 0.f;
    for (int j = 0; j < classes; ++j) sum += expf(s_logit[j] - m);
    s_max = m;
    s_sum = sum;
    loss_b[b] = -(s_logit[lab] - m - logf(sum));
  }
  __syncthreads();
  for (int j = threadIdx.x; j < classes; j += blockDim.x) {
    const float pj = expf(s_logit[j] - s_max) / s_sum;
    const float gj = (pj - (j == lab ? 1.f : 0.f)) / (float)B;
    s_g[j] = gj;
    g_logits[(int64_t)b * classes + j] = gj;
  }
  __syncthreads();
  if (in_grp)
    for (int c = cstart; c < C; c += cstride) {
      float acc = 0.f;
#pragma unroll 8
      for (int j = grp; j < classes; j += G) acc += s_g[j] * w[(int64_t)j * C + c];
      s_r1[grp * C + c] = acc;
    }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float acc = 0.f;
    for (int q = 0; q < G; ++q) acc += s_r1[q * C + c];
    s_gp[c] = acc;
    g_pooled[(int64_t)b * C + c] = acc;
  }
  __syncthreads();
  // the rows' gradient (pool backward) + the last BN's masked gradient and
  // statistics for this cloud
  if (in_grp)
    for (int c = cstart; c < C; c += cstride) {
      const float g0 = cnt > 0 ? s_gp[c] / (float)cnt : 0.f;
      const float gr = DT == VP_BF16 ? __bfloat162float(__float2bfloat16_rn(g0)) : g0;
      const float mu = hb.pre ? hb.mean[c] : 0.f;
      float s1 = 0.f, s2 = 0.f;
      for (int r0 = grp; r0 < cnt; r0 += U * G) {
        float av[U], pv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int r = r0 + u * G;
          const int64_t i = (int64_t)(st + r) * C + c;
          const bool in = r < cnt;
          av[u] = (in && hb.act) ? ld(hb.act, i) : 1.f;
          pv[u] = (in && hb.pre) ? ld(hb.pre, i) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int r = r0 + u * G;
          if (r >= cnt) break;
          const int64_t i = (int64_t)(st + r) * C + c;
          const float g = av[u] > 0.f ? gr : 0.f;
          stf(hb.gm, DT >= 0 ? DT : dtype, i, g);
          if (hb.pre) {
            s1 += g;
            s2 += g * (pv[u] - mu);
          }
        }
      }
      s_r1[grp * C + c] = s1;
      s_r2[grp * C + c] = s2;
    }
  if (!hb.pre) return;
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float s1 = 0.f, s2 = 0.f;
    for (int q = 0; q < G; ++q) {
      s1 += s_r1[q * C + c];
      s2 += s_r2[q * C + c];
    }
    hb.part[((int64_t)b * 2) * C + c] = s1;
    hb.part[((int64_t)b * 2 + 1) * C + c] = s2;
  }
}

// one 1024-thread block: fc gradients and the mean loss summed over clouds in
// order (as xent_reduce_kernel), then the last BN's finalize from the B
// per-cloud rows
// blocks [0, classes): row j of g_w (thread per channel, pooled rows read
// coalesced, the class's g_logits column staged in shared memory) summed over
// b in order; block `classes`: g_b and the mean loss; blocks after: the BN
// finalize of 32 channels each
__global__ void __launch_bounds__(256)
head_reduce_kernel(const float* __restrict__ pooled, int B, int C, int classes, const float* __restrict__ g_logits,
                   const float* __restrict__ loss_b, float* __restrict__ g_w, float* __restrict__ g_b,
                   float* __restrict__ loss, const BnEpi e) {
  ::vp::pdl_begin();
  __shared__ float s_g[1024];
  const int j = blockIdx.x;
  if (j < classes) {
    for (int b0 = 0; b0 < B; b0 += 1024) {
      const int nb = min(1024, B - b0);
      __syncthreads();
      for (int bb = threadIdx.x; bb < nb; bb += blockDim.x) s_g[bb] = g_logits[(int64_t)(b0 + bb) * classes + j];
      __syncthreads();
      for (int c = threadIdx.x; c < C; c += blockDim.x) {
        float acc = b0 == 0 ? 0.f : g_w[(int64_t)j * C + c];
#pragma unroll 16
        for (int bb = 0; bb < nb; ++bb) acc += s_g[bb] * pooled[(int64_t)(b0 + bb) * C + c];
        g_w[(int64_t)j * C + c] = acc;
      }
    }
    return;
  }
  if (j == classes) {
    for (int jj = threadIdx.x; jj < classes; jj += blockDim.x) {
      float acc = 0.f;
      for (int bb = 0; bb < B; ++bb) acc += g_logits[(int64_t)bb * classes + jj];
      g_b[jj] = acc;
    }
    if (threadIdx.x == 0) {
      float sum = 0.f;
      for (int bb = 0; bb < B; ++bb) sum += loss_b[bb];
      *loss = sum / (float)B;
    }
    return;
  }
}

__global__ void sgd_kernel(float* __restrict__ p, float* __restrict__ m, const float* __restrict__ g, int64_t n,
                           float lr, float mom, __nv_bfloat16* __restrict__ pb, int64_t nb) {
  ::vp::pdl_begin();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float mi = mom * m[i] + g[i];
    float pi = p[i] - lr * mi;
    m[i] = mi;
    p[i] = pi;
    if (pb && i < nb) pb[i] = __float2bfloat16_rn(pi);
  }
}

static int grid_for(int64_t total) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), grid_cap(16))); }

}  // namespace vp

using namespace vp;

extern "C" {

size_t vp_bn_stats_ws_bytes(int64_t cap_n, int64_t C) {
  return align_up((size_t)bn_partial_slots(cap_n, C) * 2 * C * 4, 256) + 256;  // partials + ticket
}

// Launch KERNEL<VEC, DT>: DT fixed at compile time when every tensor the kernel
// touches has one dtype (f32 or bf16), else the runtime-dtype variant.
#define VP_BN_LAUNCH(KERNEL, C, DT, ...)                                               \
  ((C) % 8 != 0          ? ::vp::launch(KERNEL<1, -1>, __VA_ARGS__)                    \
   : (DT) == VP_BF16 ? ::vp::launch(KERNEL<8, VP_BF16>, __VA_ARGS__)                   \
   : (DT) == VP_F32  ? ::vp::launch(KERNEL<8, VP_F32>, __VA_ARGS__)                    \
                     : ::vp::launch(KERNEL<8, -1>, __VA_ARGS__))

static int one_dtype(std::initializer_list<int> ds) {
  const int d = *ds.begin();
  for (int v : ds)
    if (v != d) return -1;
  return (d == VP_F32 || d == VP_BF16) ? d : -1;
}

static int* bn_ticket(void* ws, int64_t cap, int64_t C) {
  return reinterpret_cast<int*>((char*)ws + align_up((size_t)bn_partial_slots(cap, C) * 2 * C * 4, 256));
}

int vp_bn_stats(const void* x, int32_t xd, const int32_t* n_dev, int64_t cap, int64_t C, float eps, float* mean,
                float* rstd, void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(bn_shape_ok(C), VP_EVALIDATION, "bn: channels must be <= 256 or a multiple of 8 <= 2048");
  VP_REQUIRE(ws_bytes >= vp_bn_stats_ws_bytes(cap, C), VP_EVALIDATION, "bn_stats: workspace too small");
  const int nb = bn_partial_blocks(cap, C);
  int* ticket = bn_ticket(ws, cap, C);
  const BnFuse F{};
  VP_BN_LAUNCH(bn_partial_kernel, C, one_dtype({xd}), nb, kGlueThreads, 0, st, x, xd, n_dev, cap, (int)C, nullptr,
               nullptr, 0, nullptr, 0, 0, nullptr, nullptr, (float*)ws, ticket, eps, mean, rstd, F);
  VP_CHECK_LAUNCH("bn_stats");
  return VP_OK;
}

// Off by default: measured in the C3 step the cooperative launch waits for the
// whole grid to become co-resident behind the side-stream weight-gradient
// kernels and loses the programmatic-dependent-launch overlap, 1.93 ms vs
// 1.76 ms per step with the two-launch path.  VP_BN_FUSED=1 enables it.
static bool bn_fused_enabled() {
  static const bool v = getenv("VP_BN_FUSED") && atoi(getenv("VP_BN_FUSED")) == 1;
  return v;
}

int vp_bn_forward(const void* x, int32_t xd, const int32_t* n_dev, int64_t cap, int64_t C, float eps, float* mean,
                  float* rstd, const float* gamma, const float* beta, const void* res, int32_t rd, int32_t relu,
                  void* y, int32_t yd, void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(bn_shape_ok(C), VP_EVALIDATION, "bn: channels must be <= 256 or a multiple of 8 <= 2048");
  VP_REQUIRE(ws_bytes >= vp_bn_stats_ws_bytes(cap, C), VP_EVALIDATION, "bn_forward: workspace too small");
  if (bn_fused_enabled() && cap > 0) {
    const int nb = bn_partial_blocks(cap, C);
    int* ticket = bn_ticket(ws, cap, C);
    const BnFuse F{1, ticket + 16, gamma, beta, res, rd, relu, y, yd, nullptr};
    cudaError_t e = C % 8 == 0
        ? ::vp::launch_coop(bn_partial_kernel<8, -1>, nb, kGlueThreads, 0, st, x, xd, n_dev, cap, (int)C, nullptr, nullptr,
                            0, nullptr, 0, 0, nullptr, nullptr, (float*)ws, ticket, eps, mean, rstd, F)
        : ::vp::launch_coop(bn_partial_kernel<1, -1>, nb, kGlueThreads, 0, st, x, xd, n_dev, cap, (int)C, nullptr, nullptr,
                            0, nullptr, 0, 0, nullptr, nullptr, (float*)ws, ticket, eps, mean, rstd, F);
    VP_REQUIRE(e == cudaSuccess, VP_EINTERNAL, "bn_forward: cooperative launch failed");
    VP_CHECK_LAUNCH("bn_forward");
    return VP_OK;
  }
  if (cap <= 0) return vp_bn_stats(x, xd, n_dev, cap, C, eps, mean, rstd, ws, ws_bytes, stream);
  // partials only (no ticket), then the apply kernel reduces them in every block
  const int nb = bn_partial_blocks(cap, C);
  const BnFuse F{};
  VP_BN_LAUNCH(bn_partial_kernel, C, one_dtype({xd}), nb, kGlueThreads, 0, st, x, xd, n_dev, cap, (int)C, nullptr,
               nullptr, 0, nullptr, 0, 0, nullptr, nullptr, (float*)ws, (int*)nullptr, eps, mean, rstd, F);
  VP_CHECK_LAUNCH("bn_fwd_stats");
  VP_BN_LAUNCH(bn_apply_kernel, C, one_dtype({xd, yd, res ? rd : xd}), bn_grid_rows(cap, C), kGlueThreads,
               2 * C * sizeof(float), st, x, xd, n_dev, cap, (int)C, (const float*)nullptr, (const float*)nullptr,
               gamma, beta, res, rd, relu, y, yd, (const float*)ws, nb, eps, mean, rstd, (const int*)nullptr);
  VP_CHECK_LAUNCH("bn_fwd_apply");
  return VP_OK;
}

int vp_bn_apply(const void* x, int32_t xd, const int32_t* n_dev, int64_t cap, int64_t C, const float* mean,
                const float* rstd, const float* gamma, const float* beta, const void* res, int32_t rd, int32_t relu,
                void* y, int32_t yd, vp_stream_t stream) {
  VP_REQUIRE(bn_shape_ok(C), VP_EVALIDATION, "bn: channels must be <= 256 or a multiple of 8 <= 2048");
  if (cap <= 0) return VP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = bn_grid_rows(cap, C);
  VP_BN_LAUNCH(bn_apply_kernel, C, one_dtype({xd, yd, res ? rd : xd}), grid, kGlueThreads, 0, st, x, xd, n_dev, cap,
               (int)C, mean, rstd, gamma, beta, res, rd, relu, y, yd, (const float*)nullptr, 0, 0.f, (float*)nullptr,
               (float*)nullptr, (const int*)nullptr);
  VP_CHECK_LAUNCH("bn_apply");
  return VP_OK;
}

size_t vp_bn_backward_ws_bytes(int64_t cap_n, int64_t C) { return vp_bn_stats_ws_bytes(cap_n, C); }

int vp_bn_backward(const void* gy, const void* gy2, int32_t gyd, const void* y, int32_t yd, const void* x, int32_t xd,
                   const int32_t* n_dev, int64_t cap, int64_t C, const float* mean, const float* rstd,
                   const float* gamma, int32_t relu, void* gx, int32_t gxd, void* gres, float* ggamma, float* gbeta,
                   void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(bn_shape_ok(C), VP_EVALIDATION, "bn: channels must be <= 256 or a multiple of 8 <= 2048");
  VP_REQUIRE(ws_bytes >= vp_bn_backward_ws_bytes(cap, C), VP_EVALIDATION, "bn_backward: workspace too small");
  const int nb = bn_partial_blocks(cap, C, true);
  int* ticket = bn_ticket(ws, cap, C);
  if (bn_fused_enabled() && cap > 0) {
    const BnFuse F{2, ticket + 16, gamma, nullptr, nullptr, 0, relu, gx, gxd, gres};
    cudaError_t e = C % 8 == 0
        ? ::vp::launch_coop(bn_partial_kernel<8, -1>, nb, kGlueThreads, 0, st, x, xd, n_dev, cap, (int)C, gy, gy2, gyd, y,
                            yd, relu, mean, rstd, (float*)ws, ticket, 0.f, ggamma, gbeta, F)
        : ::vp::launch_coop(bn_partial_kernel<1, -1>, nb, kGlueThreads, 0, st, x, xd, n_dev, cap, (int)C, gy, gy2, gyd, y,
                            yd, relu, mean, rstd, (float*)ws, ticket, 0.f, ggamma, gbeta, F);
    VP_REQUIRE(e == cudaSuccess, VP_EINTERNAL, "bn_backward: cooperative launch failed");
    VP_CHECK_LAUNCH("bn_bwd_fused");
    return VP_OK;
  }
  const BnFuse F{};
  const int dt_stats = one_dtype({xd, gyd, relu ? yd : xd});
  // cap > 0: partials only, reduced by every block of the apply kernel
  VP_BN_LAUNCH(bn_partial_kernel, C, dt_stats, nb, kGlueThreads, 0, st, x, xd, n_dev, cap, (int)C, gy, gy2, gyd, y, yd,
               relu, mean, rstd, (float*)ws, cap > 0 ? (int*)nullptr : ticket, 0.f, ggamma, gbeta, F);
  VP_CHECK_LAUNCH("bn_bwd_stats");
  if (cap > 0) {
    const int grid = bn_grid_rows(cap, C);
    VP_BN_LAUNCH(bn_backward_apply_kernel, C, one_dtype({xd, gyd, relu ? yd : xd, gxd}), grid, kGlueThreads,
                 2 * C * sizeof(float), st, gy, gy2, gyd, y, yd, x, xd, n_dev, cap, (int)C, mean, rstd, gamma, relu,
                 (const float*)nullptr, (const float*)nullptr, gx, gxd, gres, (const float*)ws, nb, ggamma, gbeta,
                 (const int*)nullptr);
    VP_CHECK_LAUNCH("bn_bwd_apply");
  }
  return VP_OK;
}

static int bn_early() {  // early programmatic launch of the apply behind the finalize (VP_BN_EARLY)
  static const int v = getenv("VP_BN_EARLY") ? atoi(getenv("VP_BN_EARLY")) : 1;
  return v;
}

// The apply halves of the forward / backward BN whose statistics partials a
// producer wrote (vp_conv_fwd_bn / vp_conv_dgrad_bn, bn_epi.cuh): one launch
// each on the critical path instead of a statistics pass plus an apply.
int vp_bn_apply_part(const void* x, int32_t xd, const int32_t* n_dev, int64_t cap, int64_t C, float eps,
                     const void* bn_part, float* mean, float* rstd, const float* gamma, const float* beta,
                     const void* res, int32_t rd, int32_t relu, void* y, int32_t yd, vp_stream_t stream) {
  VP_REQUIRE(bn_shape_ok(C), VP_EVALIDATION, "bn: channels must be <= 256 or a multiple of 8 <= 2048");
  VP_REQUIRE(bn_part, VP_EVALIDATION, "bn_apply_part: partials required");
  cudaStream_t st = (cudaStream_t)stream;
  BnEpi e{};
  e.mode = 1;
  e.nb = (int*)bn_part;
  e.part = (float*)((char*)bn_part + kBnPartHeader);
  e.out_a = mean;
  e.out_b = rstd;
  e.eps = eps;
  e.early = bn_early();
  ::vp::launch(bn_finalize_kernel, (int)ceil_div(C, 32), 1024, 0, st, e, (int)C, n_dev, cap);
  VP_CHECK_LAUNCH("bn_finalize");
  if (cap <= 0) return VP_OK;
  VP_BN_LAUNCH(bn_apply_kernel, C, one_dtype({xd, yd, res ? rd : xd}), bn_grid_rows(cap, C), kGlueThreads, 0, st, x,
               xd, n_dev, cap, (int)C, (const float*)mean, (const float*)rstd, gamma, beta, res, rd, relu, y, yd,
               (const float*)nullptr, 0, 0.f, (float*)nullptr, (float*)nullptr, (const int*)nullptr);
  VP_CHECK_LAUNCH("bn_apply_part");
  return VP_OK;
}

int vp_bn_backward_part(const void* gm, int32_t gmd, const void* x, int32_t xd, const int32_t* n_dev, int64_t cap,
                        int64_t C, const float* mean, const float* rstd, const float* gamma, const void* bn_part,
                        void* gx, int32_t gxd, float* ggamma, float* gbeta, vp_stream_t stream) {
  VP_REQUIRE(bn_shape_ok(C), VP_EVALIDATION, "bn: channels must be <= 256 or a multiple of 8 <= 2048");
  VP_REQUIRE(bn_part, VP_EVALIDATION, "bn_backward_part: partials required");
  cudaStream_t st = (cudaStream_t)stream;
  BnEpi e{};
  e.mode = 2;
  e.nb = (int*)bn_part;
  e.part = (float*)((char*)bn_part + kBnPartHeader);
  e.out_a = ggamma;
  e.out_b = gbeta;
  e.rstd = rstd;
  e.early = bn_early();
  ::vp::launch(bn_finalize_kernel, (int)ceil_div(C, 32), 1024, 0, st, e, (int)C, n_dev, cap);
  VP_CHECK_LAUNCH("bn_finalize");
  return vp_bn_backward_apply(gm, gmd, x, xd, n_dev, cap, C, mean, rstd, gamma, ggamma, gbeta, gx, gxd, stream);
}

// the apply half of the BN backward from finished (ggamma, gbeta): gm is the
// masked gradient the producer stored (vp_conv_dgrad_bn with finalize)
int vp_bn_backward_apply(const void* gm, int32_t gmd, const void* x, int32_t xd, const int32_t* n_dev, int64_t cap,
                         int64_t C, const float* mean, const float* rstd, const float* gamma, const float* ggamma,
                         const float* gbeta, void* gx, int32_t gxd, vp_stream_t stream) {
  VP_REQUIRE(bn_shape_ok(C), VP_EVALIDATION, "bn: channels must be <= 256 or a multiple of 8 <= 2048");
  cudaStream_t st = (cudaStream_t)stream;
  if (cap <= 0) return VP_OK;
  VP_BN_LAUNCH(bn_backward_apply_kernel, C, one_dtype({xd, gmd, gxd}), bn_grid_rows(cap, C), kGlueThreads, 0, st, gm,
               (const void*)nullptr, gmd, (const void*)nullptr, gmd, x, xd, n_dev, cap, (int)C, mean, rstd, gamma, 0,
               (const float*)ggamma, (const float*)gbeta, gx, gxd, (void*)nullptr, (const float*)nullptr, 0,
               (float*)nullptr, (float*)nullptr, (const int*)nullptr);
  VP_CHECK_LAUNCH("bn_backward_part");
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
    ::vp::launch(batch_count_kernel, grid_for(cap), 256, 0, st, (const int4*)coords, n_dev, cap, B, counts);
    VP_CHECK_LAUNCH("batch_count");
  }
  ::vp::launch(batch_starts_kernel, 1, 1024, 0, st, counts, B, starts);
  VP_CHECK_LAUNCH("batch_starts");
  auto pk = xd == VP_BF16 ? pool_kernel<VP_BF16> : xd == VP_F32 ? pool_kernel<VP_F32> : pool_kernel<-1>;
  ::vp::launch(pk, std::min(B, kNumSMs * 4), C < 256 ? (int)C : 256, 0, st, x, xd, (int)C, B, counts, starts, out);
  VP_CHECK_LAUNCH("pool");
  return VP_OK;
}

int vp_global_pool_backward(const float* gout, const int32_t* coords, const int32_t* counts, const int32_t* n_dev,
                            int64_t cap, int64_t C, void* gx, int32_t gxd, vp_stream_t stream) {
  if (cap <= 0) return VP_OK;
  ::vp::launch(pool_backward_kernel, grid_for(cap * C), 256, 0, (cudaStream_t)stream, gout, (const int4*)coords, counts, n_dev,
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
  ::vp::launch(xent_sample_kernel, B, 256, (2 * classes + C) * sizeof(float), st, pooled, B, C, w, b, classes, labels, logits, g_logits,
                                                             loss_b, g_pooled);
  VP_CHECK_LAUNCH("xent_sample");
  ::vp::launch(xent_reduce_kernel, grid_for((int64_t)classes * (C + 1)), 256, 0, st, pooled, B, C, classes, g_logits, loss_b,
                                                                          g_w, g_b, loss);
  VP_CHECK_LAUNCH("xent_reduce");
  return VP_OK;
}

int vp_batch_segments(const int32_t* coords, const int32_t* n_dev, int64_t cap, int32_t B, int32_t* seg,
                      vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(B >= 1, VP_EVALIDATION, "batch_segments: B must be positive");
  cudaMemsetAsync(seg, 0, sizeof(int32_t) * B, st);
  VP_CHECK_ASYNC("batch_segments(memset)");
  if (cap > 0) {
    ::vp::launch(batch_count_kernel, grid_for(cap), 256, 0, st, (const int4*)coords, n_dev, cap, B, seg);
    VP_CHECK_LAUNCH("batch_count");
  }
  ::vp::launch(batch_starts_kernel, 1, 1024, 0, st, (const int32_t*)seg, B, seg + B);
  VP_CHECK_LAUNCH("batch_starts");
  return VP_OK;
}

size_t vp_sparse_head_ws_bytes(int32_t B, int64_t C, int32_t classes) {
  return align_up((size_t)B * classes * 4, 256) + align_up((size_t)B * 4, 256) + align_up((size_t)B * C * 4, 256);
}

int vp_sparse_head(const void* a, int32_t a_dtype, const int32_t* seg, int32_t B, int64_t C, const float* w,
                   const float* bias, int32_t classes, const int32_t* labels, float* pooled, float* logits, float* loss,
                   float* g_w, float* g_b, const void* bn_act, const void* bn_pre, const float* bn_mean,
                   const float* bn_rstd, void* gm, void* bn_part, float* ggamma, float* gbeta, void* ws,
                   size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(B >= 1 && C >= 1 && classes >= 1 && classes <= 4096, VP_EVALIDATION, "sparse_head: bad shape");
  VP_REQUIRE(ws && ws_bytes >= vp_sparse_head_ws_bytes(B, C, classes), VP_EVALIDATION, "sparse_head: workspace too small");
  VP_REQUIRE(!bn_pre || (bn_mean && bn_rstd && bn_part && ggamma && gbeta && B <= kBnPartRows), VP_EVALIDATION,
             "sparse_head: the BN statistics need mean, rstd, partial rows and outputs");
  VP_REQUIRE(gm, VP_EVALIDATION, "sparse_head: row gradient output required");
  char* p = (char*)ws;
  float* g_logits = (float*)p;
  p += align_up((size_t)B * classes * 4, 256);
  float* loss_b = (float*)p;
  p += align_up((size_t)B * 4, 256);
  float* g_pooled = (float*)p;
  HeadBn hb{bn_act, bn_pre, bn_mean, gm, bn_part ? (float*)((char*)bn_part + kBnPartHeader) : nullptr, (int*)bn_part};
  const int64_t groups = C <= kHeadThreads ? kHeadThreads / C : 1;
  const size_t smem = (size_t)(2 * C + 2 * classes + 2 * groups * C) * sizeof(float);
  auto hk = a_dtype == VP_BF16 ? head_kernel<VP_BF16> : a_dtype == VP_F32 ? head_kernel<VP_F32> : head_kernel<-1>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  ::vp::launch(hk, B, kHeadThreads, smem, st, a, a_dtype, seg, B, (int)C, w, bias, classes, labels, pooled, logits,
               g_logits, loss_b, g_pooled, hb);
  VP_CHECK_LAUNCH("sparse_head");
  BnEpi e{};
  e.mode = 2;
  e.part = hb.part;
  e.out_a = bn_pre ? ggamma : nullptr;
  e.out_b = gbeta;
  e.rstd = bn_rstd;
  // the finalize blocks need 1024 threads: a separate tiny launch keeps the fc blocks at 256
  ::vp::launch(head_reduce_kernel, classes + 1, 256, 0, st, (const float*)pooled, B, (int)C, classes,
               (const float*)g_logits, (const float*)loss_b, g_w, g_b, loss, e);
  VP_CHECK_LAUNCH("sparse_head_reduce");
  if (bn_pre) {
    e.nb = (int*)bn_part;
    ::vp::launch(bn_finalize_kernel, (int)ceil_div(C, 32), 1024, 0, st, e, (int)C, (const int32_t*)nullptr, (int64_t)B);
    VP_CHECK_LAUNCH("bn_finalize");
  }
  return VP_OK;
}

int vp_sgd_momentum(float* p, float* m, const float* g, int64_t n, float lr, float momentum, void* pb, int64_t nb,
                    vp_stream_t stream) {
  if (n <= 0) return VP_OK;
  ::vp::launch(sgd_kernel, grid_for(n), 256, 0, (cudaStream_t)stream, p, m, g, n, lr, momentum, (__nv_bfloat16*)pb, nb);
  VP_CHECK_LAUNCH("sgd");
  return VP_OK;
}

}  // extern "C"
