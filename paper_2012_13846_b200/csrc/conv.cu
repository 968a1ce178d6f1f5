// Sparse convolution float stage (conv.py:186-242) on sm_100a.
//
// Forward / dgrad: output-stationary implicit GEMM.  A CTA owns a tile of
// 128 output rows; for every kernel offset that has at least one neighbour in
// the tile (offsets in shape order, per-row accumulation order fixed =
// deterministic) and every 64-wide slice of C_in, the neighbour rows are
// gathered with cp.async (zero-fill for missing neighbours) into a
// 128B-swizzled K-major shared tile, the weight slice W_k[:, slice] is
// staged next to it, and one elected thread issues tcgen05.mma (M=128,
// N=C_out, K=16 per instruction) accumulating in TMEM.  A multi-stage
// mbarrier ring (tcgen05.commit -> stage free) overlaps gathers with MMAs.
// The epilogue reads TMEM with tcgen05.ld and writes each output row once
// (no atomics on the output path).
//
// wgrad: per offset, grad_W_k = sum over its pairs of g[u] x[v]^T.  Pairs are
// cut into fixed-size chunks; a persistent CTA walks chunks, gathers 64 pairs
// per stage into MN-major swizzled tiles (g rows -> A, x rows -> B) and
// accumulates D[C_out, C_in] in TMEM; each chunk's partial goes to a fp32
// workspace and a second kernel sums the chunks of each offset in a fixed
// order -> deterministic.
#include <algorithm>
#include <cooperative_groups.h>

#include "common.cuh"
#include "conv_fwd_tc.cuh"
#include "conv_tc_dispatch.cuh"
#include "conv_rows.cuh"
#include "conv_wgrad_tc.cuh"
#include "tc.cuh"

namespace vp {

long long* g_conv_trace_host = nullptr;  // vp_debug_conv_trace (experiments only)


// Pairwise (binary-counter) summation of n values p[0], p[stride], ... in a
// fixed order: after element i the stack holds the partial sums of blocks
// whose sizes are the binary digits of i+1, merged as soon as two equal
// blocks meet — a balanced tree, so the rounding error grows with log2(n)
// rather than n (the stride-1 centre offset of a C5 stem layer
// reduces ~1,600 chunk partials).  Deterministic: the order depends on n only.
template <typename T>
__device__ __forceinline__ T tree_sum(const T* __restrict__ p, int64_t stride, int n) {
  T stack[32];
  int top = 0;
  int i = 0;
  for (; i + 4 <= n; i += 4) {  // four loads in flight, merged in order
    T v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = p[(int64_t)(i + j) * stride];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      T s = v[j];
      for (unsigned c = (unsigned)(i + j) + 1u; (c & 1u) == 0u; c >>= 1) s = stack[--top] + s;
      stack[top++] = s;
    }
  }
  for (; i < n; ++i) {
    T s = p[(int64_t)i * stride];
    for (unsigned c = (unsigned)i + 1u; (c & 1u) == 0u; c >>= 1) s = stack[--top] + s;
    stack[top++] = s;
  }
  T acc = T(0);
  while (top > 0) acc = stack[--top] + acc;
  return acc;
}

// sum the chunk partials of each offset, pairwise in chunk order (deterministic)
// optional momentum SGD fused into the reduction (sgd_kernel's arithmetic,
// glue.cu): the finished gradient element updates its parameter at once
struct SgdFuse {
  float* p;
  float* m;
  __nv_bfloat16* pb;  // bf16 shadow of p (nullable)
  float lr, mom;
};

template <typename T>
__global__ void wgrad_reduce_kernel(const T* __restrict__ part, const int32_t* __restrict__ pptr,
                                    int K, int chunk, int64_t per, T* __restrict__ gw, const int* chunk_dev,
                                    const SgdFuse sgd) {
  ::vp::pdl_begin();
  __shared__ int s_pref[VP_MAX_OFFSETS + 1];
  __shared__ int s_ptr[VP_MAX_OFFSETS + 1];
  if (chunk_dev) chunk = *chunk_dev;  // chosen on the device by the partial kernel
  for (int k = threadIdx.x; k <= K; k += blockDim.x) s_ptr[k] = __ldg(pptr + k);  // all loads in flight
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int k = 0; k < K; ++k) {
      s_pref[k] = acc;
      acc += (s_ptr[k + 1] - s_ptr[k] + chunk - 1) / chunk;
    }
    s_pref[K] = acc;
  }
  __syncthreads();
  const int64_t total = (int64_t)K * per;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e / per);
    const int64_t o = e - (int64_t)k * per;
    const T g = tree_sum(part + (int64_t)s_pref[k] * per + o, per, s_pref[k + 1] - s_pref[k]);
    gw[e] = g;
    if (sgd.p) {  // m = mom * m + g ; p -= lr * m ; shadow
      const float mi = sgd.mom * sgd.m[e] + (float)g;
      const float pi = sgd.p[e] - sgd.lr * mi;
      sgd.m[e] = mi;
      sgd.p[e] = pi;
      if (sgd.pb) sgd.pb[e] = __float2bfloat16_rn(pi);
    }
  }
}

// ------------------------------------------------------------------ SIMT paths
// Generic widths, fp32 and f64 features.  T is the accumulation type: fp32
// for bf16/fp32 features, f64 when any operand is f64 (the reference's own
// precision, conv.py:77-105 — parity to ~1e-12 and a finite-difference
// gradient check are possible in that mode).
template <typename T>
__device__ __forceinline__ T ldv(const void* p, int dtype, int64_t i) {
  if (dtype == VP_F64) return (T)reinterpret_cast<const double*>(p)[i];
  if (dtype == VP_BF16) return (T)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  return (T)reinterpret_cast<const float*>(p)[i];
}
template <typename T>
__device__ __forceinline__ void stv(void* p, int dtype, int64_t i, T v) {
  if (dtype == VP_F64)
    reinterpret_cast<double*>(p)[i] = (double)v;
  else if (dtype == VP_BF16)
    reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn((float)v);
  else
    reinterpret_cast<float*>(p)[i] = (float)v;
}

// y[u, co] = sum_k sum_ci W[k, co, ci] x[t[u,k], ci].
// W is addressed as W[k*wk + co*wco + ci*wci] so dgrad passes W^T by strides.
template <typename T>
__global__ void conv_fwd_simt_kernel(const void* __restrict__ x, int x_dtype, int cin,
                                     const void* __restrict__ w, int w_dtype, int64_t wk, int64_t wco,
                                     int64_t wci, int cout, int K, const int32_t* __restrict__ table,
                                     int flip, const int32_t* __restrict__ perm, const int32_t* n_out_dev,
                                     int64_t cap_out, void* y, int y_dtype) {
  ::vp::pdl_begin();
  const int n_out = load_count(n_out_dev, cap_out);
  const int64_t total = (int64_t)n_out * cout;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = e / cout;
    const int co = (int)(e - u * cout);
    T acc = T(0);
    for (int k = 0; k < K; ++k) {
      const int v = table[u * K + (flip ? K - 1 - k : k)];
      if (v < 0) continue;
      for (int ci = 0; ci < cin; ++ci)
        acc += ldv<T>(w, w_dtype, k * wk + co * wco + ci * wci) * ldv<T>(x, x_dtype, (int64_t)v * cin + ci);
    }
    stv<T>(y, y_dtype, perm ? (int64_t)perm[u] * cout + co : e, acc);
  }
}

// wgrad partials: block per (chunk item); warps stride over the chunk's pairs,
// lanes over output elements; fixed-order cross-warp sum.
constexpr int kWgSimtThreads = 256;
template <typename T>
__global__ void __launch_bounds__(kWgSimtThreads)
wgrad_simt_kernel(const void* __restrict__ x, int x_dtype, int cin, const void* __restrict__ gy,
                  int g_dtype, int cout, int K, const int32_t* __restrict__ pin,
                  const int32_t* __restrict__ pout, const int32_t* __restrict__ pptr, int chunk,
                  T* __restrict__ part) {
  ::vp::pdl_begin();
  __shared__ int s_pref[VP_MAX_OFFSETS + 1];
  __shared__ T s_red[kWgSimtThreads / 32][32];
  __shared__ int s_ptr[VP_MAX_OFFSETS + 1];
  for (int k = threadIdx.x; k <= K; k += blockDim.x) s_ptr[k] = __ldg(pptr + k);  // all loads in flight
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int k = 0; k < K; ++k) {
      s_pref[k] = acc;
      acc += (s_ptr[k + 1] - s_ptr[k] + chunk - 1) / chunk;
    }
    s_pref[K] = acc;
  }
  __syncthreads();
  const int n_items = s_pref[K];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per = cin * cout;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    int k = 0;
    while (s_pref[k + 1] <= item) ++k;
    const int p0 = s_ptr[k] + (item - s_pref[k]) * chunk;
    const int p1 = min(s_ptr[k + 1], p0 + chunk);
    for (int e0 = 0; e0 < per; e0 += 32) {
      const int e = e0 + lane;
      const int co = e / cin, ci = e - (e / cin) * cin;
      T acc = T(0);
      if (e < per)
#pragma unroll 8
        for (int q = p0 + warp; q < p1; q += kWgSimtThreads / 32)
          acc += ldv<T>(gy, g_dtype, (int64_t)pout[q] * cout + co) * ldv<T>(x, x_dtype, (int64_t)pin[q] * cin + ci);
      s_red[warp][lane] = acc;
      __syncthreads();
      if (warp == 0 && e < per) {
        T s = T(0);
        for (int w2 = 0; w2 < kWgSimtThreads / 32; ++w2) s += s_red[w2][lane];
        part[(int64_t)item * per + e] = s;
      }
      __syncthreads();
    }
  }
}

// Stem weight gradient (cin = 1, bf16): gw[k][co] = sum_q g[pout[q]][co] * x[pin[q]].
// The generic SIMT kernel walks pairs per warp with one dependent load chain
// per channel; here every thread owns whole pairs (the COUT-wide g row in
// registers, kWgStemPairs pairs in flight), then a fixed-order shuffle tree
// and an ordered sum over the warps give each item's partial (deterministic).
constexpr int kWgStemThreads = 256, kWgStemPairs = 4, kWgStemChunk = kWgStemThreads * kWgStemPairs;
template <int COUT>
__global__ void __launch_bounds__(kWgStemThreads)
wgrad_stem_kernel(const bf16* __restrict__ x, const bf16* __restrict__ gy, int K, const int32_t* __restrict__ pin,
                  const int32_t* __restrict__ pout, const int32_t* __restrict__ pptr, float* __restrict__ part) {
  ::vp::pdl_begin();
  __shared__ int s_pref[VP_MAX_OFFSETS + 1];
  __shared__ float s_red[kWgStemThreads / 32][COUT];
  __shared__ int s_ptr[VP_MAX_OFFSETS + 1];
  for (int k = threadIdx.x; k <= K; k += blockDim.x) s_ptr[k] = __ldg(pptr + k);  // all loads in flight
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int k = 0; k < K; ++k) {
      s_pref[k] = acc;
      acc += (s_ptr[k + 1] - s_ptr[k] + kWgStemChunk - 1) / kWgStemChunk;
    }
    s_pref[K] = acc;
  }
  __syncthreads();
  const int n_items = s_pref[K];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    int k = 0;
    while (s_pref[k + 1] <= item) ++k;
    const int p0 = s_ptr[k] + (item - s_pref[k]) * kWgStemChunk;
    const int p1 = min(s_ptr[k + 1], p0 + kWgStemChunk);
    float acc[COUT];
#pragma unroll
    for (int c = 0; c < COUT; ++c) acc[c] = 0.f;
    uint4 row[kWgStemPairs][COUT / 8];
    float xv[kWgStemPairs];
#pragma unroll
    for (int j = 0; j < kWgStemPairs; ++j) {
      const int q = p0 + j * kWgStemThreads + threadIdx.x;
      xv[j] = 0.f;
#pragma unroll
      for (int t = 0; t < COUT / 8; ++t) row[j][t] = make_uint4(0u, 0u, 0u, 0u);
      if (q < p1) {
        const int64_t o = pout[q];
        xv[j] = __bfloat162float(x[pin[q]]);
        const uint4* src = reinterpret_cast<const uint4*>(gy + o * COUT);
#pragma unroll
        for (int t = 0; t < COUT / 8; ++t) row[j][t] = __ldg(src + t);
      }
    }
#pragma unroll
    for (int j = 0; j < kWgStemPairs; ++j)
#pragma unroll
      for (int t = 0; t < COUT / 8; ++t) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&row[j][t]);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float2 f = __bfloat1622float2(h[u]);
          acc[t * 8 + 2 * u] += f.x * xv[j];
          acc[t * 8 + 2 * u + 1] += f.y * xv[j];
        }
      }
#pragma unroll
    for (int c = 0; c < COUT; ++c) {
      float v = acc[c];
#pragma unroll
      for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
      if (lane == 0) s_red[warp][c] = v;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < COUT; c += kWgStemThreads) {
      float v = 0.f;
#pragma unroll
      for (int w2 = 0; w2 < kWgStemThreads / 32; ++w2) v += s_red[w2][c];
      part[(int64_t)item * COUT + c] = v;
    }
    __syncthreads();
  }
}

__global__ void transpose_w_kernel(const void* __restrict__ w, int w_dtype, int K, int cout, int cin,
                                   bf16* __restrict__ wt) {
  ::vp::pdl_begin();
  // wt[k, ci, co] = w[k, co, ci]
  const int64_t total = (int64_t)K * cout * cin;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / ((int64_t)cout * cin);
    const int64_t r = e - k * cout * cin;
    const int co = (int)(r / cin), ci = (int)(r - (int64_t)co * cin);
    wt[k * cin * cout + (int64_t)ci * cout + co] = __float2bfloat16_rn(ldf(w, w_dtype, e));
  }
}

__global__ void cast_kernel(const void* __restrict__ src, int sd, void* __restrict__ dst, int dd, int64_t n) {
  ::vp::pdl_begin();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    stf(dst, dd, i, ldf(src, sd, i));
}

// Small C_in (the occupancy stem, C_in = 1): thread per output row, weights
// broadcast from shared memory as [K][C_in][C_out], 32 outputs per pass.
__global__ void __launch_bounds__(128)
conv_fwd_small_kernel(const void* __restrict__ x, int x_dtype, int cin, const void* __restrict__ w, int w_dtype,
                      int cout, int K, const int32_t* __restrict__ table, int flip,
                      const int32_t* __restrict__ perm, const int32_t* n_out_dev, int64_t cap_out,
                      void* __restrict__ y, int y_dtype) {
  ::vp::pdl_begin();
  extern __shared__ float s_w[];  // [K][cin][cout]
  for (int e = threadIdx.x; e < K * cin * cout; e += blockDim.x) {
    const int k = e / (cin * cout), r = e - k * cin * cout, ci = r / cout, co = r - ci * cout;
    s_w[e] = ldf(w, w_dtype, ((int64_t)k * cout + co) * cin + ci);
  }
  __syncthreads();
  const int n_out = load_count(n_out_dev, cap_out);
  for (int64_t ut = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ut < n_out; ut += (int64_t)gridDim.x * blockDim.x) {
    const int32_t* trow = table + ut * K;
    const int64_t u = perm ? (int64_t)perm[ut] : ut;  // output row of table row ut
    float xk[27];
    const bool fast = (cin == 1 && K == 27);
    if (fast) {  // occupancy stem: all 27 index loads, then all 27 feature loads, in flight at once
      int vk[27];
#pragma unroll
      for (int k = 0; k < 27; ++k) vk[k] = __ldg(trow + (flip ? 26 - k : k));
#pragma unroll
      for (int k = 0; k < 27; ++k) xk[k] = vk[k] >= 0 ? ldf(x, x_dtype, vk[k]) : 0.f;
    }
    for (int c0 = 0; c0 < cout; c0 += 32) {
      float acc[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) acc[c] = 0.f;
      if (fast) {
#pragma unroll
        for (int k = 0; k < 27; ++k) {
          const float* wr = s_w + k * cout + c0;
#pragma unroll
          for (int c = 0; c < 32; ++c) acc[c] += (c0 + c < cout) ? wr[c] * xk[k] : 0.f;
        }
      }
      for (int k = 0; k < (fast ? 0 : K); ++k) {
        const int v = __ldg(trow + (flip ? K - 1 - k : k));
        if (v < 0) continue;
        for (int ci = 0; ci < cin; ++ci) {
          const float xv = ldf(x, x_dtype, (int64_t)v * cin + ci);
          const float* wr = s_w + (k * cin + ci) * cout + c0;
#pragma unroll
          for (int c = 0; c < 32; ++c) acc[c] += (c0 + c < cout) ? wr[c] * xv : 0.f;
        }
      }
      if (c0 + 32 <= cout && (cout & 7) == 0 && y_dtype == VP_BF16) {
        uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(y) + u * cout + c0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 pk;
          __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
          for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(acc[8 * q + 2 * e], acc[8 * q + 2 * e + 1]);
          dst[q] = pk;
        }
      } else if (c0 + 32 <= cout && (cout & 3) == 0 && y_dtype == VP_F32) {
        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + u * cout + c0);
#pragma unroll
        for (int q = 0; q < 8; ++q) dst[q] = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
      } else {
        for (int c = 0; c < 32 && c0 + c < cout; ++c) stf(y, y_dtype, u * cout + c0 + c, acc[c]);
      }
    }
  }
}

// Occupancy stem (C_in = 1, 3^3, C_out multiple of 32, bf16 out): a CTA owns
// 128 rows; the [128, 27] neighbour slice is staged coalesced in shared
// memory, each thread gathers its row's 27 inputs (all loads in flight),
// accumulates 32 outputs per pass against broadcast weights, and the bf16
// output tile is written back through shared memory with coalesced stores.
constexpr int kStemRows = 128;
// XT: input and weight dtype fixed at compile time (-1 = runtime), so the 27
// gathers of a row are independent loads in flight rather than a chain of
// dtype branches
// 16 output channels per pass keeps a thread at <= 64 registers: 8 CTAs per
// SM, so C3's ~900 tiles run as one wave (at 128 registers they took two).
constexpr int kStemPass = 16;
constexpr int kStemCluster = 4;  // CTAs per cluster when the stem also writes BN statistics
template <int XT, bool MMA = false>
__global__ void __launch_bounds__(kStemRows, 8)
conv_stem_kernel(const void* __restrict__ x, int x_dtype, const void* __restrict__ w, int w_dtype, int cout,
                 const int32_t* __restrict__ table, int flip, const int32_t* __restrict__ perm,
                 const int32_t* n_out_dev, int64_t cap_out, __nv_bfloat16* __restrict__ y, const BnEpi bn) {
  ::vp::pdl_begin();
  extern __shared__ float s_mem[];
  float* s_w = s_mem;                                             // [27][cout]
  int* s_t = reinterpret_cast<int*>(s_w + 27 * cout);             // [128][27]
  uint32_t* s_o = reinterpret_cast<uint32_t*>(s_t + kStemRows * 27);  // [128][8 + 1] packed bf16 pairs
  // BN statistics (e.mode == 1): this CTA's per-channel (sum, sum^2) of the
  // stored bf16 outputs, accumulated tile by tile by a fixed owner thread
  float* s_acc = reinterpret_cast<float*>(s_o + kStemRows * 9);   // [2][cout]
  float* s_wp = s_acc + 2 * cout;                                 // [4 warps][8 pairs][4]
  const bool stats = bn.mode == 1;
  if (stats) {
    for (int c = threadIdx.x; c < 2 * cout; c += kStemRows) s_acc[c] = 0.f;
    if (blockIdx.x == 0 && threadIdx.x == 0) *bn.nb = gridDim.x / kStemCluster;
  }
#pragma unroll 8
  for (int e = threadIdx.x; e < 27 * cout; e += kStemRows) {
    if (XT == VP_BF16)
      s_w[e] = __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(w) + e));
    else if (XT == VP_F32)
      s_w[e] = __ldg(reinterpret_cast<const float*>(w) + e);
    else
      s_w[e] = ldf(w, w_dtype, e);
  }
  const int n_out = load_count(n_out_dev, cap_out);
  const int ntiles = (n_out + kStemRows - 1) / kStemRows;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t u0 = (int64_t)tile * kStemRows;
    const int rows = min(kStemRows, (int)(n_out - u0));
    __syncthreads();
    const int32_t* tb = table + u0 * 27;
    if ((reinterpret_cast<uintptr_t>(table) & 15) == 0) {
      // 16 B loads, all in flight (a tile's table is 864 int4)
      const int n4 = rows * 27 / 4;
#pragma unroll
      for (int j = 0; j < (kStemRows * 27 / 4 + kStemRows - 1) / kStemRows; ++j) {
        const int e = threadIdx.x + j * kStemRows;
        if (e < n4) reinterpret_cast<int4*>(s_t)[e] = __ldg(reinterpret_cast<const int4*>(tb) + e);
      }
      for (int e = n4 * 4 + threadIdx.x; e < rows * 27; e += kStemRows) s_t[e] = __ldg(tb + e);
    } else {
#pragma unroll 4
      for (int e = threadIdx.x; e < rows * 27; e += kStemRows) s_t[e] = __ldg(tb + e);
    }
    __syncthreads();
    // bf16, C_out = 32: the tile is one 128 x 32 x 32 (K = 27 zero-padded)
    // product on the tensor cores (mma.sync m16n8k16, fp32 accumulate): warp
    // w owns rows 32 w .. 32 w + 31 (two m16 tiles), all four n8 tiles
    static_assert(!MMA || XT == VP_BF16, "the tensor-core stem takes bf16 inputs and weights");
    constexpr bool use_mma = MMA;  // launched only for C_out = 32
    uint32_t af[2][2][4];  // A fragments [m16 tile][k16 step][reg], gathered once per tile
    if (use_mma) {
      const int t = threadIdx.x & 31, wq = threadIdx.x >> 5;
      const unsigned short* xs = reinterpret_cast<const unsigned short*>(x);
      auto xat = [&](int row, int k) -> uint32_t {  // raw bf16 bits of A[row][k]
        if (row >= rows || k >= 27) return 0u;
        const int e = s_t[row * 27 + (flip ? 26 - k : k)];
        return e >= 0 ? (uint32_t)__ldg(xs + e) : 0u;
      };
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int row = wq * 32 + mi * 16 + (t >> 2) + ((q & 1) ? 8 : 0);
            const int k = ks * 16 + (t & 3) * 2 + ((q & 2) ? 8 : 0);
            af[mi][ks][q] = xat(row, k) | (xat(row, k + 1) << 16);
          }
    }
    float xk[27];
    const bool valid = threadIdx.x < rows;
#pragma unroll
    for (int k = 0; k < 27; ++k) {
      if (use_mma) break;
      const int v = valid ? s_t[threadIdx.x * 27 + (flip ? 26 - k : k)] : -1;
      if (XT == VP_BF16)
        xk[k] = v >= 0 ? __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(x) + v)) : 0.f;
      else if (XT == VP_F32)
        xk[k] = v >= 0 ? __ldg(reinterpret_cast<const float*>(x) + v) : 0.f;
      else
        xk[k] = v >= 0 ? ldf(x, x_dtype, v) : 0.f;
    }
    for (int c0 = 0; c0 < cout; c0 += kStemPass) {
      if (use_mma) {
        // this pass's 16 channels = n8 tiles c0/8, c0/8 + 1: B fragments from
        // the staged weights (exact bf16), 8 MMAs, packed pairs of rows r0, r0 + 8
        const int t = threadIdx.x & 31, wq = threadIdx.x >> 5;
        uint32_t bf[2][2][2];
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int k = ks * 16 + (t & 3) * 2 + h * 8, n = c0 + 8 * jj + (t >> 2);
              const float w0 = k < 27 ? s_w[k * 32 + n] : 0.f, w1 = k + 1 < 27 ? s_w[(k + 1) * 32 + n] : 0.f;
              __nv_bfloat162 hw = __floats2bfloat162_rn(w0, w1);
              bf[jj][ks][h] = *reinterpret_cast<uint32_t*>(&hw);
            }
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int ks = 0; ks < 2; ++ks)
              asm volatile(
                  "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                  "{%0,%1,%2,%3};"
                  : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                  : "r"(af[mi][ks][0]), "r"(af[mi][ks][1]), "r"(af[mi][ks][2]), "r"(af[mi][ks][3]),
                    "r"(bf[jj][ks][0]), "r"(bf[jj][ks][1]));
            const int r0 = wq * 32 + mi * 16 + (t >> 2), pair = 4 * jj + (t & 3);
            __nv_bfloat162 h0 = __floats2bfloat162_rn(d[0], d[1]), h1 = __floats2bfloat162_rn(d[2], d[3]);
            s_o[r0 * 9 + pair] = *reinterpret_cast<uint32_t*>(&h0);
            s_o[(r0 + 8) * 9 + pair] = *reinterpret_cast<uint32_t*>(&h1);
          }
      } else {
      float acc[kStemPass];
#pragma unroll
      for (int c = 0; c < kStemPass; ++c) acc[c] = 0.f;
#pragma unroll
      for (int k = 0; k < 27; ++k) {
        const float4* wr = reinterpret_cast<const float4*>(s_w + k * cout + c0);  // broadcast, 16 B aligned
#pragma unroll
        for (int q = 0; q < kStemPass / 4; ++q) {
          const float4 w4 = wr[q];
          acc[4 * q] += w4.x * xk[k];
          acc[4 * q + 1] += w4.y * xk[k];
          acc[4 * q + 2] += w4.z * xk[k];
          acc[4 * q + 3] += w4.w * xk[k];
        }
      }
#pragma unroll
      for (int c = 0; c < kStemPass / 2; ++c) {
        __nv_bfloat162 h = __floats2bfloat162_rn(acc[2 * c], acc[2 * c + 1]);
        s_o[threadIdx.x * 9 + c] = *reinterpret_cast<uint32_t*>(&h);
      }
      }  // FMA path
      __syncthreads();
      // coalesced: word e of the tile -> row e / 8, pair e % 8
      for (int el = threadIdx.x; el < rows * 8; el += kStemRows) {
        const int rr = el >> 3, c = el & 7;
        const int64_t orow = perm ? (int64_t)__ldg(perm + u0 + rr) : u0 + rr;
        reinterpret_cast<uint32_t*>(y + orow * cout + c0)[c] = s_o[rr * 9 + c];
      }
      if (stats) {
        // thread t: channel pair t & 7 over rows 8*(t>>3) .. +8, then an xor
        // tree over the warp's 4 row groups, then the 4 warps in order
        const int cp = threadIdx.x & 7, rg = threadIdx.x >> 3;
        float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int rr = rg * 8 + r;
          if (rr < rows) {
            const uint32_t pk = s_o[rr * 9 + cp];
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk));
            a0 += f.x;
            a1 += f.y;
            b0 += f.x * f.x;
            b1 += f.y * f.y;
          }
        }
#pragma unroll
        for (int m = 8; m < 32; m <<= 1) {
          a0 += __shfl_xor_sync(0xffffffffu, a0, m);
          a1 += __shfl_xor_sync(0xffffffffu, a1, m);
          b0 += __shfl_xor_sync(0xffffffffu, b0, m);
          b1 += __shfl_xor_sync(0xffffffffu, b1, m);
        }
        const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
        if (lane < 8) {
          float* d = s_wp + (wp * 8 + lane) * 4;
          d[0] = a0;
          d[1] = a1;
          d[2] = b0;
          d[3] = b1;
        }
        __syncthreads();
        if (threadIdx.x < kStemPass) {  // channel c0 + t: pair t/2, half t&1
          const int t = threadIdx.x, pr = t >> 1, hf = t & 1;
          float sa = 0.f, sb = 0.f;
#pragma unroll
          for (int w4 = 0; w4 < 4; ++w4) {
            sa += s_wp[(w4 * 8 + pr) * 4 + hf];
            sb += s_wp[(w4 * 8 + pr) * 4 + 2 + hf];
          }
          s_acc[c0 + t] += sa;
          s_acc[cout + c0 + t] += sb;
        }
      }
      __syncthreads();
    }
  }
  if (stats) {
    // the cluster's CTAs in rank order -> one partial row per cluster
    // (launched with kStemCluster-CTA clusters: a full one-wave grid, few rows)
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    if (cl.block_rank() == 0) {
      for (int c = threadIdx.x; c < 2 * cout; c += kStemRows) {
        float acc = 0.f;
        for (int r = 0; r < kStemCluster; ++r) acc += cl.map_shared_rank(s_acc, r)[c];
        bn.part[(int64_t)(blockIdx.x / kStemCluster) * 2 * cout + c] = acc;
      }
    }
    cl.sync();  // remote shared memory stays alive until rank 0 has read it
  }
}

// 32-wide sparse levels: the row-compacted mma.sync kernel (conv_rows.cuh)
// instead of the tcgen05 tile.  Opt-in (VP_CONV_ROWS=1): measured 2.1-2.3x
// slower at C3 (8 warps/SM with ~100-instruction dependent chains per offset;
// DESIGN.md §10), kept as the starting point for a compacted path.
static bool rows32_ok(int64_t cin, int64_t cout, int K) {
  static const bool on = getenv("VP_CONV_ROWS") && atoi(getenv("VP_CONV_ROWS")) == 1;
  return on && cin == 32 && cout == 32 && K <= 27;
}

template <bool WT>
static int launch_rows32(const bf16* x, const bf16* w, int K, const int32_t* table, int flip, const int32_t* perm,
                         const int32_t* n_out_dev, int64_t cap_out, void* y, int yd, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    VP_REQUIRE(cudaFuncSetAttribute(conv_rows32_kernel<WT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    RowsSmem::TOTAL) == cudaSuccess,
               VP_EINTERNAL, "conv_rows32: cannot reserve shared memory");
    attr = true;
  }
  const int64_t slices = ceil_div(cap_out, 32);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(slices, kRowsWarps), kNumSMs));
  ::vp::launch(conv_rows32_kernel<WT>, grid, kRowsWarps * 32, RowsSmem::TOTAL, st, x, w, K, table, flip, perm,
               n_out_dev, cap_out, y, yd);
  VP_CHECK_LAUNCH("conv_rows32");
  return VP_OK;
}

static bool small_fwd_ok(int64_t cin, int64_t cout, int K) { return cin <= 4 && (int64_t)K * cin * cout <= 12288; }

// epi: BN statistics from the stem kernel (mode 1) when it runs; the caller
// runs the generic pass otherwise (*fused reports which)
static int launch_small_fwd(const void* x, int xd, int cin, const void* w, int wd, int cout, int K,
                            const int32_t* table, int flip, const int32_t* perm, const int32_t* n_out_dev,
                            int64_t cap_out, void* y, int yd, cudaStream_t st, const BnEpi& epi = BnEpi{},
                            bool* fused = nullptr) {
  int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cap_out, 128), grid_cap(8)));
  if (fused) *fused = false;
  if (cin == 1 && K == 27 && cout % 32 == 0 && cout <= 256 && yd == VP_BF16) {
    const size_t smem = (size_t)27 * cout * 4 + kStemRows * 27 * 4 + kStemRows * 9 * 4 + 2 * cout * 4 + 4 * 8 * 4 * 4;
    const int dt = xd == wd ? xd : -1;
    // bf16 with C_out = 32: the mma.sync instance (VP_STEM_MMA=0: the FMA one)
    static const bool stem_mma = !(getenv("VP_STEM_MMA") && atoi(getenv("VP_STEM_MMA")) == 0);
    auto kern = dt == VP_BF16 ? ((stem_mma && cout == 32) ? conv_stem_kernel<VP_BF16, true> : conv_stem_kernel<VP_BF16>)
                : dt == VP_F32 ? conv_stem_kernel<VP_F32> : conv_stem_kernel<-1>;
    BnEpi e = epi.mode == 1 ? epi : BnEpi{};
    if (e.mode == 1) {  // clusters of kStemCluster CTAs, one partial row each
      blocks = (int)std::min<int64_t>(ceil_div(blocks, kStemCluster) * kStemCluster, (int64_t)kBnPartRows * kStemCluster);
      if (fused) *fused = true;
      ::vp::launch_cluster(kern, kStemCluster, blocks, kStemRows, smem, st, x, xd, w, wd, cout, table, flip, perm,
                           n_out_dev, cap_out, (__nv_bfloat16*)y, e);
    } else {
      ::vp::launch(kern, blocks, kStemRows, smem, st, x, xd, w, wd, cout, table, flip, perm, n_out_dev, cap_out,
                   (__nv_bfloat16*)y, e);
    }
    VP_CHECK_LAUNCH("conv_stem");
    return VP_OK;
  }
  ::vp::launch(conv_fwd_small_kernel, blocks, 128, (size_t)K * cin * cout * 4, st, x, xd, cin, w, wd, cout, K, table, flip,
                                                                         perm, n_out_dev, cap_out, y, yd);
  VP_CHECK_LAUNCH("conv_fwd_small");
  return VP_OK;
}

// ------------------------------------------------------------------ BN epilogue (generic)
// The bn_epi.cuh transform for the paths without a fused epilogue (SIMT,
// stem, fp32/f64 outputs, the row-compacted kernel): one pass over the
// conv's output rows in place after the conv.  Block b owns rows b, b+G, ...
// (lanes rows at a time); per-channel sums in a fixed order.
__device__ __forceinline__ float round_to(int dtype, float v) { return dtype == VP_BF16 ? bf16_round(v) : v; }

__global__ void __launch_bounds__(256)
bn_epi_rows_kernel(void* __restrict__ y, int yd, const int32_t* n_dev, int64_t cap, int C, const BnEpi e) {
  ::vp::pdl_begin();
  __shared__ float s_a[256], s_b[256];
  const int n = load_count(n_dev, cap);
  if (blockIdx.x == 0 && threadIdx.x == 0) *e.nb = gridDim.x;
  for (int c0 = 0; c0 < C; c0 += 256) {
    const int cc = min(256, C - c0);
    const int lanes = 256 / cc;
    const int c = c0 + (int)threadIdx.x % cc, lr = (int)threadIdx.x / cc;
    float a = 0.f, b = 0.f;
    if (lr < lanes) {
      const float mu = e.mode == 2 ? e.mean[c] : 0.f;
      for (int64_t r = (int64_t)blockIdx.x * lanes + lr; r < n; r += (int64_t)gridDim.x * lanes) {
        const int64_t i = r * C + c;
        const float v = ldf(y, yd, i);
        if (e.mode == 2) {
          float g = v + (e.add ? ldf(e.add, yd, i) : 0.f);
          g = (e.act == nullptr || ldf(e.act, yd, i) > 0.f) ? round_to(yd, g) : 0.f;
          stf(y, yd, i, g);
          a += g;
          b += g * (ldf(e.pre, yd, i) - mu);
        } else {
          a += v;
          b += v * v;
        }
      }
    }
    s_a[threadIdx.x] = a;
    s_b[threadIdx.x] = b;
    __syncthreads();
    if ((int)threadIdx.x < cc) {
      float sa = 0.f, sb = 0.f;
      for (int l = 0; l < lanes; ++l) {
        sa += s_a[l * cc + threadIdx.x];
        sb += s_b[l * cc + threadIdx.x];
      }
      e.part[((int64_t)blockIdx.x * 2) * C + c0 + threadIdx.x] = sa;
      e.part[((int64_t)blockIdx.x * 2 + 1) * C + c0 + threadIdx.x] = sb;
    }
    __syncthreads();
  }
}

static int launch_bn_finalize(const BnEpi& e, int64_t C, const int32_t* n_dev, int64_t cap, cudaStream_t st) {
  if (e.mode == 0 || e.out_a == nullptr) return VP_OK;
  ::vp::launch(bn_finalize_kernel, (int)ceil_div(C, 32), 1024, 0, st, e, (int)C, n_dev, cap);
  VP_CHECK_LAUNCH("bn_finalize");
  return VP_OK;
}

static int launch_bn_epi_rows(void* y, int yd, const int32_t* n_dev, int64_t cap, int64_t C, const BnEpi& e,
                              cudaStream_t st) {
  const int64_t lanes = std::max<int64_t>(1, 256 / std::min<int64_t>(C, 256));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(std::max<int64_t>(cap, 1), lanes * 8), kNumSMs));
  ::vp::launch(bn_epi_rows_kernel, grid, 256, 0, st, y, yd, n_dev, cap, (int)C, e);
  VP_CHECK_LAUNCH("bn_epi_rows");
  return launch_bn_finalize(e, C, n_dev, cap, st);
}

static int bn_early_env() {  // early programmatic launch of the BN apply behind the finalize (VP_BN_EARLY)
  static const int v = getenv("VP_BN_EARLY") ? atoi(getenv("VP_BN_EARLY")) : 1;
  return v;
}

// caller buffer -> BnEpi (header: int nb at 0, the finalize ticket at
// kBnTicketOffset; partial rows after kBnPartHeader bytes)
static BnEpi make_epi(int32_t mode, void* bn_part, const void* add, const void* act, const void* pre,
                      const float* mean, float eps, float* out_a, float* out_b, const float* rstd) {
  BnEpi e{};
  e.mode = bn_part ? mode : 0;
  e.nb = (int*)bn_part;
  e.part = bn_part ? (float*)((char*)bn_part + kBnPartHeader) : nullptr;
  e.add = add;
  e.act = act;
  e.pre = pre;
  e.mean = mean;
  e.out_a = out_a;
  e.out_b = out_b;
  e.rstd = rstd;
  e.eps = eps;
  e.ticket = bn_part ? (unsigned int*)((char*)bn_part + kBnTicketOffset) : nullptr;
  e.early = bn_early_env();
  return e;
}

// ------------------------------------------------------------------ dispatch
static bool tc_width(int64_t c) { return c == 32 || c == 64 || c == 128 || c == 256; }
// tile width of a tensor-core operand of c 2-byte units (c % 8 == 0: 16 B
// rows), 0 when the tensor cores do not take it
static int64_t tc_pad(int64_t c) {
  if (c < 8 || c % 8 != 0 || c > 256) return 0;
  return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : 256;
}

// wt[k, ci, co] = w[k, co, ci] in fp32 (the tf32 dgrad's K-major B operand)
__global__ void transpose_w_f32_kernel(const void* __restrict__ w, int wd, float* __restrict__ wt, int K, int cout,
                                   int cin) {
  ::vp::pdl_begin();
  const int64_t total = (int64_t)K * cin * cout;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / ((int64_t)cin * cout);
    const int64_t r = e - k * cin * cout;
    const int ci = (int)(r / cout), co = (int)(r - (int64_t)ci * cout);
    wt[e] = ldf(w, wd, (k * cout + co) * cin + ci);
  }
}

template <bool BMN>
static int conv_tc(int64_t kd, int64_t nd, const FwdParams& p, void* part, cudaStream_t st) {
  switch (kd) {
    case 32: return BMN ? conv_tc_k32_d(nd, p, part, st) : conv_tc_k32_f(nd, p, part, st);
    case 64: return BMN ? conv_tc_k64_d(nd, p, part, st) : conv_tc_k64_f(nd, p, part, st);
    case 128: return BMN ? conv_tc_k128_d(nd, p, part, st) : conv_tc_k128_f(nd, p, part, st);
    case 256: return BMN ? conv_tc_k256_d(nd, p, part, st) : conv_tc_k256_f(nd, p, part, st);
  }
  return VP_EINTERNAL;
}

static size_t split_ws_bytes(int64_t nd) { return align_up((size_t)kSplitItems * 128 * nd * 4, 256); }

// the split-phase weight gradient of the training step (vp_conv_wgrad_sgd,
// phases 1 / 2) runs on the side streams beside the critical path: its
// persistent grid is capped at 96 of the 148 SMs (VP_WGRAD_SMS; C3 A/B on
// one box: 148 -> 54.65k, 130 -> 54.87k, 110 -> 55.1k, 96 -> 55.2k, 84-90
// -> 55.2k, 74 -> 54.7k clouds/s).  A single-call weight gradient (the
// operator API, phase 0) takes the whole GPU.
constexpr int kWgSms = 96;
// ... for layers up to this pair capacity (C3's largest: 131,072 rows x 27);
// the C5-scale layers' weight gradients (tens of millions of pairs) keep all
// SMs (capped, C5 11.76k -> 11.53k clouds/s)
constexpr int64_t kWgSideCapPairs = 4 << 20;

static int wgrad_cps() {  // CTAs per SM of the weight-gradient kernel where two fit (VP_WGRAD_CPS overrides)
  static const int v = getenv("VP_WGRAD_CPS") ? atoi(getenv("VP_WGRAD_CPS")) : 2;
  return v;
}

template <int CIN, int COUT, int CPS>
static int launch_wg_tc_cps(const WgParams& p, int max_items, cudaStream_t st) {
  using C = WgTC<CIN, COUT, CPS>;
  auto kern = conv_wgrad_tc_kernel<CIN, COUT, CPS>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  // persistent, on at most kWgSms SMs: the weight gradient runs on a side
  // stream next to the critical path (BN / dgrad); leaving SMs free for the
  // high-priority kernels shortens the step (VP_WGRAD_SMS overrides)
  const int grid = std::max(1, std::min(max_items, p.sms * CPS));
  ::vp::launch(kern, grid, kTcThreads, C::SMEM, st, p);
  VP_CHECK_LAUNCH("conv_wgrad_tc");
  return VP_OK;
}

template <int CIN, int COUT>
static int launch_wg_tc(const WgParams& p, int max_items, cudaStream_t st) {
  if constexpr (WgTC<CIN, COUT, 2>::FITS) {
    if (wgrad_cps() == 2) return launch_wg_tc_cps<CIN, COUT, 2>(p, max_items, st);
  }
  return launch_wg_tc_cps<CIN, COUT, 1>(p, max_items, st);
}

template <int CIN>
static int wg_tc_cout(int64_t cout, const WgParams& p, int mi, cudaStream_t st) {
  switch (cout) {
    case 32: return launch_wg_tc<CIN, 32>(p, mi, st);
    case 64: return launch_wg_tc<CIN, 64>(p, mi, st);
    case 128: return launch_wg_tc<CIN, 128>(p, mi, st);
    case 256: return launch_wg_tc<CIN, 256>(p, mi, st);
  }
  return VP_EINTERNAL;
}

static int wg_tc(int64_t cin, int64_t cout, const WgParams& p, int mi, cudaStream_t st) {
  switch (cin) {
    case 32: return wg_tc_cout<32>(cout, p, mi, st);
    case 64: return wg_tc_cout<64>(cout, p, mi, st);
    case 128: return wg_tc_cout<128>(cout, p, mi, st);
    case 256: return wg_tc_cout<256>(cout, p, mi, st);
  }
  return VP_EINTERNAL;
}

// pairs per work item: ~2 items per SM at the pair capacity, multiple of 64,
// depends only on static capacities -> results independent of timing
static int wgrad_chunk(int64_t cap_pairs) {
  // cap on the chunk (VP_WGRAD_MAX_CHUNK, tuning; multiple of 64, <= kWgMaxChunk)
  static const int64_t cap = getenv("VP_WGRAD_MAX_CHUNK")
                                 ? std::max<int64_t>(256, std::min<int64_t>(kWgMaxChunk, atoll(getenv("VP_WGRAD_MAX_CHUNK")) / 64 * 64))
                                 : kWgMaxChunk;
  int64_t c = ceil_div(std::max<int64_t>(cap_pairs, 1), 2 * kNumSMs);
  c = ceil_div(c, 64) * 64;
  return (int)std::min<int64_t>(std::max<int64_t>(c, 256), cap);
}

}  // namespace vp

using namespace vp;

extern "C" {

int vp_debug_conv_trace(long long* buf) {
  g_conv_trace_host = buf;
  return VP_OK;
}

// weights cast / transposed (up to fp32) + the split-K partials of the padded tile width
static int64_t split_width(int64_t c) { return std::max<int64_t>(tc_pad(c), std::min<int64_t>(c, 256)); }
int32_t vp_conv_tc_grid(int64_t nd, int64_t cap_out) {
  // the default config's CTA count of a tensor-core conv writing nd-wide rows
  // (launch_conv_tc): the G of the grouping's tile schedule
  const int64_t w = tc_pad(nd);
  if (w == 0) return 0;
  const int64_t tiles = ceil_div(std::max<int64_t>(cap_out, 1), 128);
  return (int32_t)std::min<int64_t>(tiles * kMaxSplit, (int64_t)kNumSMs * kCfgCps[conv_cfg(w, cap_out)]);
}

size_t vp_conv_fwd_ws_bytes(int64_t cin, int64_t cout, int32_t K) {
  return align_up((size_t)K * cin * cout * 4, 256) + split_ws_bytes(split_width(cout));
}

static int conv_fwd_impl(const void* x, int32_t x_dtype, int64_t x_rows, int64_t cin, const void* w, int32_t w_dtype,
                         int64_t cout, int32_t K, const int32_t* table, int32_t flip, const int32_t* perm,
                         const int32_t* n_out_dev, int64_t cap_out, void* y, int32_t y_dtype, void* ws, size_t ws_bytes,
                         const BnEpi& epi, cudaStream_t st);

int vp_conv_fwd(const void* x, int32_t x_dtype, int64_t x_rows, int64_t cin, const void* w, int32_t w_dtype, int64_t cout,
                int32_t K, const int32_t* table, int32_t flip, const int32_t* perm, const int32_t* n_out_dev,
                int64_t cap_out, void* y, int32_t y_dtype, void* ws, size_t ws_bytes, vp_stream_t stream) {
  return conv_fwd_impl(x, x_dtype, x_rows, cin, w, w_dtype, cout, K, table, flip, perm, n_out_dev, cap_out, y, y_dtype,
                       ws, ws_bytes, BnEpi{}, (cudaStream_t)stream);
}

size_t vp_bn_part_bytes(int64_t C) { return kBnPartHeader + (size_t)kBnPartRows * 2 * std::max<int64_t>(C, 1) * 4; }

int vp_conv_fwd_bn(const void* x, int32_t x_dtype, int64_t x_rows, int64_t cin, const void* w, int32_t w_dtype,
                   int64_t cout, int32_t K, const int32_t* table, int32_t flip, const int32_t* perm,
                   const int32_t* n_out_dev, int64_t cap_out, void* y, int32_t y_dtype, void* ws, size_t ws_bytes,
                   int32_t bn_mode, void* bn_part, const void* bn_add, const void* bn_act, const void* bn_pre,
                   const float* bn_mean, float bn_eps, float* bn_out_a, float* bn_out_b, const float* bn_rstd,
                   vp_stream_t stream) {
  VP_REQUIRE(bn_mode >= 0 && bn_mode <= 2 && (bn_mode == 0 || bn_part), VP_EVALIDATION, "conv_fwd_bn: bad bn mode");
  VP_REQUIRE(bn_mode != 2 || (bn_pre && bn_mean), VP_EVALIDATION, "conv_fwd_bn: mode 2 needs pre and mean");
  VP_REQUIRE(!bn_out_a == !bn_out_b && (bn_mode != 2 || !bn_out_a || bn_rstd), VP_EVALIDATION,
             "conv_fwd_bn: finalize outputs (and rstd for mode 2) go together");
  return conv_fwd_impl(x, x_dtype, x_rows, cin, w, w_dtype, cout, K, table, flip, perm, n_out_dev, cap_out, y, y_dtype,
                       ws, ws_bytes,
                       make_epi(bn_mode, bn_part, bn_add, bn_act, bn_pre, bn_mean, bn_eps, bn_out_a, bn_out_b, bn_rstd),
                       (cudaStream_t)stream);
}

static int conv_fwd_impl(const void* x, int32_t x_dtype, int64_t x_rows, int64_t cin, const void* w, int32_t w_dtype,
                         int64_t cout, int32_t K, const int32_t* table, int32_t flip, const int32_t* perm,
                         const int32_t* n_out_dev, int64_t cap_out, void* y, int32_t y_dtype, void* ws, size_t ws_bytes,
                         const BnEpi& epi, cudaStream_t st) {
  // the generic BN pass after any conv path without a fused epilogue
  auto epi_after = [&](int rc) -> int {
    if (rc != VP_OK || epi.mode == 0) return rc;
    return launch_bn_epi_rows(y, y_dtype, n_out_dev, cap_out, cout, epi, st);
  };
  VP_REQUIRE(K >= 1 && K <= VP_MAX_OFFSETS, VP_EVALIDATION, "kernel offset count out of range");
  VP_REQUIRE(cin >= 1 && cout >= 1, VP_EVALIDATION, "channel widths must be positive");
  VP_REQUIRE(y_dtype == VP_F32 || y_dtype == VP_BF16 || y_dtype == VP_F64, VP_EVALIDATION,
             "output dtype must be f32, bf16 or f64");
  if (cap_out <= 0) return epi_after(VP_OK);
  const bool f64 = x_dtype == VP_F64 || w_dtype == VP_F64 || y_dtype == VP_F64;
  if (x_dtype == VP_TF32) {
    // fp32 features, tf32 tensor-core math: the bf16 tile machinery over
    // 2-byte units (an fp32 row of C is 2C units; K = 8 tf32 per MMA = 32 B)
    if (!f64 && tc_pad(2 * cin) && tc_pad(cout) && y_dtype != VP_F64) {
      VP_REQUIRE(ws && ws_bytes >= vp_conv_fwd_ws_bytes(cin, cout, K), VP_EVALIDATION, "conv_fwd: workspace too small");
      const float* wf = (const float*)w;
      if (w_dtype != VP_F32 && w_dtype != VP_TF32) {
        const int64_t cnt = (int64_t)K * cin * cout;
        ::vp::launch(cast_kernel, (int)std::min<int64_t>(ceil_div(cnt, 256), 1184), 256, 0, st, w, w_dtype, ws, VP_F32, cnt);
        VP_CHECK_LAUNCH("conv_fwd: cast w (tf32)");
        wf = (const float*)ws;
      }
      char* part = (char*)ws + align_up((size_t)K * cin * cout * 4, 256);
      FwdParams p{(const bf16*)x, (const bf16*)wf, K, table, flip, perm, n_out_dev, cap_out, y, y_dtype, nullptr, 1, 0, 0};
      p.kreal = (int)(2 * cin);
      p.nreal = (int)cout;
      return epi_after(conv_tc_tf32(tc_pad(2 * cin), tc_pad(cout), p, part, st));
    }
    x_dtype = VP_F32;  // exact fp32 SIMT path
  }
  if (w_dtype == VP_TF32) w_dtype = VP_F32;
  if (!f64 && x_dtype == VP_BF16 && tc_pad(cin) && tc_pad(cout)) {
    VP_REQUIRE(ws && ws_bytes >= vp_conv_fwd_ws_bytes(cin, cout, K), VP_EVALIDATION, "conv_fwd: workspace too small");
    const bool exact = tc_pad(cin) == cin && tc_pad(cout) == cout;
    const bf16* wb = (const bf16*)w;
    char* part = (char*)ws + align_up((size_t)K * cin * cout * 4, 256);
    if (w_dtype != VP_BF16) {
      int64_t cnt = (int64_t)K * cin * cout;
      ::vp::launch(cast_kernel, (int)std::min<int64_t>(ceil_div(cnt, 256), 1184), 256, 0, st, w, w_dtype, ws, VP_BF16, cnt);
      VP_CHECK_LAUNCH("conv_fwd: cast w");
      wb = (const bf16*)ws;
    }
    (void)x_rows;  // the cp.async gather zero-fills missing neighbours itself
    if (exact && rows32_ok(cin, cout, K))
      return epi_after(
          launch_rows32<false>((const bf16*)x, wb, K, table, flip, perm, n_out_dev, cap_out, y, y_dtype, st));
    FwdParams p{(const bf16*)x, wb, K, table, flip, perm, n_out_dev, cap_out, y, y_dtype, nullptr, 1, 0, 0};
    p.kreal = (int)cin;
    p.nreal = (int)cout;
    if (y_dtype == VP_BF16 && exact) {
      p.epi = epi;  // fused into the epilogue / split-K reduction
      return conv_tc<false>(cin, cout, p, part, st);
    }
    if (exact) return epi_after(conv_tc<false>(cin, cout, p, part, st));
    return epi_after(conv_tc_pad_fwd(tc_pad(cin), tc_pad(cout), p, part, st));
  }
  if (!f64 && small_fwd_ok(cin, cout, K)) {
    bool fused = false;
    const int rc = launch_small_fwd(x, x_dtype, (int)cin, w, w_dtype, (int)cout, K, table, flip, perm, n_out_dev,
                                    cap_out, y, y_dtype, st, epi, &fused);
    if (rc != VP_OK) return rc;
    return fused ? launch_bn_finalize(epi, cout, n_out_dev, cap_out, st) : epi_after(rc);
  }
  const int64_t total = cap_out * cout;
  int blocks = (int)std::min<int64_t>(ceil_div(total, 256), grid_cap(16));
  ::vp::launch(f64 ? conv_fwd_simt_kernel<double> : conv_fwd_simt_kernel<float>, blocks, 256, 0, st, x, x_dtype,
               (int)cin, w, w_dtype, cout * cin, cin, 1, (int)cout, K, table, flip, perm, n_out_dev, cap_out, y,
               y_dtype);
  VP_CHECK_LAUNCH("conv_fwd_simt");
  return epi_after(VP_OK);
}

size_t vp_conv_dgrad_ws_bytes(int64_t cin, int64_t cout, int32_t K) {
  return align_up((size_t)K * cin * cout * 4, 256) + split_ws_bytes(split_width(cin));
}

static int conv_dgrad_impl(const void* g, int32_t g_dtype, int64_t g_rows, int64_t cout, const void* w, int32_t w_dtype,
                           int64_t cin, int32_t K, const int32_t* table, int32_t flip, const int32_t* perm,
                           const int32_t* n_in_dev, int64_t cap_in, void* gi, int32_t gi_dtype, void* ws,
                           size_t ws_bytes, const BnEpi& epi, cudaStream_t st);

int vp_conv_dgrad(const void* g, int32_t g_dtype, int64_t g_rows, int64_t cout, const void* w, int32_t w_dtype, int64_t cin,
                  int32_t K, const int32_t* table, int32_t flip, const int32_t* perm, const int32_t* n_in_dev,
                  int64_t cap_in, void* gi, int32_t gi_dtype, void* ws, size_t ws_bytes, vp_stream_t stream) {
  return conv_dgrad_impl(g, g_dtype, g_rows, cout, w, w_dtype, cin, K, table, flip, perm, n_in_dev, cap_in, gi,
                         gi_dtype, ws, ws_bytes, BnEpi{}, (cudaStream_t)stream);
}

int vp_conv_dgrad_bn(const void* g, int32_t g_dtype, int64_t g_rows, int64_t cout, const void* w, int32_t w_dtype,
                     int64_t cin, int32_t K, const int32_t* table, int32_t flip, const int32_t* perm,
                     const int32_t* n_in_dev, int64_t cap_in, void* gi, int32_t gi_dtype, void* ws, size_t ws_bytes,
                     int32_t bn_mode, void* bn_part, const void* bn_add, const void* bn_act, const void* bn_pre,
                     const float* bn_mean, float bn_eps, float* bn_out_a, float* bn_out_b, const float* bn_rstd,
                     vp_stream_t stream) {
  VP_REQUIRE(bn_mode >= 0 && bn_mode <= 2 && (bn_mode == 0 || bn_part), VP_EVALIDATION, "conv_dgrad_bn: bad bn mode");
  VP_REQUIRE(bn_mode != 2 || (bn_pre && bn_mean), VP_EVALIDATION, "conv_dgrad_bn: mode 2 needs pre and mean");
  VP_REQUIRE(!bn_out_a == !bn_out_b && (bn_mode != 2 || !bn_out_a || bn_rstd), VP_EVALIDATION,
             "conv_dgrad_bn: finalize outputs (and rstd for mode 2) go together");
  return conv_dgrad_impl(g, g_dtype, g_rows, cout, w, w_dtype, cin, K, table, flip, perm, n_in_dev, cap_in, gi,
                         gi_dtype, ws, ws_bytes,
                         make_epi(bn_mode, bn_part, bn_add, bn_act, bn_pre, bn_mean, bn_eps, bn_out_a, bn_out_b, bn_rstd),
                         (cudaStream_t)stream);
}

static int conv_dgrad_impl(const void* g, int32_t g_dtype, int64_t g_rows, int64_t cout, const void* w, int32_t w_dtype,
                           int64_t cin, int32_t K, const int32_t* table, int32_t flip, const int32_t* perm,
                           const int32_t* n_in_dev, int64_t cap_in, void* gi, int32_t gi_dtype, void* ws,
                           size_t ws_bytes, const BnEpi& epi, cudaStream_t st) {
  auto epi_after = [&](int rc) -> int {
    if (rc != VP_OK || epi.mode == 0) return rc;
    return launch_bn_epi_rows(gi, gi_dtype, n_in_dev, cap_in, cin, epi, st);
  };
  VP_REQUIRE(K >= 1 && K <= VP_MAX_OFFSETS, VP_EVALIDATION, "kernel offset count out of range");
  VP_REQUIRE(gi_dtype == VP_F32 || gi_dtype == VP_BF16 || gi_dtype == VP_F64, VP_EVALIDATION,
             "grad_in dtype must be f32, bf16 or f64");
  if (cap_in <= 0) return epi_after(VP_OK);
  const bool f64 = g_dtype == VP_F64 || w_dtype == VP_F64 || gi_dtype == VP_F64;
  if (g_dtype == VP_TF32) {
    // tf32: grad_in = sum_k W_k^T g[table] with W^T staged K-major in fp32
    if (!f64 && tc_pad(2 * cout) && tc_pad(cin) && gi_dtype != VP_F64) {
      VP_REQUIRE(ws && ws_bytes >= vp_conv_dgrad_ws_bytes(cin, cout, K), VP_EVALIDATION,
                 "conv_dgrad: workspace too small");
      const int64_t cnt = (int64_t)K * cin * cout;
      ::vp::launch(transpose_w_f32_kernel, (int)std::min<int64_t>(ceil_div(cnt, 256), 1184), 256, 0, st, w,
                   w_dtype == VP_TF32 ? (int)VP_F32 : (int)w_dtype, (float*)ws, K, (int)cout, (int)cin);
      VP_CHECK_LAUNCH("conv_dgrad: transpose w (tf32)");
      char* part = (char*)ws + align_up((size_t)K * cin * cout * 4, 256);
      FwdParams p{(const bf16*)g, (const bf16*)ws, K, table, flip, perm, n_in_dev, cap_in, gi, gi_dtype, nullptr, 1, 0, 0};
      p.kreal = (int)(2 * cout);
      p.nreal = (int)cin;
      return epi_after(conv_tc_tf32(tc_pad(2 * cout), tc_pad(cin), p, part, st));
    }
    g_dtype = VP_F32;
  }
  if (w_dtype == VP_TF32) w_dtype = VP_F32;
  if (!f64 && g_dtype == VP_BF16 && tc_pad(cin) && tc_pad(cout)) {
    VP_REQUIRE(ws && ws_bytes >= vp_conv_dgrad_ws_bytes(cin, cout, K), VP_EVALIDATION,
               "conv_dgrad: workspace too small");
    const bool exact = tc_pad(cin) == cin && tc_pad(cout) == cout;
    const bf16* wb = (const bf16*)w;
    char* part = (char*)ws + align_up((size_t)K * cin * cout * 4, 256);
    if (w_dtype != VP_BF16) {
      int64_t cnt = (int64_t)K * cin * cout;
      ::vp::launch(cast_kernel, (int)std::min<int64_t>(ceil_div(cnt, 256), 1184), 256, 0, st, w, w_dtype, ws, VP_BF16, cnt);
      VP_CHECK_LAUNCH("conv_dgrad: cast w");
      wb = (const bf16*)ws;
    }
    // grad_in = sum_k W_k^T g[table]: GEMM K-dim = C_out, N = C_in, W read as MN-major B
    (void)g_rows;
    if (exact && rows32_ok(cout, cin, K))
      return epi_after(
          launch_rows32<true>((const bf16*)g, wb, K, table, flip, perm, n_in_dev, cap_in, gi, gi_dtype, st));
    FwdParams p{(const bf16*)g, wb, K, table, flip, perm, n_in_dev, cap_in, gi, gi_dtype, nullptr, 1, 0, 0};
    p.kreal = (int)cout;
    p.nreal = (int)cin;
    if (gi_dtype == VP_BF16 && exact) {
      p.epi = epi;
      return conv_tc<true>(cout, cin, p, part, st);
    }
    if (exact) return epi_after(conv_tc<true>(cout, cin, p, part, st));
    return epi_after(conv_tc_pad_dgrad(tc_pad(cout), tc_pad(cin), p, part, st));
  }
  const int64_t total = cap_in * cin;
  int blocks = (int)std::min<int64_t>(ceil_div(total, 256), grid_cap(16));
  // W^T[k, ci, co] = W[k, co, ci]: strides (k: cout*cin, "co"=ci: 1, "ci"=co: cin)
  ::vp::launch(f64 ? conv_fwd_simt_kernel<double> : conv_fwd_simt_kernel<float>, blocks, 256, 0, st, g, g_dtype,
               (int)cout, w, w_dtype, cout * cin, 1, cin, (int)cin, K, table, flip, perm, n_in_dev, cap_in, gi,
               gi_dtype);
  VP_CHECK_LAUNCH("conv_dgrad_simt");
  return epi_after(VP_OK);
}

constexpr int kWgSimtChunk = 512;  // SIMT path: short chunks, many CTAs
constexpr size_t kWgHeader = 256;  // tail of the wgrad workspace: the device-chosen chunk

// fp32 partials of the SIMT chunk size; the f64 path runs chunks twice as
// long, so 8-byte partials of (cap/2chunk + K + 1) items fit the same
// budget with 2(K+1) slack items
size_t vp_conv_wgrad_ws_bytes(int64_t cin, int64_t cout, int32_t K, int64_t cap_pairs) {
  const int chunk = std::min(wgrad_chunk(cap_pairs), kWgSimtChunk);
  const int64_t items = cap_pairs / chunk + 2 * ((int64_t)K + 1);
  return align_up((size_t)items * cin * cout * 4, 256) + kWgHeader;  // + the device-chosen chunk word
}

// phase: 0 = partials + reduction, 1 = partials only, 2 = reduction only
static int conv_wgrad_impl(const void* x, int32_t x_dtype, int64_t cin, const void* g, int32_t g_dtype, int64_t cout,
                           int32_t K, const int32_t* pin, const int32_t* pout, const int32_t* pptr, int64_t cap_pairs,
                           void* gw_out, void* ws, size_t ws_bytes, const SgdFuse& sgd, int phase, cudaStream_t st,
                           bool side = false);

int vp_conv_wgrad(const void* x, int32_t x_dtype, int64_t cin, const void* g, int32_t g_dtype, int64_t cout,
                  int32_t K, const int32_t* pin, const int32_t* pout, const int32_t* pptr, int64_t cap_pairs,
                  void* gw_out, void* ws, size_t ws_bytes, vp_stream_t stream) {
  return conv_wgrad_impl(x, x_dtype, cin, g, g_dtype, cout, K, pin, pout, pptr, cap_pairs, gw_out, ws, ws_bytes,
                         SgdFuse{}, 0, (cudaStream_t)stream);
}

int vp_conv_wgrad_side(const void* x, int32_t x_dtype, int64_t cin, const void* g, int32_t g_dtype, int64_t cout,
                       int32_t K, const int32_t* pin, const int32_t* pout, const int32_t* pptr, int64_t cap_pairs,
                       void* gw_out, void* ws, size_t ws_bytes, vp_stream_t stream) {
  return conv_wgrad_impl(x, x_dtype, cin, g, g_dtype, cout, K, pin, pout, pptr, cap_pairs, gw_out, ws, ws_bytes,
                         SgdFuse{}, 0, (cudaStream_t)stream, true);
}

int vp_conv_wgrad_sgd(const void* x, int32_t x_dtype, int64_t cin, const void* g, int32_t g_dtype, int64_t cout,
                      int32_t K, const int32_t* pin, const int32_t* pout, const int32_t* pptr, int64_t cap_pairs,
                      void* gw_out, void* ws, size_t ws_bytes, float* p, float* m, void* p_bf16, float lr,
                      float momentum, int32_t phase, vp_stream_t stream) {
  VP_REQUIRE(p && m, VP_EVALIDATION, "conv_wgrad_sgd: parameter and momentum buffers required");
  VP_REQUIRE(phase >= 0 && phase <= 2, VP_EVALIDATION, "conv_wgrad_sgd: phase must be 0, 1 or 2");
  VP_REQUIRE(x_dtype != VP_F64 && g_dtype != VP_F64, VP_EVALIDATION, "conv_wgrad_sgd: fp32 parameters only");
  return conv_wgrad_impl(x, x_dtype, cin, g, g_dtype, cout, K, pin, pout, pptr, cap_pairs, gw_out, ws, ws_bytes,
                         SgdFuse{p, m, (__nv_bfloat16*)p_bf16, lr, momentum}, phase, (cudaStream_t)stream);
}

static int conv_wgrad_impl(const void* x, int32_t x_dtype, int64_t cin, const void* g, int32_t g_dtype, int64_t cout,
                           int32_t K, const int32_t* pin, const int32_t* pout, const int32_t* pptr, int64_t cap_pairs,
                           void* gw_out, void* ws, size_t ws_bytes, const SgdFuse& sgd, int phase, cudaStream_t st,
                           bool side) {
  VP_REQUIRE(K >= 1 && K <= VP_MAX_OFFSETS, VP_EVALIDATION, "kernel offset count out of range");
  VP_REQUIRE(ws && ws_bytes >= vp_conv_wgrad_ws_bytes(cin, cout, K, cap_pairs), VP_EVALIDATION,
             "conv_wgrad: workspace too small");
  if (x_dtype == VP_TF32) x_dtype = VP_F32;  // fp32 storage; the weight gradient is exact fp32
  if (g_dtype == VP_TF32) g_dtype = VP_F32;
  const int chunk = wgrad_chunk(cap_pairs);
  const int max_items = (int)(cap_pairs / chunk + K + 1);
  float* part = (float*)ws;
  float* gw = (float*)gw_out;
  const int64_t total = (int64_t)K * cin * cout;
  int rblocks = (int)std::min<int64_t>(ceil_div(total, 256), grid_cap(8));
  // the training step's reduction + SGD (phase 2) runs beside the critical
  // path: blocks capped (VP_WGRAD_RED_BLOCKS, tuning)
  static const int red_cap = getenv("VP_WGRAD_RED_BLOCKS") ? std::max(1, atoi(getenv("VP_WGRAD_RED_BLOCKS"))) : 0;
  if (phase == 2 && red_cap > 0) rblocks = std::min(rblocks, red_cap);
  if (x_dtype == VP_F64 || g_dtype == VP_F64) {  // the reference's precision: f64 partials, f64 grad_w
    const int dchunk = 2 * std::min(chunk, kWgSimtChunk);
    const int ditems = (int)(cap_pairs / dchunk + K + 1);
    double* dpart = (double*)ws;
    if (phase != 2) ::vp::launch(wgrad_simt_kernel<double>, std::max(1, std::min(ditems, grid_cap(8))), kWgSimtThreads, 0, st, x,
                 x_dtype, (int)cin, g, g_dtype, (int)cout, K, pin, pout, pptr, dchunk, dpart);
    if (phase != 2) VP_CHECK_LAUNCH("conv_wgrad_simt_f64");
    if (phase != 1) ::vp::launch(wgrad_reduce_kernel<double>, rblocks, 256, 0, st, (const double*)dpart, pptr, K, dchunk,
                 (int64_t)cin * cout, (double*)gw_out, (const int*)nullptr, SgdFuse{});
    if (phase != 1) VP_CHECK_LAUNCH("wgrad_reduce_f64");
    return VP_OK;
  }
  if (x_dtype == VP_BF16 && g_dtype == VP_BF16 && tc_width(cin) && tc_width(cout)) {
    // pairs per item: from the static pair capacity, or chosen on the device
    // from the live pair count (bounded by the partials the workspace holds)
    // default: the capacity rule — in the concurrent training step fewer,
    // longer items leave more SMs to the critical path (C3: 1.309 vs 1.319
    // ms/step), although the live-count chunk runs the 128-wide layers
    // standalone 25% faster (VP_WGRAD_DEVICE_CHUNK=1)
    static const bool static_chunk = !(getenv("VP_WGRAD_DEVICE_CHUNK") && atoi(getenv("VP_WGRAD_DEVICE_CHUNK")) == 1);
    const int64_t ws_items = (int64_t)((ws_bytes - kWgHeader) / ((size_t)cin * cout * 4));
    int* chunk_dev = (int*)((char*)ws + ws_bytes - kWgHeader);
    // floor: gathered bytes per item >= f/2 x its C_out x C_in fp32 partial (VP_WGRAD_MIN_F, default 1)
    static const int min_f = getenv("VP_WGRAD_MIN_F") ? std::max(0, atoi(getenv("VP_WGRAD_MIN_F"))) : 1;
    const int chunk_min = (int)std::min<int64_t>(2 * cin * cout / (cin + cout) * min_f, kWgMaxChunk);
    static const int side_sms = getenv("VP_WGRAD_SMS") ? std::max(1, atoi(getenv("VP_WGRAD_SMS"))) : kWgSms;
    WgParams p{(const bf16*)x, (const bf16*)g, K, pin, pout, pptr, static_chunk ? chunk : 0, part,
               (int)std::min<int64_t>(ws_items, 1 << 30), chunk_dev, chunk_min,
               ((phase != 0 || side) && cap_pairs <= kWgSideCapPairs) ? side_sms : kNumSMs};
    const int grid_items = static_chunk ? max_items : (int)std::min<int64_t>(ws_items, 1 << 30);
    if (phase != 2) {
      int rc = wg_tc(cin, cout, p, grid_items, st);
      if (rc != VP_OK) return rc;
    }
    if (phase != 1) ::vp::launch(wgrad_reduce_kernel<float>, rblocks, 256, 0, st, (const float*)part, pptr, K, chunk,
                 (int64_t)cin * cout, gw, static_chunk ? (const int*)nullptr : (const int*)chunk_dev, sgd);
    if (phase != 1) VP_CHECK_LAUNCH("wgrad_reduce");
    return VP_OK;
  }
  if (cin == 1 && (cout == 16 || cout == 32 || cout == 64) && x_dtype == VP_BF16 && g_dtype == VP_BF16) {
    // kWgStemChunk >= kWgSimtChunk: fewer items than the workspace is sized for
    const int items = (int)(cap_pairs / kWgStemChunk + K + 1);
    const int grid = std::max(1, std::min(items, grid_cap(8)));
    const bf16 *xb = (const bf16*)x, *gb = (const bf16*)g;
    if (phase == 2) {
    } else if (cout == 16)
      ::vp::launch(wgrad_stem_kernel<16>, grid, kWgStemThreads, 0, st, xb, gb, K, pin, pout, pptr, part);
    else if (cout == 32)
      ::vp::launch(wgrad_stem_kernel<32>, grid, kWgStemThreads, 0, st, xb, gb, K, pin, pout, pptr, part);
    else
      ::vp::launch(wgrad_stem_kernel<64>, grid, kWgStemThreads, 0, st, xb, gb, K, pin, pout, pptr, part);
    if (phase != 2) VP_CHECK_LAUNCH("conv_wgrad_stem");
    if (phase != 1) ::vp::launch(wgrad_reduce_kernel<float>, rblocks, 256, 0, st, (const float*)part, pptr, K, kWgStemChunk,
                 (int64_t)cin * cout, gw, (const int*)nullptr, sgd);
    if (phase != 1) VP_CHECK_LAUNCH("wgrad_reduce");
    return VP_OK;
  }
  const int schunk = std::min(chunk, kWgSimtChunk);
  const int sitems = (int)(cap_pairs / schunk + K + 1);
  const int grid = std::max(1, std::min(sitems, grid_cap(8)));
  if (phase != 2) ::vp::launch(wgrad_simt_kernel<float>, grid, kWgSimtThreads, 0, st, x, x_dtype, (int)cin, g, g_dtype, (int)cout, K,
               pin, pout, pptr, schunk, part);
  if (phase != 2) VP_CHECK_LAUNCH("conv_wgrad_simt");
  if (phase != 1) ::vp::launch(wgrad_reduce_kernel<float>, rblocks, 256, 0, st, (const float*)part, pptr, K, schunk,
               (int64_t)cin * cout, gw, (const int*)nullptr, sgd);
  if (phase != 1) VP_CHECK_LAUNCH("wgrad_reduce");
  return VP_OK;
}

int vp_cast(const void* src, int32_t sd, void* dst, int32_t dd, int64_t n, vp_stream_t stream) {
  if (n <= 0) return VP_OK;
  ::vp::launch(cast_kernel, (int)std::min<int64_t>(ceil_div(n, 256), grid_cap(8)), 256, 0, (cudaStream_t)stream, src, sd, dst,
                                                                                                      dd, n);
  VP_CHECK_LAUNCH("cast");
  return VP_OK;
}

}  // extern "C"
