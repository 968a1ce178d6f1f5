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

#include "common.cuh"
#include "tc.cuh"

namespace vp {

using bf16 = __nv_bfloat16;
constexpr int kTileM = 128;
constexpr int kConvThreads = 128;
constexpr int kMaskWords = (VP_MAX_OFFSETS + 31) / 32;

template <int CIN, int COUT>
struct FwdCfg {
  static constexpr int KC = CIN >= 64 ? 64 : CIN;  // K elements per stage
  static constexpr int NC = CIN / KC;              // stages per offset
  static constexpr int PITCH = KC * 2;             // bytes per smem row
  static constexpr uint32_t SWZ = PITCH == 128 ? tc::kSwizzle128 : tc::kSwizzle64;
  static constexpr int A_BYTES = kTileM * PITCH;
  static constexpr int B_BYTES = COUT * PITCH;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (4 * STAGE_BYTES <= 200 * 1024) ? 4 : 3;
  static constexpr int TMEM_COLS = COUT < 32 ? 32 : COUT;
  static constexpr uint32_t IDESC = tc::idesc_bf16(kTileM, COUT, 0, 0);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 2048 /*bookkeeping*/;
};

// byte offset of 16B chunk j of row r in a K-major swizzled tile
template <int PITCH>
__device__ __forceinline__ uint32_t kmajor_off(int r, int j) {
  if (PITCH == 128) return (uint32_t)(r * 128 + ((j ^ (r & 7)) << 4));
  return (uint32_t)(r * 64 + ((j ^ ((r >> 1) & 3)) << 4));
}

template <int CIN, int COUT>
__global__ void __launch_bounds__(kConvThreads, 1)
conv_fwd_tc_kernel(const bf16* __restrict__ x, const bf16* __restrict__ w, int K,
                   const int32_t* __restrict__ table, int flip, const int32_t* n_out_dev,
                   int64_t cap_out, void* __restrict__ y, int y_dtype) {
  using C = FwdCfg<CIN, COUT>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* book = smem + C::STAGES * C::STAGE_BYTES;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(book);                 // STAGES
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(book + 64);
  uint32_t* s_mask = reinterpret_cast<uint32_t*>(book + 128);         // kMaskWords
  int16_t* s_active = reinterpret_cast<int16_t*>(book + 192);         // <= 343 entries
  int* s_nact = reinterpret_cast<int*>(book + 192 + 2 * VP_MAX_OFFSETS + 2);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int n_out = load_count(n_out_dev, cap_out);
  const int ntiles = (n_out + kTileM - 1) / kTileM;
  if ((int)blockIdx.x >= ntiles) return;

  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) tc::mbar_init(&mbar[s], 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(s_tmem, C::TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const uint32_t smem_base = tc::smem_u32(smem);

  uint32_t g = 0;  // global pipeline iteration (stage = g % STAGES)
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t u = (int64_t)tile * kTileM + tid;
    const bool valid = u < n_out;
    const int32_t* trow = table + u * K;
    // ---- active offsets of this tile (bit k set iff some row has neighbour k)
    if (tid < kMaskWords) s_mask[tid] = 0;
    __syncthreads();
    if (valid) {
      for (int kb = 0; kb < K; kb += 32) {
        uint32_t bits = 0;
        const int kend = min(32, K - kb);
        for (int j = 0; j < kend; ++j) {
          int k = kb + j;
          int col = flip ? K - 1 - k : k;
          if (__ldg(trow + col) >= 0) bits |= 1u << j;
        }
        if (bits) atomicOr(&s_mask[kb >> 5], bits);
      }
    }
    __syncthreads();
    if (tid == 0) {
      int na = 0;
      for (int k = 0; k < K; ++k)
        if (s_mask[k >> 5] & (1u << (k & 31))) s_active[na++] = (int16_t)k;
      *s_nact = na;
    }
    __syncthreads();
    const int n_iter = *s_nact * C::NC;

    auto load_stage = [&](int it, uint32_t gi) {
      const int stage = gi % C::STAGES;
      const int k = s_active[it / C::NC];
      const int c = it % C::NC;
      const uint32_t a_s = smem_base + stage * C::STAGE_BYTES;
      const uint32_t b_s = a_s + C::A_BYTES;
      // A: row tid <- x[table[u, col]] slice c (zero-fill on miss)
      const int col = flip ? K - 1 - k : k;
      const int v = valid ? __ldg(trow + col) : -1;
      const bf16* src = x + (int64_t)(v >= 0 ? v : 0) * CIN + c * C::KC;
      const int nbytes = v >= 0 ? 16 : 0;
#pragma unroll
      for (int j = 0; j < C::KC / 8; ++j) tc::cp_async16(a_s + kmajor_off<C::PITCH>(tid, j), src + j * 8, nbytes);
      // B: W_k[n, slice c] for n in [0, COUT)
      const bf16* wk = w + ((int64_t)k * COUT) * CIN + c * C::KC;
      constexpr int CHUNKS = COUT * (C::KC / 8);
#pragma unroll
      for (int e = tid; e < CHUNKS; e += kConvThreads) {
        const int n = e / (C::KC / 8), j = e % (C::KC / 8);
        tc::cp_async16(b_s + kmajor_off<C::PITCH>(n, j), wk + (int64_t)n * CIN + j * 8, 16);
      }
    };

    // ---- prologue
    for (int p = 0; p < C::STAGES - 1; ++p) {
      if (p < n_iter) {
        const uint32_t gi = g + p;
        if (gi >= (uint32_t)C::STAGES) tc::mbar_wait(&mbar[gi % C::STAGES], ((gi / C::STAGES) - 1) & 1);
        load_stage(p, gi);
      }
      tc::cp_async_commit();
    }
    // ---- main loop
    for (int it = 0; it < n_iter; ++it) {
      const int nxt = it + C::STAGES - 1;
      if (nxt < n_iter) {
        const uint32_t gi = g + nxt;
        if (gi >= (uint32_t)C::STAGES) tc::mbar_wait(&mbar[gi % C::STAGES], ((gi / C::STAGES) - 1) & 1);
        load_stage(nxt, gi);
      }
      tc::cp_async_commit();
      tc::cp_async_wait<C::STAGES - 1>();
      tc::fence_proxy_async_smem();
      __syncthreads();
      if (tid == 0) {
        tc::tc_fence_after();
        const uint32_t gi = g + it;
        const int stage = gi % C::STAGES;
        const uint32_t a_s = smem_base + stage * C::STAGE_BYTES;
        const uint32_t b_s = a_s + C::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < C::KC / 16; ++kk) {
          const uint64_t ad = tc::smem_desc(a_s + kk * 32, 16, 8 * C::PITCH, C::SWZ);
          const uint64_t bd = tc::smem_desc(b_s + kk * 32, 16, 8 * C::PITCH, C::SWZ);
          tc::mma_bf16(tmem, ad, bd, C::IDESC, (it > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit(&mbar[stage]);
      }
    }
    // ---- epilogue: wait for the last MMA of this tile
    if (n_iter > 0) {
      const uint32_t gl = g + n_iter - 1;
      tc::mbar_wait(&mbar[gl % C::STAGES], (gl / C::STAGES) & 1);
      tc::tc_fence_after();
    }
    g += n_iter;
#pragma unroll 1
    for (int c0 = 0; c0 < COUT; c0 += 32) {
      float v[32];
      tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
      if (n_iter == 0) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
      const int64_t row = (int64_t)tile * kTileM + warp * 32 + lane;
      if (row < n_out) {
        if (y_dtype == VP_BF16) {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(y) + row * COUT + c0);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 pk;
            __nv_bfloat162 h0 = __floats2bfloat162_rn(v[8 * q + 0], v[8 * q + 1]);
            __nv_bfloat162 h1 = __floats2bfloat162_rn(v[8 * q + 2], v[8 * q + 3]);
            __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * q + 4], v[8 * q + 5]);
            __nv_bfloat162 h3 = __floats2bfloat162_rn(v[8 * q + 6], v[8 * q + 7]);
            pk.x = *reinterpret_cast<uint32_t*>(&h0);
            pk.y = *reinterpret_cast<uint32_t*>(&h1);
            pk.z = *reinterpret_cast<uint32_t*>(&h2);
            pk.w = *reinterpret_cast<uint32_t*>(&h3);
            dst[q] = pk;
          }
        } else {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + row * COUT + c0);
#pragma unroll
          for (int q = 0; q < 8; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
      }
    }
    // TMEM reads done before the next tile's first MMA overwrites the accumulator
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, C::TMEM_COLS);
}

// ------------------------------------------------------------------ wgrad (tcgen05)
template <int CIN, int COUT>
struct WgCfg {
  static constexpr int PK = 64;                        // pairs per stage (MMA K)
  static constexpr int MPAD = COUT < 64 ? 64 : COUT;   // A MN extent in smem
  static constexpr int NPAD = CIN < 64 ? 64 : CIN;     // B MN extent in smem
  static constexpr int M = COUT >= 128 ? 128 : 64;     // MMA M
  static constexpr int MT = COUT > 128 ? 2 : 1;        // accumulators (M blocks)
  static constexpr int N = CIN;                        // MMA N
  static constexpr int A_BYTES = MPAD * PK * 2;
  static constexpr int B_BYTES = NPAD * PK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (4 * STAGE_BYTES <= 200 * 1024) ? 4 : (3 * STAGE_BYTES <= 200 * 1024 ? 3 : 2);
  static constexpr int COLS = MT * N;
  static constexpr int TMEM_COLS = COLS <= 32 ? 32 : COLS <= 64 ? 64 : COLS <= 128 ? 128 : COLS <= 256 ? 256 : 512;
  static constexpr uint32_t IDESC = tc::idesc_bf16(M, N, 1, 1);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 1024;
  static constexpr int LBO = 8 * 1024;  // stride between 64-wide MN blocks (PK=64 -> 8 k-groups)
  static constexpr int SBO = 1024;      // stride between 8-row k groups
};

// byte offset of element chunk (mn/8) for pair-row kk in an MN-major SW128 tile
__device__ __forceinline__ uint32_t mnmajor_off(int mn_chunk, int kk) {
  const int blk = mn_chunk >> 3, j = mn_chunk & 7;
  return (uint32_t)(blk * 8192 + (kk >> 3) * 1024 + (kk & 7) * 128 + ((j ^ (kk & 7)) << 4));
}

template <int CIN, int COUT>
__global__ void __launch_bounds__(kConvThreads, 1)
conv_wgrad_tc_kernel(const bf16* __restrict__ x, const bf16* __restrict__ gy, int K,
                     const int32_t* __restrict__ pin, const int32_t* __restrict__ pout,
                     const int32_t* __restrict__ pptr, int chunk, float* __restrict__ part) {
  using C = WgCfg<CIN, COUT>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* book = smem + C::STAGES * C::STAGE_BYTES;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(book);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(book + 64);
  int* s_pref = reinterpret_cast<int*>(book + 128);  // K+1 item prefix (K <= 125 here)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    int acc = 0;
    for (int k = 0; k < K; ++k) {
      s_pref[k] = acc;
      int p = pptr[k + 1] - pptr[k];
      acc += (p + chunk - 1) / chunk;
    }
    s_pref[K] = acc;
    for (int s = 0; s < C::STAGES; ++s) tc::mbar_init(&mbar[s], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  const int n_items = s_pref[K];
  if ((int)blockIdx.x >= n_items) return;
  if (warp == 0) tc::tmem_alloc(s_tmem, C::TMEM_COLS);
  const uint32_t smem_base = tc::smem_u32(smem);
  // zero padding regions once (never written by loads)
  if (COUT < 64 || CIN < 64) {
    for (int s = 0; s < C::STAGES; ++s) {
      uint4* p = reinterpret_cast<uint4*>(smem + s * C::STAGE_BYTES);
      for (int i = tid; i < C::STAGE_BYTES / 16; i += kConvThreads) p[i] = make_uint4(0, 0, 0, 0);
    }
    tc::fence_proxy_async_smem();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *s_tmem;

  uint32_t g = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    int k = 0;
    while (s_pref[k + 1] <= item) ++k;
    const int p0 = pptr[k] + (item - s_pref[k]) * chunk;
    const int p1 = min(pptr[k + 1], p0 + chunk);
    const int n_iter = (p1 - p0 + C::PK - 1) / C::PK;

    auto load_stage = [&](int it, uint32_t gi) {
      const int stage = gi % C::STAGES;
      const uint32_t a_s = smem_base + stage * C::STAGE_BYTES;
      const uint32_t b_s = a_s + C::A_BYTES;
      const int q0 = p0 + it * C::PK;
      constexpr int CA = COUT / 8, CB = CIN / 8;
#pragma unroll
      for (int e = tid; e < C::PK * CA; e += kConvThreads) {
        const int kk = e / CA, j = e % CA;
        const int q = q0 + kk;
        const bool ok = q < p1;
        const int uo = ok ? __ldg(pout + q) : 0;
        tc::cp_async16(a_s + mnmajor_off(j, kk), gy + (int64_t)uo * COUT + j * 8, ok ? 16 : 0);
      }
#pragma unroll
      for (int e = tid; e < C::PK * CB; e += kConvThreads) {
        const int kk = e / CB, j = e % CB;
        const int q = q0 + kk;
        const bool ok = q < p1;
        const int vi = ok ? __ldg(pin + q) : 0;
        tc::cp_async16(b_s + mnmajor_off(j, kk), x + (int64_t)vi * CIN + j * 8, ok ? 16 : 0);
      }
    };

    for (int p = 0; p < C::STAGES - 1; ++p) {
      if (p < n_iter) {
        const uint32_t gi = g + p;
        if (gi >= (uint32_t)C::STAGES) tc::mbar_wait(&mbar[gi % C::STAGES], ((gi / C::STAGES) - 1) & 1);
        load_stage(p, gi);
      }
      tc::cp_async_commit();
    }
    for (int it = 0; it < n_iter; ++it) {
      const int nxt = it + C::STAGES - 1;
      if (nxt < n_iter) {
        const uint32_t gi = g + nxt;
        if (gi >= (uint32_t)C::STAGES) tc::mbar_wait(&mbar[gi % C::STAGES], ((gi / C::STAGES) - 1) & 1);
        load_stage(nxt, gi);
      }
      tc::cp_async_commit();
      tc::cp_async_wait<C::STAGES - 1>();
      tc::fence_proxy_async_smem();
      __syncthreads();
      if (tid == 0) {
        tc::tc_fence_after();
        const uint32_t gi = g + it;
        const int stage = gi % C::STAGES;
        const uint32_t a_s = smem_base + stage * C::STAGE_BYTES;
        const uint32_t b_s = a_s + C::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < C::PK / 16; ++kk) {
          const uint64_t bd = tc::smem_desc(b_s + kk * 2048, C::LBO, C::SBO, tc::kSwizzle128);
#pragma unroll
          for (int mt = 0; mt < C::MT; ++mt) {
            const uint64_t ad = tc::smem_desc(a_s + mt * 2 * C::LBO + kk * 2048, C::LBO, C::SBO, tc::kSwizzle128);
            tc::mma_bf16(tmem + mt * C::N, ad, bd, C::IDESC, (it > 0 || kk > 0) ? 1u : 0u);
          }
        }
        tc::mma_commit(&mbar[stage]);
      }
    }
    if (n_iter > 0) {
      const uint32_t gl = g + n_iter - 1;
      tc::mbar_wait(&mbar[gl % C::STAGES], (gl / C::STAGES) & 1);
      tc::tc_fence_after();
    }
    g += n_iter;
    float* dst = part + (int64_t)item * COUT * CIN;
#pragma unroll 1
    for (int mt = 0; mt < C::MT; ++mt) {
#pragma unroll 1
      for (int c0 = 0; c0 < CIN; c0 += 32) {
        float v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + mt * C::N + c0, v);
        int m;
        bool ok;
        if (C::M == 128) {
          m = mt * 128 + warp * 32 + lane;
          ok = true;
        } else {  // M=64: row r lives in TMEM lane (r%16) + 32*(r/16)
          m = warp * 16 + lane;
          ok = lane < 16;
        }
        ok = ok && m < COUT;
        if (ok) {
          float4* d = reinterpret_cast<float4*>(dst + (int64_t)m * CIN + c0);
          if (n_iter == 0) {
#pragma unroll
            for (int q = 0; q < 8; ++q) d[q] = make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) d[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          }
        }
      }
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, C::TMEM_COLS);
}

// sum the chunk partials of each offset in chunk order (deterministic)
__global__ void wgrad_reduce_kernel(const float* __restrict__ part, const int32_t* __restrict__ pptr,
                                    int K, int chunk, int64_t per, float* __restrict__ gw) {
  __shared__ int s_pref[VP_MAX_OFFSETS + 1];
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int k = 0; k < K; ++k) {
      s_pref[k] = acc;
      acc += (pptr[k + 1] - pptr[k] + chunk - 1) / chunk;
    }
    s_pref[K] = acc;
  }
  __syncthreads();
  const int64_t total = (int64_t)K * per;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e / per);
    const int64_t o = e - (int64_t)k * per;
    float acc = 0.f;
    for (int it = s_pref[k]; it < s_pref[k + 1]; ++it) acc += part[(int64_t)it * per + o];
    gw[e] = acc;
  }
}

// ------------------------------------------------------------------ SIMT paths
// Generic widths / fp32 features: y[u, co] = sum_k sum_ci W[k, co, ci] x[t[u,k], ci].
// W is addressed as W[k*wk + co*wco + ci*wci] so dgrad passes W^T by strides.
__global__ void conv_fwd_simt_kernel(const void* __restrict__ x, int x_dtype, int cin,
                                     const void* __restrict__ w, int w_dtype, int64_t wk, int64_t wco,
                                     int64_t wci, int cout, int K, const int32_t* __restrict__ table,
                                     int flip, const int32_t* n_out_dev, int64_t cap_out, void* y,
                                     int y_dtype) {
  const int n_out = load_count(n_out_dev, cap_out);
  const int64_t total = (int64_t)n_out * cout;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = e / cout;
    const int co = (int)(e - u * cout);
    float acc = 0.f;
    for (int k = 0; k < K; ++k) {
      const int v = table[u * K + (flip ? K - 1 - k : k)];
      if (v < 0) continue;
      for (int ci = 0; ci < cin; ++ci)
        acc += ldf(w, w_dtype, k * wk + co * wco + ci * wci) * ldf(x, x_dtype, (int64_t)v * cin + ci);
    }
    stf(y, y_dtype, e, acc);
  }
}

// wgrad partials: block per (chunk item); warps stride over the chunk's pairs,
// lanes over output elements; fixed-order cross-warp sum.
constexpr int kWgSimtThreads = 256;
__global__ void __launch_bounds__(kWgSimtThreads)
wgrad_simt_kernel(const void* __restrict__ x, int x_dtype, int cin, const void* __restrict__ gy,
                  int g_dtype, int cout, int K, const int32_t* __restrict__ pin,
                  const int32_t* __restrict__ pout, const int32_t* __restrict__ pptr, int chunk,
                  float* __restrict__ part) {
  __shared__ int s_pref[VP_MAX_OFFSETS + 1];
  __shared__ float s_red[kWgSimtThreads / 32][32];
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int k = 0; k < K; ++k) {
      s_pref[k] = acc;
      acc += (pptr[k + 1] - pptr[k] + chunk - 1) / chunk;
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
    const int p0 = pptr[k] + (item - s_pref[k]) * chunk;
    const int p1 = min(pptr[k + 1], p0 + chunk);
    for (int e0 = 0; e0 < per; e0 += 32) {
      const int e = e0 + lane;
      const int co = e / cin, ci = e - (e / cin) * cin;
      float acc = 0.f;
      if (e < per)
        for (int q = p0 + warp; q < p1; q += kWgSimtThreads / 32)
          acc += ldf(gy, g_dtype, (int64_t)pout[q] * cout + co) * ldf(x, x_dtype, (int64_t)pin[q] * cin + ci);
      s_red[warp][lane] = acc;
      __syncthreads();
      if (warp == 0 && e < per) {
        float s = 0.f;
        for (int w2 = 0; w2 < kWgSimtThreads / 32; ++w2) s += s_red[w2][lane];
        part[(int64_t)item * per + e] = s;
      }
      __syncthreads();
    }
  }
}

__global__ void transpose_w_kernel(const void* __restrict__ w, int w_dtype, int K, int cout, int cin,
                                   bf16* __restrict__ wt) {
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
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    stf(dst, dd, i, ldf(src, sd, i));
}

// ------------------------------------------------------------------ dispatch
static bool tc_width(int64_t c) { return c == 32 || c == 64 || c == 128 || c == 256; }

template <int CIN, int COUT>
static int launch_fwd_tc(const bf16* x, const bf16* w, int K, const int32_t* table, int flip,
                         const int32_t* n_out_dev, int64_t cap_out, void* y, int y_dtype, cudaStream_t st) {
  using C = FwdCfg<CIN, COUT>;
  auto kern = conv_fwd_tc_kernel<CIN, COUT>;
  static int occ = -1;  // immutable per-instantiation occupancy cache
  if (occ < 0) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kConvThreads, C::SMEM);
    occ = std::max(1, std::min(o, 512 / C::TMEM_COLS));
  }
  const int64_t tiles = ceil_div(cap_out, kTileM);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)kNumSMs * occ));
  kern<<<grid, kConvThreads, C::SMEM, st>>>(x, w, K, table, flip, n_out_dev, cap_out, y, y_dtype);
  VP_CHECK_LAUNCH("conv_fwd_tc");
  return VP_OK;
}

template <int CIN>
static int fwd_tc_cout(int64_t cout, const bf16* x, const bf16* w, int K, const int32_t* table, int flip,
                       const int32_t* n, int64_t cap, void* y, int yd, cudaStream_t st) {
  switch (cout) {
    case 32: return launch_fwd_tc<CIN, 32>(x, w, K, table, flip, n, cap, y, yd, st);
    case 64: return launch_fwd_tc<CIN, 64>(x, w, K, table, flip, n, cap, y, yd, st);
    case 128: return launch_fwd_tc<CIN, 128>(x, w, K, table, flip, n, cap, y, yd, st);
    case 256: return launch_fwd_tc<CIN, 256>(x, w, K, table, flip, n, cap, y, yd, st);
  }
  return VP_EINTERNAL;
}

static int fwd_tc(int64_t cin, int64_t cout, const bf16* x, const bf16* w, int K, const int32_t* table,
                  int flip, const int32_t* n, int64_t cap, void* y, int yd, cudaStream_t st) {
  switch (cin) {
    case 32: return fwd_tc_cout<32>(cout, x, w, K, table, flip, n, cap, y, yd, st);
    case 64: return fwd_tc_cout<64>(cout, x, w, K, table, flip, n, cap, y, yd, st);
    case 128: return fwd_tc_cout<128>(cout, x, w, K, table, flip, n, cap, y, yd, st);
    case 256: return fwd_tc_cout<256>(cout, x, w, K, table, flip, n, cap, y, yd, st);
  }
  return VP_EINTERNAL;
}

template <int CIN, int COUT>
static int launch_wg_tc(const bf16* x, const bf16* gy, int K, const int32_t* pin, const int32_t* pout,
                        const int32_t* pptr, int chunk, int max_items, float* part, cudaStream_t st) {
  using C = WgCfg<CIN, COUT>;
  auto kern = conv_wgrad_tc_kernel<CIN, COUT>;
  static int occ = -1;
  if (occ < 0) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kConvThreads, C::SMEM);
    occ = std::max(1, std::min(o, 512 / C::TMEM_COLS));
  }
  const int grid = std::max(1, std::min(max_items, kNumSMs * occ));
  kern<<<grid, kConvThreads, C::SMEM, st>>>(x, gy, K, pin, pout, pptr, chunk, part);
  VP_CHECK_LAUNCH("conv_wgrad_tc");
  return VP_OK;
}

template <int CIN>
static int wg_tc_cout(int64_t cout, const bf16* x, const bf16* gy, int K, const int32_t* pin,
                      const int32_t* pout, const int32_t* pptr, int chunk, int mi, float* part, cudaStream_t st) {
  switch (cout) {
    case 32: return launch_wg_tc<CIN, 32>(x, gy, K, pin, pout, pptr, chunk, mi, part, st);
    case 64: return launch_wg_tc<CIN, 64>(x, gy, K, pin, pout, pptr, chunk, mi, part, st);
    case 128: return launch_wg_tc<CIN, 128>(x, gy, K, pin, pout, pptr, chunk, mi, part, st);
    case 256: return launch_wg_tc<CIN, 256>(x, gy, K, pin, pout, pptr, chunk, mi, part, st);
  }
  return VP_EINTERNAL;
}

static int wg_tc(int64_t cin, int64_t cout, const bf16* x, const bf16* gy, int K, const int32_t* pin,
                 const int32_t* pout, const int32_t* pptr, int chunk, int mi, float* part, cudaStream_t st) {
  switch (cin) {
    case 32: return wg_tc_cout<32>(cout, x, gy, K, pin, pout, pptr, chunk, mi, part, st);
    case 64: return wg_tc_cout<64>(cout, x, gy, K, pin, pout, pptr, chunk, mi, part, st);
    case 128: return wg_tc_cout<128>(cout, x, gy, K, pin, pout, pptr, chunk, mi, part, st);
    case 256: return wg_tc_cout<256>(cout, x, gy, K, pin, pout, pptr, chunk, mi, part, st);
  }
  return VP_EINTERNAL;
}

static int wgrad_chunk(int64_t cin, int64_t cout) {
  (void)cin;
  (void)cout;
  return 1024;  // pairs per partial (fixed: results independent of timing)
}

}  // namespace vp

using namespace vp;

extern "C" {

size_t vp_conv_fwd_ws_bytes(int64_t cin, int64_t cout, int32_t K) {
  return align_up((size_t)K * cin * cout * 2, 256);
}

int vp_conv_fwd(const void* x, int32_t x_dtype, int64_t cin, const void* w, int32_t w_dtype, int64_t cout,
                int32_t K, const int32_t* table, int32_t flip, const int32_t* n_out_dev, int64_t cap_out,
                void* y, int32_t y_dtype, void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(K >= 1 && K <= VP_MAX_OFFSETS, VP_EVALIDATION, "kernel offset count out of range");
  VP_REQUIRE(cin >= 1 && cout >= 1, VP_EVALIDATION, "channel widths must be positive");
  VP_REQUIRE(y_dtype == VP_F32 || y_dtype == VP_BF16, VP_EVALIDATION, "output dtype must be f32 or bf16");
  if (cap_out <= 0) return VP_OK;
  if (x_dtype == VP_BF16 && tc_width(cin) && tc_width(cout)) {
    const bf16* wb = (const bf16*)w;
    if (w_dtype != VP_BF16) {
      VP_REQUIRE(ws && ws_bytes >= vp_conv_fwd_ws_bytes(cin, cout, K), VP_EVALIDATION,
                 "conv_fwd: workspace too small for weight conversion");
      int64_t cnt = (int64_t)K * cin * cout;
      cast_kernel<<<(int)std::min<int64_t>(ceil_div(cnt, 256), 1184), 256, 0, st>>>(w, w_dtype, ws, VP_BF16, cnt);
      VP_CHECK_LAUNCH("conv_fwd: cast w");
      wb = (const bf16*)ws;
    }
    return fwd_tc(cin, cout, (const bf16*)x, wb, K, table, flip, n_out_dev, cap_out, y, y_dtype, st);
  }
  const int64_t total = cap_out * cout;
  int blocks = (int)std::min<int64_t>(ceil_div(total, 256), kNumSMs * 16);
  conv_fwd_simt_kernel<<<blocks, 256, 0, st>>>(x, x_dtype, (int)cin, w, w_dtype, cout * cin, cin, 1, (int)cout,
                                                K, table, flip, n_out_dev, cap_out, y, y_dtype);
  VP_CHECK_LAUNCH("conv_fwd_simt");
  return VP_OK;
}

size_t vp_conv_dgrad_ws_bytes(int64_t cin, int64_t cout, int32_t K) {
  return align_up((size_t)K * cin * cout * 2, 256);
}

int vp_conv_dgrad(const void* g, int32_t g_dtype, int64_t cout, const void* w, int32_t w_dtype, int64_t cin,
                  int32_t K, const int32_t* table, int32_t flip, const int32_t* n_in_dev, int64_t cap_in,
                  void* gi, int32_t gi_dtype, void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(K >= 1 && K <= VP_MAX_OFFSETS, VP_EVALIDATION, "kernel offset count out of range");
  if (cap_in <= 0) return VP_OK;
  if (g_dtype == VP_BF16 && tc_width(cin) && tc_width(cout)) {
    VP_REQUIRE(ws && ws_bytes >= vp_conv_dgrad_ws_bytes(cin, cout, K), VP_EVALIDATION,
               "conv_dgrad: workspace too small");
    int64_t cnt = (int64_t)K * cin * cout;
    transpose_w_kernel<<<(int)std::min<int64_t>(ceil_div(cnt, 256), 1184), 256, 0, st>>>(w, w_dtype, K, (int)cout,
                                                                                       (int)cin, (bf16*)ws);
    VP_CHECK_LAUNCH("conv_dgrad: transpose w");
    // grad_in = sum_k (W_k^T) g[table] : a forward conv with C_in'=cout, C_out'=cin
    return fwd_tc(cout, cin, (const bf16*)g, (const bf16*)ws, K, table, flip, n_in_dev, cap_in, gi, gi_dtype, st);
  }
  const int64_t total = cap_in * cin;
  int blocks = (int)std::min<int64_t>(ceil_div(total, 256), kNumSMs * 16);
  // W^T[k, ci, co] = W[k, co, ci]: strides (k: cout*cin, "co"=ci: 1, "ci"=co: cin)
  conv_fwd_simt_kernel<<<blocks, 256, 0, st>>>(g, g_dtype, (int)cout, w, w_dtype, cout * cin, 1, cin, (int)cin,
                                                K, table, flip, n_in_dev, cap_in, gi, gi_dtype);
  VP_CHECK_LAUNCH("conv_dgrad_simt");
  return VP_OK;
}

size_t vp_conv_wgrad_ws_bytes(int64_t cin, int64_t cout, int32_t K, int64_t cap_pairs) {
  const int chunk = wgrad_chunk(cin, cout);
  const int64_t items = cap_pairs / chunk + K + 1;
  return align_up((size_t)items * cin * cout * 4, 256);
}

int vp_conv_wgrad(const void* x, int32_t x_dtype, int64_t cin, const void* g, int32_t g_dtype, int64_t cout,
                  int32_t K, const int32_t* pin, const int32_t* pout, const int32_t* pptr, int64_t cap_pairs,
                  float* gw, void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(K >= 1 && K <= VP_MAX_OFFSETS, VP_EVALIDATION, "kernel offset count out of range");
  VP_REQUIRE(ws && ws_bytes >= vp_conv_wgrad_ws_bytes(cin, cout, K, cap_pairs), VP_EVALIDATION,
             "conv_wgrad: workspace too small");
  const int chunk = wgrad_chunk(cin, cout);
  const int max_items = (int)(cap_pairs / chunk + K + 1);
  float* part = (float*)ws;
  if (x_dtype == VP_BF16 && g_dtype == VP_BF16 && tc_width(cin) && tc_width(cout) && K <= 125) {
    int r = wg_tc(cin, cout, (const bf16*)x, (const bf16*)g, K, pin, pout, pptr, chunk, max_items, part, st);
    if (r) return r;
  } else {
    const int grid = std::max(1, std::min(max_items, kNumSMs * 8));
    wgrad_simt_kernel<<<grid, kWgSimtThreads, 0, st>>>(x, x_dtype, (int)cin, g, g_dtype, (int)cout, K, pin, pout,
                                                       pptr, chunk, part);
    VP_CHECK_LAUNCH("conv_wgrad_simt");
  }
  const int64_t total = (int64_t)K * cin * cout;
  wgrad_reduce_kernel<<<(int)std::min<int64_t>(ceil_div(total, 256), kNumSMs * 8), 256, 0, st>>>(
      part, pptr, K, chunk, cin * cout, gw);
  VP_CHECK_LAUNCH("wgrad_reduce");
  return VP_OK;
}

int vp_cast(const void* src, int32_t sd, void* dst, int32_t dd, int64_t n, vp_stream_t stream) {
  if (n <= 0) return VP_OK;
  cast_kernel<<<(int)std::min<int64_t>(ceil_div(n, 256), kNumSMs * 8), 256, 0, (cudaStream_t)stream>>>(src, sd, dst,
                                                                                                      dd, n);
  VP_CHECK_LAUNCH("cast");
  return VP_OK;
}

}  // extern "C"
