// Warp-specialized output-stationary implicit GEMM for the sparse conv
// forward (conv.py:186-208) and dgrad (conv.py:240) on sm_100a tcgen05.
//
//   out[r, n] = sum_{k active} sum_{c} A_k[r, c] * B_k[n, c]
//   forward: A_k[r] = x[table[r, k]] (C_in wide), B_k = W_k        (K-major)
//   dgrad  : A_k[r] = g[table[r, k]] (C_out wide), B_k = W_k^T     (W read
//            directly as an MN-major operand: no transposed copy)
//
// CTA = 9 warps: warps 0-3 produce (cp.async gathers of 128 neighbour rows +
// the weight slice into a 128B-swizzled stage ring, completion signalled per
// stage on an mbarrier after a proxy fence), warp 8 issues tcgen05.mma from
// one elected lane into a double-buffered TMEM accumulator, warps 4-7 drain
// TMEM (tcgen05.ld) and store each output row exactly once.  Work items are
// (128-row tile, split) pairs; when the tile count cannot fill the grid the
// active offsets of a tile are split across CTAs (fp32 partials, reduced in a
// fixed order afterwards) -> deterministic with no atomics on the output.
// C_in = 32 packs two offsets into one 64-wide K stage.
#pragma once
#include "common.cuh"
#include "tc.cuh"

namespace vp {

using bf16 = __nv_bfloat16;

struct FwdParams {
  const bf16* x;
  const bf16* w;
  int K;
  const int32_t* table;
  int flip;
  const int32_t* n_out_dev;
  int64_t cap_out;
  void* y;
  int y_dtype;
  float* part;    // split-K partials (grid * 128 * ND floats), may be null if max_split == 1
  int max_split;  // >= 1
};

constexpr int kTcProd = 128, kTcEpi = 128, kTcThreads = kTcProd + kTcEpi + 32;
constexpr int kNbrSmemK = 32;  // neighbour table cached in smem when K <= 32
constexpr int kTcMaskWords = (VP_MAX_OFFSETS + 31) / 32;

template <int KD, int ND, bool BMN>
struct FwdTC {
  static constexpr bool PAIR = (KD == 32);
  static constexpr int NCH = PAIR ? 1 : KD / 64;
  static constexpr int A_BYTES = 128 * 128;
  static constexpr int NPAD = (BMN && ND < 64) ? 64 : ND;
  static constexpr int B_BYTES = NPAD * 128;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES_RAW = (180 * 1024) / STAGE;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : (STAGES_RAW < 3 ? 3 : STAGES_RAW);
  static constexpr int ACC = (2 * ND <= 512) ? 2 : 1;
  static constexpr int COLS = ACC * ND;
  static constexpr int TMEM_COLS = COLS <= 32 ? 32 : COLS <= 64 ? 64 : COLS <= 128 ? 128 : COLS <= 256 ? 256 : 512;
  static constexpr uint32_t IDESC = tc::idesc_bf16(128, ND, 0, BMN ? 1 : 0);
  static constexpr int BOOK = 4096 + 128 * (kNbrSmemK + 1) * 4;
  static constexpr int SMEM = STAGES * STAGE + 1024 + BOOK;
};

__device__ __forceinline__ int split_count(int ntiles, int grid, int max_split) {
  if (ntiles <= 0 || max_split <= 1 || ntiles * 2 > grid) return 1;
  int s = grid / ntiles;
  return s > max_split ? max_split : s;
}

template <int KD, int ND, bool BMN>
__global__ void __launch_bounds__(kTcThreads, 1) conv_tc_kernel(const __grid_constant__ FwdParams p) {
  using C = FwdTC<KD, ND, BMN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* book = smem + C::STAGES * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(book);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + C::ACC;
  uint64_t* ifull = tempty + C::ACC;
  uint64_t* iempty = ifull + 2;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(iempty + 2);
  int* s_info = reinterpret_cast<int*>(book + 512);          // [2] units per work item (for MMA)
  int* s_work = s_info + 4;                                  // u0, n_units, n_act (producers)
  uint32_t* s_mask = reinterpret_cast<uint32_t*>(book + 640);
  int16_t* s_act = reinterpret_cast<int16_t*>(book + 1024);  // <= 343 entries
  int32_t* s_nbr = reinterpret_cast<int32_t*>(book + 4096);  // [128][kNbrSmemK+1]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = p.K;
  const int n_out = load_count(p.n_out_dev, p.cap_out);
  const int ntiles = (n_out + 127) / 128;
  const int S = split_count(ntiles, gridDim.x, p.max_split);
  const int total = ntiles * S;
  if ((int)blockIdx.x >= total) return;

  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      tc::mbar_init(&full[s], kTcProd);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < C::ACC; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], kTcEpi);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&ifull[i], 1);
      tc::mbar_init(&iempty[i], 1);
    }
    tc::fence_mbar_init();
  }
  if (warp == 8) tc::tmem_alloc(s_tmem, C::TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const uint32_t sbase = tc::smem_u32(smem);
  const bool nbr_smem = K <= kNbrSmemK;

  if (warp < 4) {
    // ============================ producers ============================
    uint32_t g = 0;
    int ii = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x, ++ii) {
      const int tile = w / S, split = w - (w / S) * S;
      const int64_t u = (int64_t)tile * 128 + tid;
      const bool valid = u < n_out;
      const int32_t* trow = p.table + u * K;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tid < kTcMaskWords) s_mask[tid] = 0;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      for (int kb = 0; kb < K; kb += 32) {
        uint32_t bits = 0;
        const int kend = min(32, K - kb);
        for (int j = 0; j < kend; ++j) {
          const int k = kb + j;
          const int v = valid ? __ldg(trow + (p.flip ? K - 1 - k : k)) : -1;
          if (nbr_smem) s_nbr[tid * (kNbrSmemK + 1) + k] = v;
          if (v >= 0) bits |= 1u << j;
        }
        bits = __reduce_or_sync(0xffffffffu, bits);
        if (lane == 0 && bits) atomicOr(&s_mask[kb >> 5], bits);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tid == 0) {
        int na = 0;
        for (int k = 0; k < K; ++k)
          if (s_mask[k >> 5] & (1u << (k & 31))) s_act[na++] = (int16_t)k;
        const int nu = C::PAIR ? (na + 1) / 2 : na * C::NCH;
        const int u0 = (int)((int64_t)nu * split / S), u1 = (int)((int64_t)nu * (split + 1) / S);
        s_work[0] = u0;
        s_work[1] = u1 - u0;
        s_work[2] = na;
        const int slot = ii & 1;
        if (ii >= 2) tc::mbar_wait(&iempty[slot], ((ii >> 1) - 1) & 1);
        s_info[slot] = max(u1 - u0, 1);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&ifull[slot])) : "memory");
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const int u0 = s_work[0], nun = s_work[1], na = s_work[2];
      const int neff = nun > 0 ? nun : 1;
      for (int j = 0; j < neff; ++j, ++g) {
        const int stage = g % C::STAGES;
        if (g >= (uint32_t)C::STAGES) tc::mbar_wait(&empty[stage], ((g / C::STAGES) - 1) & 1);
        const uint32_t a_s = sbase + stage * C::STAGE;
        const uint32_t b_s = a_s + C::A_BYTES;
        const int unit = u0 + j;
        // ---- which offsets / K slice this unit covers
        int ka, kb = -1, cs = 0;
        if (nun == 0) {
          ka = -1;  // zero unit: A = 0, B = any finite weights
        } else if (C::PAIR) {
          ka = s_act[2 * unit];
          kb = (2 * unit + 1 < na) ? s_act[2 * unit + 1] : -1;
        } else {
          ka = s_act[unit / C::NCH];
          cs = unit % C::NCH;
        }
        // ---- A: row tid, 8 x 16 B chunks
        auto nb_of = [&](int k) -> int {
          if (k < 0 || !valid) return -1;
          const int col = p.flip ? K - 1 - k : k;
          return nbr_smem ? s_nbr[tid * (kNbrSmemK + 1) + k] : __ldg(trow + col);
        };
        if (C::PAIR) {
          const int va = nb_of(ka), vb = nb_of(kb);
          const bf16* sa = p.x + (int64_t)(va >= 0 ? va : 0) * KD;
          const bf16* sb = p.x + (int64_t)(vb >= 0 ? vb : 0) * KD;
#pragma unroll
          for (int q = 0; q < 4; ++q) tc::cp_async16(a_s + tid * 128 + ((q ^ (tid & 7)) << 4), sa + q * 8, va >= 0 ? 16 : 0);
#pragma unroll
          for (int q = 4; q < 8; ++q)
            tc::cp_async16(a_s + tid * 128 + ((q ^ (tid & 7)) << 4), sb + (q - 4) * 8, vb >= 0 ? 16 : 0);
        } else {
          const int va = nb_of(ka);
          const bf16* sa = p.x + (int64_t)(va >= 0 ? va : 0) * KD + cs * 64;
#pragma unroll
          for (int q = 0; q < 8; ++q) tc::cp_async16(a_s + tid * 128 + ((q ^ (tid & 7)) << 4), sa + q * 8, va >= 0 ? 16 : 0);
        }
        // ---- B
        const int kA = ka >= 0 ? ka : 0;
        const int kB = kb >= 0 ? kb : kA;
        if (!BMN) {  // B[n][kk] = W[k][n][slice]  (K-major rows of W)
          constexpr int CH = ND * 8;
#pragma unroll
          for (int e = tid; e < CH; e += kTcProd) {
            const int n = e >> 3, q = e & 7;
            const bf16* src;
            if (C::PAIR) {
              const int k = q < 4 ? kA : kB;
              src = p.w + ((int64_t)k * ND + n) * KD + (q & 3) * 8;
            } else {
              src = p.w + ((int64_t)kA * ND + n) * KD + cs * 64 + q * 8;
            }
            tc::cp_async16(b_s + n * 128 + ((q ^ (n & 7)) << 4), src, 16);
          }
        } else {  // B(n, kk) = W[k][kk][n]: row kk of W_k is N-contiguous (MN-major)
          constexpr int NCHK = ND / 8;
          constexpr int CH = 64 * NCHK;
#pragma unroll
          for (int e = tid; e < CH; e += kTcProd) {
            const int kk = e / NCHK, j = e - (e / NCHK) * NCHK;
            const bf16* src;
            if (C::PAIR) {
              const int k = kk < 32 ? kA : kB;
              src = p.w + ((int64_t)k * KD + (kk & 31)) * ND + j * 8;
            } else {
              src = p.w + ((int64_t)kA * KD + cs * 64 + kk) * ND + j * 8;
            }
            const uint32_t off = (uint32_t)((j >> 3) * 8192 + (kk >> 3) * 1024 + (kk & 7) * 128 + (((j & 7) ^ (kk & 7)) << 4));
            tc::cp_async16(b_s + off, src, 16);
          }
        }
        // the stage's full barrier completes when every producer's copies have landed
        tc::cp_async_arrive_noinc(&full[stage]);
      }
    }
    tc::cp_async_wait<0>();
  } else if (warp < 8) {
    // ============================ epilogue ============================
    const int ep = warp - 4;
    int ii = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x, ++ii) {
      const int tile = w / S, split = w - (w / S) * S;
      const int a = ii % C::ACC;
      tc::mbar_wait(&tfull[a], (ii / C::ACC) & 1);
      tc::tc_fence_after();
      const int lrow = ep * 32 + lane;
      const int64_t row = (int64_t)tile * 128 + lrow;
#pragma unroll 1
      for (int c0 = 0; c0 < ND; c0 += 32) {
        float v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(ep * 32) << 16) + a * ND + c0, v);
        if (row < n_out) {
          if (S > 1) {
            float4* dst = reinterpret_cast<float4*>(p.part + (((int64_t)split * ntiles + tile) * 128 + lrow) * ND + c0);
#pragma unroll
            for (int q = 0; q < 8; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          } else if (p.y_dtype == VP_BF16) {
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(p.y) + row * ND + c0);
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
            float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.y) + row * ND + c0);
#pragma unroll
            for (int q = 0; q < 8; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&tempty[a]);
    }
  } else if (lane == 0) {
    // ============================ MMA issuer ============================
    uint32_t g = 0;
    int ii = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x, ++ii) {
      const int slot = ii & 1;
      tc::mbar_wait(&ifull[slot], (ii >> 1) & 1);
      const int neff = s_info[slot];
      tc::mbar_arrive(&iempty[slot]);
      const int a = ii % C::ACC;
      const int use = ii / C::ACC;
      if (use >= 1) tc::mbar_wait(&tempty[a], (use - 1) & 1);
      tc::tc_fence_after();
      const uint32_t d = tmem + a * ND;
      for (int j = 0; j < neff; ++j, ++g) {
        const int stage = g % C::STAGES;
        tc::mbar_wait(&full[stage], (g / C::STAGES) & 1);
        tc::tc_fence_after();
        const uint32_t a_s = sbase + stage * C::STAGE;
        const uint32_t b_s = a_s + C::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ad = tc::smem_desc(a_s + kk * 32, 16, 1024, tc::kSwizzle128);
          const uint64_t bd = BMN ? tc::smem_desc(b_s + kk * 2048, 8192, 1024, tc::kSwizzle128)
                                  : tc::smem_desc(b_s + kk * 32, 16, 1024, tc::kSwizzle128);
          tc::mma_bf16(d, ad, bd, C::IDESC, (j > 0 || kk > 0) ? 1u : 0u);
        }
        tc::mma_commit(&empty[stage]);
      }
      tc::mma_commit(&tfull[a]);
    }
  }
  __syncthreads();
  if (warp == 8) tc::tmem_dealloc(tmem, C::TMEM_COLS);
}

// out[r, n] = sum over splits of the fp32 partials, in split order.
__global__ void split_reduce_kernel(const float* __restrict__ part, const int32_t* n_out_dev, int64_t cap_out, int ND,
                                    int grid, int max_split, void* __restrict__ y, int y_dtype) {
  const int n_out = load_count(n_out_dev, cap_out);
  const int ntiles = (n_out + 127) / 128;
  const int S = split_count(ntiles, grid, max_split);
  if (S <= 1) return;
  const int64_t total = (int64_t)n_out * ND / 4;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t idx = e * 4;
    const int64_t r = idx / ND;
    const int n = (int)(idx - r * ND);
    const int tile = (int)(r >> 7), lr = (int)(r & 127);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < S; ++s) {
      const float4 v = *reinterpret_cast<const float4*>(part + (((int64_t)s * ntiles + tile) * 128 + lr) * ND + n);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    if (y_dtype == VP_BF16) {
      __nv_bfloat162* d = reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<bf16*>(y) + idx);
      d[0] = __floats2bfloat162_rn(acc.x, acc.y);
      d[1] = __floats2bfloat162_rn(acc.z, acc.w);
    } else {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + idx) = acc;
    }
  }
}

}  // namespace vp
