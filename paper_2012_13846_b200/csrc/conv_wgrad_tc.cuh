// Warp-specialized weight gradient (conv.py:241) on sm_100a tcgen05:
//   grad_W_k[m, n] = sum over the pairs (v, u) of offset k of g[u, m] * x[v, n]
// Work items are (offset k, chunk of `chunk` pairs).  Warps 0-3 stage each
// item's pair indices in shared memory and gather 64 pairs per stage with
// cp.async into MN-major 128B-swizzled tiles (g rows -> A: M = C_out,
// x rows -> B: N = C_in; the pair index is the MMA K dimension); warp 8
// issues tcgen05.mma into TMEM; warps 4-7 drain TMEM.  Every chunk writes an fp32 partial and a separate fully parallel kernel
// (wgrad_reduce_kernel) sums each offset's partials in chunk order ->
// deterministic, no atomics.
#pragma once
#include "common.cuh"
#include "conv_fwd_tc.cuh"
#include "tc.cuh"

namespace vp {

constexpr int kWgMaxChunk = 2048;

struct WgParams {
  const __nv_bfloat16* x;
  const __nv_bfloat16* g;
  int K;
  const int32_t* pin;
  const int32_t* pout;
  const int32_t* pptr;
  int chunk;        // pairs per item (multiple of 64, <= kWgMaxChunk); 0 = chosen on the device
  float* part;      // partials, items * C_out * C_in
  int max_items;    // partials the workspace holds (device-chosen chunk)
  int* chunk_out;   // device-chosen chunk, for wgrad_reduce_kernel
  int chunk_min;    // device-chosen chunk floor (keeps C_out x C_in partials small next to the gathers)
  int sms;          // (host) SMs the persistent grid may occupy
};

// Pairs per work item from the LIVE pair count (pptr[K], on the device):
// about one item per CTA so every SM works and the chains stay short, but
// long enough that the partials fit the workspace.  Depends only on the
// pair count and the launch shape -> deterministic.
__device__ __forceinline__ int wg_device_chunk(int total, int K, int grid, int max_items, int chunk_min) {
  // items <= total / c + K (one partial chunk per offset): aim at <= grid
  const int slots = max(grid - K - 1, grid / 2);
  int c = max((total + slots - 1) / slots, chunk_min);
  const int room = max_items - K - 1;
  if (room > 0) c = max(c, (total + room - 1) / room);
  c = (c + 63) / 64 * 64;
  return min(max(c, 64), kWgMaxChunk);
}

// (kTcProd / kTcEpi / kTcThreads from conv_fwd_tc.cuh: warps 0-3 produce,
// 4-7 drain TMEM, 8 issues the MMAs)

// CPS CTAs per SM: the gathers are bound by the producers' cp.async issue
// rate, so two independent CTAs per SM (half the ring each) move more pairs
// per microsecond where two rings of >= 4 stages fit (C_in, C_out <= 128).
template <int CIN, int COUT, int CPS = 1>
struct WgTC {
  static constexpr int PK = 64;
  static constexpr int MPAD = COUT < 64 ? 64 : COUT;
  static constexpr int NPAD = CIN < 64 ? 64 : CIN;
  static constexpr int M = COUT >= 128 ? 128 : 64;
  static constexpr int MT = COUT > 128 ? 2 : 1;
  static constexpr int N = CIN;
  static constexpr int A_BYTES = MPAD * PK * 2;
  static constexpr int B_BYTES = NPAD * PK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int IDX_BYTES = kWgMaxChunk * 8;
  static constexpr int STAGES_RAW = ((CPS == 1 ? 196 : 104) * 1024 - IDX_BYTES) / STAGE;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : (STAGES_RAW < 3 ? 3 : STAGES_RAW);
  static constexpr bool FITS = STAGES_RAW >= (CPS == 1 ? 3 : 4);
  static constexpr int COLS = MT * N;
  static constexpr int ACC = 2 * COLS <= 512 ? 2 : 1;
  static constexpr int TCOLS = ACC * COLS <= 32 ? 32 : ACC * COLS <= 64 ? 64 : ACC * COLS <= 128 ? 128
                               : ACC * COLS <= 256 ? 256 : 512;
  static constexpr uint32_t IDESC = tc::idesc_bf16(M, N, 1, 1);
  static constexpr int SMEM = STAGES * STAGE + 1024 + IDX_BYTES + 4096;
};

// MN-major SW128 tile: 16 B chunk `c` (8 elements along M/N) of pair-row kk
__device__ __forceinline__ uint32_t wg_off(int c, int kk) {
  return (uint32_t)((c >> 3) * 8192 + (kk >> 3) * 1024 + (kk & 7) * 128 + (((c & 7) ^ (kk & 7)) << 4));
}

template <int CIN, int COUT, int CPS = 1>
__global__ void __launch_bounds__(kTcThreads, CPS) conv_wgrad_tc_kernel(const __grid_constant__ WgParams p) {
  ::vp::pdl_begin();
  using C = WgTC<CIN, COUT, CPS>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  int32_t* s_pin = reinterpret_cast<int32_t*>(smem + C::STAGES * C::STAGE);
  int32_t* s_pout = s_pin + kWgMaxChunk;
  uint8_t* book = reinterpret_cast<uint8_t*>(s_pout + kWgMaxChunk);
  uint64_t* full = reinterpret_cast<uint64_t*>(book);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + C::ACC;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tempty + C::ACC);
  int* s_pref = reinterpret_cast<int*>(book + 512);  // K+1 <= 344 ints

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = p.K;
  __shared__ int s_chunk;
  // the pair pointers, all K + 1 loads in flight (a serial loop over them
  // costs K dependent L2 round trips before the first item)
  __shared__ int s_ptr[VP_MAX_OFFSETS + 1];
  for (int k = tid; k <= K; k += blockDim.x) s_ptr[k] = __ldg(p.pptr + k);
  __syncthreads();
  if (tid == 0) {
    s_chunk = p.chunk > 0 ? p.chunk : wg_device_chunk(s_ptr[K] - s_ptr[0], K, gridDim.x, p.max_items, p.chunk_min);
    if (blockIdx.x == 0 && p.chunk_out) *p.chunk_out = s_chunk;
  }
  __syncthreads();
  const int chunk = s_chunk;
  if (tid == 0) {
    int acc = 0;
    for (int k = 0; k < K; ++k) {
      s_pref[k] = acc;
      acc += (s_ptr[k + 1] - s_ptr[k] + chunk - 1) / chunk;
    }
    s_pref[K] = acc;
    for (int s = 0; s < C::STAGES; ++s) {
      tc::mbar_init(&full[s], kTcProd);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < C::ACC; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], kTcEpi);
    }
    tc::fence_mbar_init();
  }
  __syncthreads();
  const int n_items = s_pref[K];
  if ((int)blockIdx.x >= n_items) return;
  if (warp == 8) tc::tmem_alloc(s_tmem, C::TCOLS);
  if ((COUT < 64 || CIN < 64) && warp < 4) {  // zero the never-loaded padding once
    for (int s = 0; s < C::STAGES; ++s) {
      uint4* q = reinterpret_cast<uint4*>(smem + s * C::STAGE);
      for (int i = tid; i < C::STAGE / 16; i += kTcProd) q[i] = make_uint4(0, 0, 0, 0);
    }
    tc::fence_proxy_async_smem();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const uint32_t sbase = tc::smem_u32(smem);

  auto item_range = [&](int item, int& k, int& p0, int& p1) {
    k = 0;
    while (s_pref[k + 1] <= item) ++k;
    p0 = s_ptr[k] + (item - s_pref[k]) * chunk;
    p1 = min(s_ptr[k + 1], p0 + chunk);
  };

  if (warp < 4) {
    // ============================ producers ============================
    uint32_t g = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      int k, p0, p1;
      item_range(item, k, p0, p1);
      const int np = p1 - p0;
      asm volatile("bar.sync 1, 128;" ::: "memory");  // previous item's indices consumed
#pragma unroll 4
      for (int i = tid; i < np; i += kTcProd) {
        s_pin[i] = __ldg(p.pin + p0 + i);
        s_pout[i] = __ldg(p.pout + p0 + i);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const int n_iter = (np + C::PK - 1) / C::PK;
      for (int it = 0; it < n_iter; ++it, ++g) {
        const int stage = g % C::STAGES;
        if (g >= (uint32_t)C::STAGES) tc::mbar_wait(&empty[stage], ((g / C::STAGES) - 1) & 1);
        const uint32_t a_s = sbase + stage * C::STAGE;
        const uint32_t b_s = a_s + C::A_BYTES;
        const int q0 = it * C::PK;
        constexpr int CA = COUT / 8, CB = CIN / 8;
#pragma unroll 4
        for (int e = tid; e < C::PK * CA; e += kTcProd) {
          const int kk = e / CA, c = e - (e / CA) * CA;
          const int q = q0 + kk;
          const bool ok = q < np;
          const int uo = ok ? s_pout[q] : 0;
          tc::cp_async16(a_s + wg_off(c, kk), p.g + (int64_t)uo * COUT + c * 8, ok ? 16 : 0);
        }
#pragma unroll 4
        for (int e = tid; e < C::PK * CB; e += kTcProd) {
          const int kk = e / CB, c = e - (e / CB) * CB;
          const int q = q0 + kk;
          const bool ok = q < np;
          const int vi = ok ? s_pin[q] : 0;
          tc::cp_async16(b_s + wg_off(c, kk), p.x + (int64_t)vi * CIN + c * 8, ok ? 16 : 0);
        }
        // the stage's full barrier completes when every producer's copies have landed
        tc::cp_async_arrive_noinc(&full[stage]);
      }
    }
    tc::cp_async_wait<0>();
  } else if (warp < 8) {
    // ============================ epilogue ============================
    const int ep = warp - 4;
    constexpr int PER = COUT * CIN;
    int ii = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++ii) {
      const int a = ii % C::ACC;
      tc::mbar_wait(&tfull[a], (ii / C::ACC) & 1);
      tc::tc_fence_after();
      float* dst = p.part + (int64_t)item * PER;  // chunk partial; wgrad_reduce_kernel sums in chunk order
#pragma unroll 1
      for (int mt = 0; mt < C::MT; ++mt) {
#pragma unroll 1
        for (int c0 = 0; c0 < CIN; c0 += 32) {
          float v[32];
          tc::tmem_ld32(tmem + ((uint32_t)(ep * 32) << 16) + a * C::COLS + mt * C::N + c0, v);
          int m;
          bool ok;
          if (C::M == 128) {
            m = mt * 128 + ep * 32 + lane;
            ok = true;
          } else {  // M=64: row r lives in TMEM lane (r % 16) + 32 * (r / 16)
            m = ep * 16 + lane;
            ok = lane < 16;
          }
          if (ok && m < COUT) {
            float4* d = reinterpret_cast<float4*>(dst + (int64_t)m * CIN + c0);
#pragma unroll
            for (int q = 0; q < 8; ++q) d[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
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
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++ii) {
      int k, p0, p1;
      item_range(item, k, p0, p1);
      const int n_iter = (p1 - p0 + C::PK - 1) / C::PK;
      const int a = ii % C::ACC;
      const int use = ii / C::ACC;
      if (use >= 1) tc::mbar_wait(&tempty[a], (use - 1) & 1);
      tc::tc_fence_after();
      const uint32_t d = tmem + a * C::COLS;
      for (int it = 0; it < n_iter; ++it, ++g) {
        const int stage = g % C::STAGES;
        tc::mbar_wait(&full[stage], (g / C::STAGES) & 1);
        tc::tc_fence_after();
        const uint32_t a_s = sbase + stage * C::STAGE;
        const uint32_t b_s = a_s + C::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < C::PK / 16; ++kk) {
          const uint64_t bd = tc::smem_desc(b_s + kk * 2048, 8192, 1024, tc::kSwizzle128);
#pragma unroll
          for (int mt = 0; mt < C::MT; ++mt) {
            const uint64_t ad = tc::smem_desc(a_s + mt * 2 * 8192 + kk * 2048, 8192, 1024, tc::kSwizzle128);
            tc::mma_bf16(d + mt * C::N, ad, bd, C::IDESC, (it > 0 || kk > 0) ? 1u : 0u);
          }
        }
        tc::mma_commit(&empty[stage]);
      }
      tc::mma_commit(&tfull[a]);
    }
  }
  __syncthreads();
  if (warp == 8) tc::tmem_dealloc(tmem, C::TCOLS);
}

}  // namespace vp
