// Row-compacted sparse conv for the 32-wide levels (C_in = C_out = 32, bf16,
// K <= 27): forward (conv.py:186-208) and dgrad (conv.py:240).
//
// At C3's levels 0-1 a row has ~3-7 of its 27 neighbours.  The tcgen05
// implicit GEMM gathers every active offset for all 128 rows of a tile, so
// ~75% of its row slots are zero-fill and a tile is a 14-stage latency chain.
// Here a warp owns 32 output rows:
//   * each lane keeps its row's 27 neighbour indices in registers;
//   * offsets are taken in ascending order and packed into groups of <= kRowsCap
//     gathered rows (ballot + popc positions); each lane cp.async-gathers its
//     own neighbour rows, so one wait covers a whole group (typically 1-2 per
//     32 rows) instead of one per offset;
//   * per offset, mma.sync m16n8k16 over the compacted rows (16 at a time)
//     against W_k (all 27 weight slices staged once per CTA in shared memory),
//     and the fragments are added into the rows' fp32 accumulators in the
//     warp's shared memory.
// Every output row sums its offsets in ascending order through one warp ->
// fixed summation order (deterministic), no atomics, each row stored once.
#pragma once

#include "common.cuh"
#include "tc.cuh"

namespace vp {

constexpr int kRowsWarps = 8;            // warps per CTA, each independent
constexpr int kRowsCap = 64;             // gathered rows per group (per warp, double-buffered)
constexpr int kRowsStride = 40;          // bf16 per staged row (32 + 8 pad: conflict-free ldmatrix)
constexpr int kRowsAccStride = 40;       // fp32 per accumulator row
constexpr int kRowsW = 32 * kRowsStride; // bf16 per staged weight slice [32][40]

struct RowsSmem {
  static constexpr int W_BYTES = 27 * kRowsW * 2;
  static constexpr int A_BYTES = (kRowsCap + 16) * kRowsStride * 2;
  static constexpr int ACC_BYTES = 32 * kRowsAccStride * 4;
  static constexpr int DST_BYTES = (kRowsCap + 16) * 4;
  static constexpr int WARP_BYTES = 2 * A_BYTES + ACC_BYTES + 2 * DST_BYTES;
  static constexpr int TOTAL = W_BYTES + kRowsWarps * WARP_BYTES;
};

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void mma_bf16_16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// WT = false: out[r, co] = sum_k sum_ci W[k, co, ci] x[t[r,k], ci]      (forward)
// WT = true : out[r, ci] = sum_k sum_co W[k, co, ci] x[t[r,k], co]      (dgrad, x = g)
template <bool WT>
__global__ void __launch_bounds__(kRowsWarps * 32, 1)
conv_rows32_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w, int K,
                   const int32_t* __restrict__ table, int flip, const int32_t* __restrict__ perm,
                   const int32_t* __restrict__ n_out_dev, int64_t cap_out, void* __restrict__ y, int y_dtype) {
  extern __shared__ __align__(128) uint8_t smem[];
  __nv_bfloat16* sW = reinterpret_cast<__nv_bfloat16*>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wsm = smem + RowsSmem::W_BYTES + warp * RowsSmem::WARP_BYTES;
  __nv_bfloat16* sA = reinterpret_cast<__nv_bfloat16*>(wsm);
  float* sAcc = reinterpret_cast<float*>(wsm + 2 * RowsSmem::A_BYTES);
  int* sDst = reinterpret_cast<int*>(wsm + 2 * RowsSmem::A_BYTES + RowsSmem::ACC_BYTES);  // [2][kRowsCap + 16]

  // (the weights may come from a cast kernel just before: wait first)
  ::vp::pdl_begin();
  for (int e = threadIdx.x * 8; e < K * 1024; e += blockDim.x * 8) {
    const int kk = e >> 10, r = e & 1023, co = r >> 5, ci = r & 31;
    const uint4 v = *reinterpret_cast<const uint4*>(w + e);
    if (!WT) {
      *reinterpret_cast<uint4*>(sW + kk * kRowsW + co * kRowsStride + ci) = v;
    } else {
      const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
      for (int u = 0; u < 8; ++u) sW[kk * kRowsW + (ci + u) * kRowsStride + co] = h[u];
    }
  }
  __syncthreads();

  const int n_out = load_count(n_out_dev, cap_out);
  const int nslices = (n_out + 31) >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const uint32_t sA_u = tc::smem_u32(sA), sW_u = tc::smem_u32(sW);

  for (int slice = blockIdx.x * kRowsWarps + warp; slice < nslices; slice += gridDim.x * kRowsWarps) {
    const int t = slice * 32 + lane;
    const bool valid = t < n_out;
    int nb[27];
#pragma unroll
    for (int kk = 0; kk < 27; ++kk)
      nb[kk] = (valid && kk < K) ? __ldg(table + (int64_t)t * K + (flip ? K - 1 - kk : kk)) : -1;
#pragma unroll
    for (int c = 0; c < 32; c += 4)
      *reinterpret_cast<float4*>(sAcc + lane * kRowsAccStride + c) = make_float4(0.f, 0.f, 0.f, 0.f);

    // Offsets are gathered in groups of <= kRowsCap rows into two staging
    // buffers: the next group's cp.async gathers fly while this one computes.
    int kk = 0;
    int gk0[2], gk1[2], gfill[2], gst[2][27];
    auto form = [&](int bsel) {
      const uint32_t abase = sA_u + (uint32_t)(bsel * RowsSmem::A_BYTES);
      int* dsts = sDst + bsel * (kRowsCap + 16);
      int fill = 0;
      gk0[bsel] = kk;
#pragma unroll 1
      for (; kk < K; ++kk) {
        int v = -1;
#pragma unroll
        for (int q = 0; q < 27; ++q)
          if (q == kk) v = nb[q];
        const uint32_t mask = __ballot_sync(0xffffffffu, v >= 0);
        const int m = __popc(mask);
        if (fill > 0 && fill + m > kRowsCap) break;
        gst[bsel][kk - gk0[bsel]] = fill;
        if (v >= 0) {
          const int pos = fill + __popc(mask & ((1u << lane) - 1u));
          dsts[pos] = lane;
          const __nv_bfloat16* src = x + (int64_t)v * 32;
          const uint32_t dst = abase + (uint32_t)(pos * kRowsStride) * 2u;
#pragma unroll
          for (int q = 0; q < 4; ++q) tc::cp_async16(dst + q * 16, src + q * 8, 16);
        }
        fill += m;
      }
      gk1[bsel] = kk;
      gfill[bsel] = fill;
      tc::cp_async_commit();
    };
    auto compute = [&](int bsel) {
      const uint32_t abase = sA_u + (uint32_t)(bsel * RowsSmem::A_BYTES);
      const int* dsts = sDst + bsel * (kRowsCap + 16);
      const int nk = gk1[bsel] - gk0[bsel];
#pragma unroll 1
      for (int j = 0; j < nk; ++j) {
        const int s0 = gst[bsel][j];
        const int s1 = (j + 1 < nk) ? gst[bsel][j + 1] : gfill[bsel];
        if (s1 == s0) continue;
        const int k = gk0[bsel] + j;
        // B fragments of W_k: [n-tile 0..3][k16 step 0..1] x 2 regs
        uint32_t b[4][2][2];
#pragma unroll
        for (int np = 0; np < 2; ++np)
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const int n = np * 16 + ((lane >> 4) << 3) + (lane & 7);
            const int kd = ks * 16 + (((lane >> 3) & 1) << 3);
            uint32_t r0, r1, r2, r3;
            ldsm_x4(sW_u + (uint32_t)(k * kRowsW + n * kRowsStride + kd) * 2u, r0, r1, r2, r3);
            b[np * 2][ks][0] = r0;
            b[np * 2][ks][1] = r1;
            b[np * 2 + 1][ks][0] = r2;
            b[np * 2 + 1][ks][1] = r3;
          }
#pragma unroll 1
        for (int base = s0; base < s1; base += 16) {
          float c[4][4];
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) c[nt][0] = c[nt][1] = c[nt][2] = c[nt][3] = 0.f;
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            uint32_t a[4];
            const int row = base + (lane & 15);
            const int kd = ks * 16 + ((lane >> 4) << 3);
            ldsm_x4(abase + (uint32_t)(row * kRowsStride + kd) * 2u, a[0], a[1], a[2], a[3]);
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) mma_bf16_16816(c[nt], a, b[nt][ks][0], b[nt][ks][1]);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i = base + g + h * 8;
            if (i < s1) {
              float* dst = sAcc + dsts[i] * kRowsAccStride + tig * 2;
#pragma unroll
              for (int nt = 0; nt < 4; ++nt) {
                float2 o = *reinterpret_cast<float2*>(dst + nt * 8);
                o.x += c[nt][2 * h];
                o.y += c[nt][2 * h + 1];
                *reinterpret_cast<float2*>(dst + nt * 8) = o;
              }
            }
          }
          __syncwarp();
        }
      }
    };
    int cur = 0;
    form(0);
    while (true) {
      const bool more = kk < K;
      if (more) {
        form(cur ^ 1);
        tc::cp_async_wait<1>();
      } else {
        tc::cp_async_wait<0>();
      }
      __syncwarp();
      compute(cur);
      __syncwarp();
      if (!more) break;
      cur ^= 1;
    }
    // ---- each lane stores its own row once
    if (valid) {
      const int64_t orow = perm ? (int64_t)perm[t] : (int64_t)t;
      const float* a = sAcc + lane * kRowsAccStride;
      if (y_dtype == VP_BF16) {
        uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(y) + orow * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 r;
          __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
          for (int u = 0; u < 4; ++u) h[u] = __floats2bfloat162_rn(a[q * 8 + 2 * u], a[q * 8 + 2 * u + 1]);
          o[q] = r;
        }
      } else {
        float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + orow * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] = *reinterpret_cast<const float4*>(a + q * 4);
      }
    }
    __syncwarp();
  }
}

}  // namespace vp
