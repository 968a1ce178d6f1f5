// Batch-norm statistics fused into the producer of the BN input (the conv
// forward epilogue) or of its gradient (the dgrad epilogue of the NEXT conv,
// or the split-K reduction that finishes either).  No reference code exists
// for this glue (SPEC.md:184-185 non-goal); it replaces the separate
// statistics pass over the rows (bn_partial_kernel) on the training step's
// critical path.
//
//   mode 1 (forward):  y = conv output, rounded to the output dtype;
//                      partials (sum y, sum y^2) per channel.
//   mode 2 (backward): g = round(y) (+ add) , zeroed where act <= 0 (ReLU),
//                      stored rounded in place of y;
//                      partials (sum g, sum g * (pre - mean)) per channel
//                      (pre = the BN layer's input; rstd is applied when the
//                      partials are reduced: vp_bn_backward_part).
//
// Partials are [nb][2][C] fp32 rows after a 256-byte header whose first int
// is nb (written by the producer on the device, so the consumer needs no host
// sync).  Every producer reduces in a fixed order (warp transpose tree, then
// warps in order, then the producer's item order) -> deterministic.
#pragma once
#include "common.cuh"

namespace vp {

constexpr int kBnPartHeader = 256;  // bytes before the partial rows
constexpr int kBnPartRows = 3 * kNumSMs;  // most partial rows any producer writes (conv grid <= 3 CTAs/SM)

struct BnEpi {
  int mode;               // 0 off, 1 forward stats, 2 backward (masked gradient + stats)
  float* part;            // [nb][2][C]
  int* nb;                // header: rows written
  const void* add;        // mode 2, nullable: second gradient branch (same dtype as the output)
  const void* act;        // mode 2, nullable: ReLU output of the BN layer (mask act > 0)
  const void* pre;        // mode 2: BN input (the BN layer's conv output)
  const float* mean;      // mode 2: BN batch mean
  // finalize in the producer chain (out_a != null): mode 1 -> out_a = mean,
  // out_b = rstd (eps); mode 2 -> out_a = ggamma = rstd * sum g(x-mean),
  // out_b = gbeta = sum g
  float* out_a;
  float* out_b;
  const float* rstd;
  float eps;
  unsigned int* ticket;   // header word (zero before first use; re-arms itself)
  int early;              // trigger the dependent (apply) launch at the start of the finalizing kernel
  int rows_pass;          // conv epilogue stores raw rows; the split-K reduction kernel transforms them
};

constexpr int kBnTicketOffset = 64;  // bytes into the header

// The partial rows -> the BN statistics, channels [32 cb, 32 cb + 32): a
// 1024-thread block, lane = channel, warps 0-15 sum column 0 (sum y | sum g)
// and 16-31 column 1 over rows w, w + 16, ... (8 loads in flight), in double,
// then the 16 warps in order.  Fixed order -> deterministic.
__device__ __forceinline__ void bn_finalize_block(const float* __restrict__ part, int nb, int C, int n, int mode,
                                                  float eps, const float* __restrict__ rstd_in, float* __restrict__ out_a,
                                                  float* __restrict__ out_b, int cb, double (*s)[33]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = warp >> 4, wg = warp & 15;
  const int c = cb * 32 + lane;
  double acc = 0.0;
  if (c < C) {
    for (int b0 = wg; b0 < nb; b0 += 16 * 8) {
      float v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int b = b0 + 16 * q;
        v[q] = b < nb ? __ldcg(part + ((int64_t)b * 2 + h) * C + c) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) acc += v[q];
    }
  }
  s[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && c < C) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int w = 0; w < 16; ++w) {
      s0 += s[w][lane];
      s1 += s[16 + w][lane];
    }
    if (mode == 1) {
      const double mu = n > 0 ? s0 / n : 0.0;
      double var = n > 0 ? s1 / n - mu * mu : 0.0;
      if (var < 0) var = 0;
      out_a[c] = (float)mu;
      out_b[c] = (float)(1.0 / sqrt(var + (double)eps));
    } else {
      out_a[c] = (float)(s1 * (double)rstd_in[c]);
      out_b[c] = (float)s0;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ float bf16_round(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }

__device__ __forceinline__ void bf16x8_unpack(const uint4& r, float* o) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 f = __bfloat1622float2(h[q]);
    o[2 * q] = f.x;
    o[2 * q + 1] = f.y;
  }
}

// One row's 32-channel chunk [c0, c0+32) of a bf16 output with leading
// dimension ND: apply the epilogue mode to the fp32 results v, store the
// bf16 row (valid rows only), and return per lane (for channel c0 + lane) the
// warp's sums of the two statistics.  Called by all 32 lanes.
//
// The sums are a transpose tree (lane l ends with element l summed over the
// warp, every add in a fixed order).  Its first exchange pairs element i with
// i + 16, so channels are produced in those pairs (8 + 8 at a time) and only
// 16 + 16 partial values stay live: the epilogue runs inside the conv
// kernel's register budget.
template <int ND>
__device__ __forceinline__ void bn_epi_chunk32(const BnEpi& e, const float (&v)[32], bool valid, int64_t orow, int c0,
                                               __nv_bfloat16* __restrict__ y, float& s1, float& s2) {
  const int lane = threadIdx.x & 31;
  const bool up16 = (lane & 16) != 0;
  float a[16], b[16];
  const int64_t base = orow * ND + c0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // channels [8h, 8h+8) and [16+8h, 16+8h+8)
    float lo[8], hi[8], blo[8], bhi[8];
    if (valid && e.mode == 2) {
      const uint4* pa = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(e.add) + base);
      const uint4* pc = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(e.act) + base);
      const uint4* pp = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(e.pre) + base);
      const uint4 z = make_uint4(0u, 0u, 0u, 0u), one = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
      const uint4 ra0 = e.add ? __ldg(pa + h) : z, ra1 = e.add ? __ldg(pa + 2 + h) : z;
      const uint4 rc0 = e.act ? __ldg(pc + h) : one, rc1 = e.act ? __ldg(pc + 2 + h) : one;
      const uint4 rp0 = __ldg(pp + h), rp1 = __ldg(pp + 2 + h);
      float fa[8], fc[8], fp[8];
      bf16x8_unpack(ra0, fa);
      bf16x8_unpack(rc0, fc);
      bf16x8_unpack(rp0, fp);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float g = bf16_round(v[8 * h + j]) + fa[j];
        lo[j] = fc[j] > 0.f ? bf16_round(g) : 0.f;
        blo[j] = lo[j] * (fp[j] - __ldg(e.mean + c0 + 8 * h + j));
      }
      bf16x8_unpack(ra1, fa);
      bf16x8_unpack(rc1, fc);
      bf16x8_unpack(rp1, fp);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float g = bf16_round(v[16 + 8 * h + j]) + fa[j];
        hi[j] = fc[j] > 0.f ? bf16_round(g) : 0.f;
        bhi[j] = hi[j] * (fp[j] - __ldg(e.mean + c0 + 16 + 8 * h + j));
      }
    } else if (valid) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        lo[j] = bf16_round(v[8 * h + j]);
        hi[j] = bf16_round(v[16 + 8 * h + j]);
        blo[j] = lo[j] * lo[j];
        bhi[j] = hi[j] * hi[j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) lo[j] = hi[j] = blo[j] = bhi[j] = 0.f;
    }
    if (valid) {
      uint4 pk0, pk1;
      __nv_bfloat162* h0 = reinterpret_cast<__nv_bfloat162*>(&pk0);
      __nv_bfloat162* h1 = reinterpret_cast<__nv_bfloat162*>(&pk1);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        h0[j] = __floats2bfloat162_rn(lo[2 * j], lo[2 * j + 1]);
        h1[j] = __floats2bfloat162_rn(hi[2 * j], hi[2 * j + 1]);
      }
      uint4* dst = reinterpret_cast<uint4*>(y + base);
      dst[h] = pk0;
      dst[2 + h] = pk1;
    }
    // first transpose exchange (element i with i + 16)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float sa = up16 ? lo[j] : hi[j], ka = up16 ? hi[j] : lo[j];
      const float sb = up16 ? blo[j] : bhi[j], kb = up16 ? bhi[j] : blo[j];
      a[8 * h + j] = ka + __shfl_xor_sync(0xffffffffu, sa, 16);
      b[8 * h + j] = kb + __shfl_xor_sync(0xffffffffu, sb, 16);
    }
  }
#pragma unroll
  for (int w = 8; w >= 1; w >>= 1) {
    const bool up = (lane & w) != 0;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float sa = up ? a[i] : a[i + w], ka = up ? a[i + w] : a[i];
      const float sb = up ? b[i] : b[i + w], kb = up ? b[i + w] : b[i];
      a[i] = ka + __shfl_xor_sync(0xffffffffu, sa, w);
      b[i] = kb + __shfl_xor_sync(0xffffffffu, sb, w);
    }
  }
  s1 = a[0];
  s2 = b[0];
}

// standalone finalize (producers without a fused split-K reduction): one
// 1024-thread block per 32 channels
static __global__ void __launch_bounds__(1024)
bn_finalize_kernel(const BnEpi e, int C, const int32_t* n_dev, int64_t cap) {
  ::vp::pdl_begin();
  if (e.early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ double s[32][33];
  bn_finalize_block(e.part, *e.nb, C, load_count(n_dev, cap), e.mode, e.eps, e.rstd, e.out_a, e.out_b, blockIdx.x, s);
}

}  // namespace vp
