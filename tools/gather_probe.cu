// Microbenchmark: producer-side cost of gathering 128 random 128-byte rows
// per pipeline stage into shared memory on sm_100a, for several completion
// mechanisms.  One CTA per SM, 4 producer warps + 1 consumer thread that only
// waits for "full" and releases "empty" (no MMA), STAGES-deep ring.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/gather_probe.cu -o tools/gather_probe
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

constexpr int STAGES = 8;
constexpr int STAGE_BYTES = 128 * 128;
constexpr int NSTAGE = 2000;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
          su32(b)),
      "r"(ph), "r"(0x989680)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, int n) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}

// pseudo-random row (or -1 = miss) computed in registers: measures only the copy path
__device__ __forceinline__ int pick(int b, int g, int r, int nrows, float hit) {
  uint32_t x = (uint32_t)(b * 7919 + g * 131071 + r * 2654435761u);
  x ^= x >> 15; x *= 2246822519u; x ^= x >> 13; x *= 3266489917u; x ^= x >> 16;
  return ((x & 0xffff) < (uint32_t)(hit * 65536.f)) ? (int)((x >> 8) % (uint32_t)nrows) : -1;
}

// variant: 0 = per-thread noinc arrive (count 128)
//          1 = wait_group<4> + fence + lane-0 arrive (count 4)
//          2 = wait_group<4> + lane-0 arrive, no proxy fence
//          3 = ld.global.v4 -> st.shared + lane-0 arrive after syncwarp
//          4 = cp.async.bulk (1 per hit row, issued by the row's lane 0) + expect_tx
//          5 = cp.async hits only (no zero fill) + wait_group(6) + warp arrive
template <int VARIANT>
__global__ void __launch_bounds__(160, 1) probe(const uint4* __restrict__ table, int nrows, const int* __restrict__ idx,
                                                 float hit_rate, long long* out_cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], VARIANT == 0 ? 128 : (VARIANT == 4 ? 4 : 4));
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  long long t0 = clock64();
  if (warp < 4) {
    const int q = tid & 7, rb = tid >> 3;
    for (int g = 0; g < NSTAGE; ++g) {
      const int st = g % STAGES;
      if (g >= STAGES) mbar_wait(&empty[st], ((g / STAGES) - 1) & 1);
      const uint32_t a = su32(smem + st * STAGE_BYTES);
      if (VARIANT == 4) {
        // lane l issues the bulk copies for rows 4l..4l+3 of this warp's 32-row slice
        int vv[4], nb = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          vv[j] = pick(blockIdx.x, g, warp * 32 + (lane * 4 + j) % 32, nrows, hit_rate);
          nb += vv[j] >= 0;
        }
        for (int o = 16; o > 0; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(nb * 128)
                       : "memory");
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (vv[j] >= 0)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];" ::"r"(
                             a + (warp * 32 + (lane * 4 + j) % 32) * 128),
                         "l"(table + (size_t)vv[j] * 8), "r"(su32(&full[st]))
                         : "memory");
        continue;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = rb + 16 * i;
        const int v = pick(blockIdx.x, g, r, nrows, hit_rate);
        const bool hit = v >= 0;
        const uint4* src = table + (size_t)(hit ? v : 0) * 8 + q;
        const uint32_t dst = a + r * 128 + ((q ^ (r & 7)) << 4);
        if (VARIANT == 5) {
          if (hit) cp16(dst, src, 16);
          continue;
        }
        if (VARIANT == 6) {  // predicated (no divergence): only hit lanes issue a request
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %2, 0;\n@p cp.async.cg.shared.global [%0], [%1], 16;\n}\n" ::"r"(dst),
                       "l"(src), "r"((int)hit) : "memory");
          continue;
        }
        if (VARIANT == 3) {
          uint4 x = hit ? __ldg(src) : make_uint4(0, 0, 0, 0);
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(dst), "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w));
        } else {
          cp16(dst, src, hit ? 16 : 0);
        }
      }
      if (VARIANT == 4) {
        // the 8 expect_tx arrives per warp... only lane 0's first counts: use one extra arrive
      } else if (VARIANT == 5 || VARIANT == 6) {
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (g >= 6) {
          asm volatile("cp.async.wait_group 6;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[(g - 6) % STAGES]);
        }
      } else if (VARIANT == 0) {
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[st])) : "memory");
      } else if (VARIANT == 1 || VARIANT == 2) {
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (g >= 4) {
          asm volatile("cp.async.wait_group 4;" ::: "memory");
          if (VARIANT == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[(g - 4) % STAGES]);
        }
      } else {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[st]);
      }
    }
    if (VARIANT == 1 || VARIANT == 2) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        for (int g = NSTAGE - 4; g < NSTAGE; ++g) mbar_arrive(&full[g % STAGES]);
    }
    if (VARIANT == 5 || VARIANT == 6) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        for (int g = NSTAGE - 6; g < NSTAGE; ++g) mbar_arrive(&full[g % STAGES]);
    }
  } else if (tid == 128) {
    for (int g = 0; g < NSTAGE; ++g) {
      const int st = g % STAGES;
      mbar_wait(&full[st], (g / STAGES) & 1);
      mbar_arrive(&empty[st]);
    }
  }
  __syncthreads();
  if (tid == 0) out_cycles[blockIdx.x] = clock64() - t0;
}

template <int V>
void run(const uint4* table, int nrows, const int* idx, long long* dcyc, float hit, const char* name) {
  cudaFuncSetAttribute(probe<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * STAGE_BYTES);
  probe<V><<<148, 160, STAGES * STAGE_BYTES>>>(table, nrows, idx, hit, dcyc);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<V><<<148, 160, STAGES * STAGE_BYTES>>>(table, nrows, idx, hit, dcyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  printf("%-44s hit=%.2f : %.3f us/stage/SM  (%.1f GB/s useful)  %s\n", name, hit, ms * 1e3 / NSTAGE,
         148.0 * NSTAGE * 128 * 128 * hit / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
}

int main() {
  const int nrows = 200000;
  uint4* table;
  cudaMalloc(&table, (size_t)nrows * 128);
  cudaMemset(table, 1, (size_t)nrows * 128);
  int* idx;
  cudaMalloc(&idx, (1 << 20) * 4);
  long long* dcyc;
  cudaMalloc(&dcyc, 148 * 8);
  for (float hit : {1.0f, 0.25f, 0.1f}) {
    std::vector<int> h(1 << 20);
    uint32_t s = 12345;
    for (auto& v : h) {
      s = s * 1664525u + 1013904223u;
      float u = (s >> 8) / 16777216.0f;
      s = s * 1664525u + 1013904223u;
      v = u < hit ? (int)(s % nrows) : -1;
    }
    cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    run<0>(table, nrows, idx, dcyc, hit, "cp.async + per-thread noinc arrive");
    run<1>(table, nrows, idx, dcyc, hit, "cp.async + wait_group(4) + fence + warp arrive");
    run<2>(table, nrows, idx, dcyc, hit, "cp.async + wait_group(4) + warp arrive");
    run<3>(table, nrows, idx, dcyc, hit, "ldg.128 -> st.shared + warp arrive");
    run<4>(table, nrows, idx, dcyc, hit, "cp.async.bulk per hit row + expect_tx");
    run<5>(table, nrows, idx, dcyc, hit, "cp.async hits only + wait_group(6) + warp arrive");
    run<6>(table, nrows, idx, dcyc, hit, "predicated cp.async hits + wait_group(6)");
  }
  return 0;
}
