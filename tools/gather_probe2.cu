// Microbenchmark: what bounds the producer-side gather of 128 random 128-byte
// rows per pipeline stage on sm_100a?  Sweeps ring depth, producer warp
// count and the lane->row mapping (thread-per-row vs 8 lanes per row); the
// consumer thread only waits "full" and releases "empty" (no MMA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/gather_probe2.cu -o tools/gather_probe2
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

constexpr int STAGE_BYTES = 128 * 128;
constexpr int NSTAGE = 3000;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ int g_waitmode = 0;
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph, int mode) {
  if (mode == 0) {
    asm volatile(
        "{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
            su32(b)),
        "r"(ph), "r"(0x989680)
        : "memory");
  } else if (mode == 1) {
    asm volatile(
        "{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
            su32(b)),
        "r"(ph)
        : "memory");
  } else {
    asm volatile(
        "{\n.reg .pred P1;\nW: mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
            su32(b)),
        "r"(ph)
        : "memory");
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, int n) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ int pick(int b, int g, int r, int nrows) {
  uint32_t x = (uint32_t)(b * 7919 + g * 131071 + r * 2654435761u);
  x ^= x >> 15; x *= 2246822519u; x ^= x >> 13; x *= 3266489917u; x ^= x >> 16;
  return (int)(x % (uint32_t)nrows);
}

// MAP 0: thread t of the PW*32 producers owns rows t, t+P, ... (8 x 16B each)
// MAP 1: 8 lanes per row, a warp instruction covers 4 full rows
// MAP 2: like 1 but ld.global.v4 + st.shared (register staged), warp arrive
template <int STAGES, int PW, int MAP, int WM, int RB = 1, int HIT4 = 4>
__global__ void probe(const uint4* __restrict__ table, int nrows, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  constexpr int P = PW * 32;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], (MAP == 2 || MAP == 5) ? PW : P);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp < PW) {
    for (int g = 0; g < NSTAGE; ++g) {
      const int st = g % STAGES;
      if (g >= STAGES) mbar_wait(&empty[st], ((g / STAGES) - 1) & 1, WM);
      const uint32_t a = su32(smem + st * STAGE_BYTES * RB);
      if (MAP == 0) {
        for (int r = tid; r < 128; r += P) {
          const uint4* src = table + (size_t)pick(blockIdx.x, g, r, nrows) * 8;
#pragma unroll
          for (int q = 0; q < 8; ++q) cp16(a + r * 128 + ((q ^ (r & 7)) << 4), src + q, 16);
        }
      } else {
        const int q = lane & 7;
        const int rmax = MAP == 4 ? 128 * HIT4 / 4 : 128;  // MAP 4: only HIT4/4 of the rows, compacted
        for (int r = warp * 4 + (lane >> 3); r < rmax; r += PW * 4) {
          const int pk = pick(blockIdx.x, g, r, nrows / RB);
          const uint4* src = table + (size_t)pk * 8 * RB + q;
          const uint32_t dst = a + r * 128 + ((q ^ (r & 7)) << 4);
          if (MAP == 4 || MAP == 5) {
            cp16(dst, src, 16);
          } else if (MAP == 1) {
            if (HIT4 >= 4 || (pk & 3) < HIT4) {
#pragma unroll
              for (int rb = 0; rb < RB; ++rb) cp16(dst + rb * STAGE_BYTES, src + rb * 8, 16);
            }
          } else if (MAP == 3) {  // zero-fill the misses (src-size 0) instead of skipping them
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) cp16(dst + rb * STAGE_BYTES, src + rb * 8, (pk & 3) < HIT4 ? 16 : 0);
          } else {
            uint4 x = __ldg(src);
            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(dst), "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w));
          }
        }
      }
      if (MAP == 2) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[st]);
      } else if (MAP == 5) {
        constexpr int D = STAGES - 1;
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (g >= D) {
          asm volatile("cp.async.wait_group %0;" ::"n"(D) : "memory");
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[(g - D) % STAGES]);
        }
        if (g == NSTAGE - 1) {
          asm volatile("cp.async.wait_group 0;" ::: "memory");
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0)
            for (int gg = NSTAGE - D; gg < NSTAGE; ++gg) mbar_arrive(&full[gg % STAGES]);
        }
      } else {
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[st])) : "memory");
      }
    }
  } else if (tid == P) {
    for (int g = 0; g < NSTAGE; ++g) {
      const int st = g % STAGES;
      mbar_wait(&full[st], (g / STAGES) & 1, WM);
      mbar_arrive(&empty[st]);
    }
  }
  __syncthreads();
  if (tid == 0) out[blockIdx.x] = 0;
}

template <int STAGES, int PW, int MAP, int WM = 0, int RB = 1, int HIT4 = 4>
void run(const uint4* table, int nrows, long long* d, int ctas_per_sm) {
  auto k = probe<STAGES, PW, MAP, WM, RB, HIT4>;
  const int smem = STAGES * STAGE_BYTES * RB;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = 148 * ctas_per_sm;
  k<<<grid, PW * 32 + 32, smem>>>(table, nrows, d);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<grid, PW * 32 + 32, smem>>>(table, nrows, d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double stages_per_sm = (double)NSTAGE * ctas_per_sm;
  printf("HIT4=%d RB=%d WM=%d STAGES=%2d PW=%d MAP=%d ctas/SM=%d : %.3f us/16KB/SM  %.0f GB/s  %s\n", HIT4, RB, WM, STAGES, PW, MAP, ctas_per_sm,
         ms * 1e3 / stages_per_sm / RB, 148.0 * stages_per_sm * STAGE_BYTES * RB / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int nrows = 200000;  // 25.6 MB: L2 resident
  uint4* table;
  cudaMalloc(&table, (size_t)nrows * 128);
  cudaMemset(table, 1, (size_t)nrows * 128);
  long long* d;
  cudaMalloc(&d, 148 * 8 * 8);
  run<3, 4, 1, 0, 1, 4>(table, nrows, d, 1);
  run<3, 4, 5, 0, 1, 4>(table, nrows, d, 1);
  run<6, 4, 5, 0, 1, 4>(table, nrows, d, 1);
  run<3, 4, 5, 0, 1, 4>(table, nrows, d, 2);
  run<4, 4, 5, 0, 1, 4>(table, nrows, d, 2);
  run<3, 4, 1, 0, 1, 4>(table, nrows, d, 2);
  run<2, 4, 1, 0, 1, 4>(table, nrows, d, 3);
  run<3, 4, 5, 0, 1, 4>(table, nrows, d, 3);
  return 0;
}
