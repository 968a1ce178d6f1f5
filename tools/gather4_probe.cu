// Throughput probe: 128 random rows of ROWB bytes per pipeline stage into a
// 128B-swizzled shared tile, cp.async (4 producer warps, 8 lanes per 128 B
// row) vs TMA tile::gather4 (one warp; lane i issues rows 4i..4i+3; the
// stage completes as transaction bytes on its mbarrier).  A consumer thread
// only waits "full" / releases "empty" (no MMA).  Misses (row -1) are
// zero-filled by both: cp.async src-size 0 / gather4 out-of-bounds rows.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/gather4_probe.cu -o tools/gather4_probe -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

constexpr int NSTAGE = 3000;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
          su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ int pick(int b, int g, int r, int nrows, int hit4) {
  uint32_t x = (uint32_t)(b * 7919 + g * 131071 + r * 2654435761u);
  x ^= x >> 15; x *= 2246822519u; x ^= x >> 13; x *= 3266489917u; x ^= x >> 16;
  if ((int)((x >> 20) & 3) >= hit4) return -1;  // a miss: zero row
  return (int)(x % (uint32_t)nrows);
}

// MODE 0: cp.async (4 warps); MODE 1: gather4 (warp 0)
template <int STAGES, int MODE, int ROWB>
__global__ void probe(const __grid_constant__ CUtensorMap tm, const uint8_t* __restrict__ table, int nrows, int hit4,
                      long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr int STAGE = 128 * 128;  // a 128-row tile of 128 B swizzled rows (ROWB <= 128)
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], MODE == 0 ? 128 : 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp < 4) {
    if (MODE == 1 && warp > 0) {
    } else {
      for (int g = 0; g < NSTAGE; ++g) {
        const int st = g % STAGES;
        if (g >= STAGES) mbar_wait(&empty[st], ((g / STAGES) - 1) & 1);
        const uint32_t a = su32(smem + st * STAGE);
        if (MODE == 0) {
          const int q = lane & 7;
          constexpr int QN = ROWB / 16;  // 16 B chunks per row
          for (int r = warp * 4 + (lane >> 3); r < 128; r += 16) {
            const int pk = pick(blockIdx.x, g, r, nrows, hit4);
            if (q < QN) {
              const uint8_t* src = table + (size_t)(pk < 0 ? 0 : pk) * ROWB + q * 16;
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(a + r * 128 + ((q ^ (r & 7)) << 4)),
                           "l"(src), "r"(pk < 0 ? 0 : 16)
                           : "memory");
            }
          }
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[st])) : "memory");
        } else {
          if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])),
                         "r"(128 * ROWB)
                         : "memory");
          __syncwarp();
          int rr[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) rr[j] = pick(blockIdx.x, g, 4 * lane + j, nrows, hit4);  // -1 = out of bounds
          const uint32_t dst = a + lane * 4 * 128;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
              "l"(&tm), "r"(0), "r"(rr[0]), "r"(rr[1]), "r"(rr[2]), "r"(rr[3]), "r"(su32(&full[st]))
              : "memory");
        }
      }
    }
  } else if (tid == 128) {
    for (int g = 0; g < NSTAGE; ++g) {
      const int st = g % STAGES;
      mbar_wait(&full[st], (g / STAGES) & 1);
      mbar_arrive(&empty[st]);
    }
  }
  __syncthreads();
  if (tid == 0) out[blockIdx.x] = 0;
}

template <int STAGES, int MODE, int ROWB>
void run(const CUtensorMap& tm, const uint8_t* table, int nrows, int hit4, long long* d, int cps) {
  auto k = probe<STAGES, MODE, ROWB>;
  const int smem = STAGES * 128 * 128 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = 148 * cps;
  k<<<grid, 160, smem>>>(tm, table, nrows, hit4, d);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<grid, 160, smem>>>(tm, table, nrows, hit4, d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double stages = (double)NSTAGE * cps;
  printf("%-8s rowB=%3d hit=%d/4 stages=%d ctas/SM=%d : %.3f us/stage/SM, useful %.0f GB/s  %s\n",
         MODE ? "gather4" : "cp.async", ROWB, hit4, STAGES, cps, ms * 1e3 / stages,
         148.0 * stages * 128 * ROWB * hit4 / 4.0 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int nrows = 200000;
  for (int rowb : {64, 128}) {
    uint8_t* table;
    cudaMalloc(&table, (size_t)nrows * rowb);
    cudaMemset(table, 1, (size_t)nrows * rowb);
    long long* d;
    cudaMalloc(&d, 148 * 8 * 8);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap tm;
    const int cols = rowb / 2;  // bf16 elements per row
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)nrows};
    cuuint64_t strides[1] = {(cuuint64_t)rowb};
    cuuint32_t box[2] = {(cuuint32_t)cols, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, table, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, rowb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("encode failed %d\n", (int)r);
    for (int hit : {1, 4})
      for (int cps : {1, 2, 3}) {
        if (rowb == 64) {
          run<4, 0, 64>(tm, table, nrows, hit, d, cps);
          run<4, 1, 64>(tm, table, nrows, hit, d, cps);
        } else {
          run<4, 0, 128>(tm, table, nrows, hit, d, cps);
          run<4, 1, 128>(tm, table, nrows, hit, d, cps);
        }
      }
    cudaFree(table);
    cudaFree(d);
  }
  return 0;
}
