// Probe: TMA tile::gather4 semantics on sm_100a (box {64,1}, SWIZZLE_128B,
// OOB rows zero-filled, complete_tx bytes).  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a tools/tma_gather4_probe.cu -o /tmp/probe
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap tm, int n_rows, const int* rows, unsigned short* out) {
  __shared__ __align__(1024) unsigned char buf[128 * 128];
  __shared__ __align__(8) unsigned long long bar;
  unsigned mb = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(128 * 128));
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    int i = threadIdx.x;
    unsigned dst = (unsigned)__cvta_generic_to_shared(buf + i * 512);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(&tm), "r"(0), "r"(rows[4 * i]), "r"(rows[4 * i + 1]), "r"(rows[4 * i + 2]), "r"(rows[4 * i + 3]), "r"(mb)
        : "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile(
        "{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(mb));
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 128 * 64; e += blockDim.x) out[e] = reinterpret_cast<unsigned short*>(buf)[e];
}

int main() {
  const int N = 1000, C = 64;
  std::vector<unsigned short> h(N * C);
  for (int r = 0; r < N; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = (unsigned short)(r * 64 + c);  // payload = element id
  unsigned short* d;
  cudaMalloc(&d, h.size() * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  std::vector<int> rows(128);
  for (int i = 0; i < 128; ++i) rows[i] = (i * 37 + 11) % N;
  rows[5] = N;      // OOB -> zeros
  rows[77] = N + 5; // OOB
  int* drows;
  cudaMalloc(&drows, 128 * 4);
  cudaMemcpy(drows, rows.data(), 128 * 4, cudaMemcpyHostToDevice);
  unsigned short* dout;
  cudaMalloc(&dout, 128 * 64 * 2);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)N};
  cuuint64_t strides[1] = {(cuuint64_t)C * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  probe<<<1, 128>>>(tm, N, drows, dout);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<unsigned short> out(128 * 64);
  cudaMemcpy(out.data(), dout, out.size() * 2, cudaMemcpyDeviceToHost);
  // expected: smem row i (128 B) holds source row rows[i], 16B chunk j stored at chunk j ^ (i & 7)
  int bad = 0;
  for (int i = 0; i < 128; ++i)
    for (int c = 0; c < 64; ++c) {
      int j = c / 8, w = c % 8;
      int phys = i * 64 + ((j ^ (i & 7)) * 8) + w;
      unsigned short expv = rows[i] < N ? (unsigned short)(rows[i] * 64 + c) : 0;
      if (out[phys] != expv) {
        if (bad < 5) printf("mismatch row %d col %d got %d want %d\n", i, c, out[phys], expv);
        ++bad;
      }
    }
  printf("gather4 probe: %s (%d mismatches)\n", bad ? "FAIL" : "OK", bad);
  return bad != 0;
}
