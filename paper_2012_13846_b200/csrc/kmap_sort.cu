// Neighbour-mask row ordering for the output-stationary implicit GEMM.
//
// A 128-row tile of the conv kernels pays one gather stage (and one MMA) per
// kernel offset that ANY of its rows uses.  In voxelization (first-seen)
// order a tile's rows are scattered over the cloud, so almost all 27 offsets
// are active while each row has only ~3 neighbours (surface clouds): ~9x
// the useful tensor work and gather stages.  Sorting the output rows by
// their 27-bit neighbour mask (stable LSD radix sort, cub) groups rows that
// use the same offsets, so a tile's active-offset set shrinks to about what
// its rows really use.  The conv kernels then read the permuted table and
// write output row perm[i] for table row i: every output row is still
// written exactly once, with the same per-row accumulation order (skipped
// offsets only contributed exact zeros) -> results identical to the
// unsorted order, deterministic, no atomics.
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace vp {

constexpr int kSortMaxK = 30;  // mask + the "empty row" sentinel bit fit a 32-bit key

__global__ void mask_keys_kernel(const int32_t* __restrict__ table, const int32_t* n_dev, int64_t cap, int K,
                                 uint32_t* __restrict__ keys, int32_t* __restrict__ rows) {
  ::vp::pdl_begin();
  const int n = load_count(n_dev, cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t m = 0;
    if (i < n) {
      const int32_t* t = table + i * K;
      for (int k = 0; k < K; ++k) m |= (uint32_t)(__ldg(t + k) >= 0) << k;
    } else {
      m = 1u << K;  // rows past the live count sort last
    }
    keys[i] = m;
    rows[i] = (int32_t)i;
  }
}

// table_sorted[i, :] = table[perm[i], :] (warp per row group, coalesced writes)
__global__ void permute_rows_kernel(const int32_t* __restrict__ table, const int32_t* __restrict__ perm,
                                    const int32_t* n_dev, int64_t cap, int K, int32_t* __restrict__ out) {
  ::vp::pdl_begin();
  const int n = load_count(n_dev, cap);
  const int64_t total = (int64_t)n * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / K;
    const int k = (int)(e - i * K);
    out[e] = __ldg(table + (int64_t)__ldg(perm + i) * K + k);
  }
}

static size_t cub_temp_bytes(int64_t cap, int K) {
  size_t t = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)std::max<int64_t>(cap, 1), 0,
                                  K + 1);
  return t;
}

}  // namespace vp

using namespace vp;

extern "C" {

size_t vp_kernel_map_sort_ws_bytes(int64_t cap, int32_t K) {
  const int kk = K <= kSortMaxK ? K : kSortMaxK;
  Carver c(nullptr, 0);
  c.take<uint32_t>(std::max<int64_t>(cap, 1));
  c.take<uint32_t>(std::max<int64_t>(cap, 1));
  c.take<int32_t>(std::max<int64_t>(cap, 1));
  c.take<char>(cub_temp_bytes(cap, kk));
  return c.off;
}

int vp_kernel_map_sort(const int32_t* table, const int32_t* n_dev, int64_t cap, int32_t K, int32_t* perm,
                       int32_t* table_sorted, void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(K >= 1 && K <= VP_MAX_OFFSETS, VP_EVALIDATION, "kernel offset count out of range");
  VP_REQUIRE(K <= kSortMaxK, VP_EVALIDATION, "kernel_map_sort: at most 30 offsets (mask key)");
  if (cap <= 0) return VP_OK;
  VP_REQUIRE(cap < (1ll << 31), VP_EVALIDATION, "kernel_map_sort: too many rows");
  Carver c(ws, ws_bytes);
  uint32_t* keys = c.take<uint32_t>(cap);
  uint32_t* keys_out = c.take<uint32_t>(cap);
  int32_t* rows = c.take<int32_t>(cap);
  size_t tb = cub_temp_bytes(cap, K);
  char* temp = c.take<char>(tb);
  VP_REQUIRE(c.ok(), VP_EVALIDATION, "kernel_map_sort: workspace too small");
  const int blocks = (int)std::min<int64_t>(ceil_div(cap, 256), grid_cap(8));
  ::vp::launch(mask_keys_kernel, blocks, 256, 0, st, table, n_dev, cap, K, keys, rows);
  VP_CHECK_LAUNCH("map_sort: keys");
  // stable LSD radix sort over the K+1 key bits (deterministic)
  VP_REQUIRE(cub::DeviceRadixSort::SortPairs(temp, tb, keys, keys_out, rows, perm, (int)cap, 0, K + 1, st) ==
                 cudaSuccess,
             VP_EINTERNAL, "map_sort: radix sort failed");
  {
    int _st = ::vp::check_launch("map_sort: radix", 6);  // cub onesweep: histogram, scan, 4 digit passes
    if (_st != VP_OK) return _st;
  }
  const int pblocks = (int)std::min<int64_t>(ceil_div(cap * K, 256), grid_cap(16));
  ::vp::launch(permute_rows_kernel, pblocks, 256, 0, st, table, perm, n_dev, cap, K, table_sorted);
  VP_CHECK_LAUNCH("map_sort: permute");
  return VP_OK;
}

}  // extern "C"
