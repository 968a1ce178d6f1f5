// Wide-coordinate integer stage: the GPU counterpart of the reference's
// TupleCoordIndex fallback (kernels.py:95-122), used when rows do not fit the
// packed 64-bit key (kernels.py:40-78: D > 3 axes, or axis values beyond the
// 16-bit fields) — the reference then indexes whole coordinate tuples in a
// dict; here the rows are int64 [N, 1 + D] (D <= 7) and the index is an
// open-addressing table of row numbers whose probe compares the whole tuple
// against the stored row (first occurrence wins: atomicMin on equal keys, as
// the dict's setdefault keeps the first row).
//
//   vp_wide_validate       tensor.py:49-78 invariants (duplicates, batch >= 0,
//                          stride multiples) on wide rows
//   vp_wide_output_coords  conv.py:124-146: floor-div by the new stride (int64,
//                          Python floor semantics), unique rows in first-seen order
//   vp_wide_kernel_map     conv.py:149-183: per offset the pairs (in, out) with
//                          in == out + off * in_stride, ascending out rows, plus
//                          the dense nbr table (shared scan/emit with kmap.cu)
// Deterministic: every output is a function of the inputs only.
#include <algorithm>

#include "common.cuh"

namespace vp {

int map_scan_emit(const int32_t* nbr, const int32_t* n_out_dev, int64_t cap_out, int K, int32_t* counts,
                  int32_t* totals, int ntiles, int32_t* pair_in, int32_t* pair_out, int32_t* pair_ptr,
                  const uint32_t* masks, cudaStream_t st);

constexpr int kWideMaxD1 = 8;  // batch + up to 7 axes
constexpr int kWideTile = 128;  // output rows per probe tile (== kmap.cu kMapTile)
constexpr uint32_t kWideEmpty = 0xFFFFFFFFu;

struct WideOffsets {
  int64_t d[VP_MAX_OFFSETS * (kWideMaxD1 - 1)];  // off * in_stride per axis
};

__device__ __forceinline__ uint32_t wide_hash(const int64_t* r, int d1) {
  uint64_t h = 0x9E3779B97F4A7C15ull;
  for (int a = 0; a < d1; ++a) h = mix64(h ^ (uint64_t)r[a]);
  return (uint32_t)h;
}

__device__ __forceinline__ bool rows_equal(const int64_t* __restrict__ a, const int64_t* b, int d1) {
  for (int i = 0; i < d1; ++i)
    if (a[i] != b[i]) return false;
  return true;
}

// table[s] = row index (first occurrence of its tuple), kWideEmpty = free
__device__ __forceinline__ void wide_insert(uint32_t* t, uint32_t mask, const int64_t* __restrict__ rows, int d1,
                                            uint32_t i) {
  const int64_t* r = rows + (int64_t)i * d1;
  uint32_t s = wide_hash(r, d1) & mask;
  while (true) {
    const uint32_t prev = atomicCAS(&t[s], kWideEmpty, i);
    if (prev == kWideEmpty) return;
    if (rows_equal(rows + (int64_t)prev * d1, r, d1)) {
      atomicMin(&t[s], i);
      return;
    }
    s = (s + 1) & mask;
  }
}

__device__ __forceinline__ int wide_find(const uint32_t* __restrict__ t, uint32_t mask,
                                         const int64_t* __restrict__ rows, int d1, const int64_t* q) {
  uint32_t s = wide_hash(q, d1) & mask;
  while (true) {
    const uint32_t v = __ldg(t + s);
    if (v == kWideEmpty) return -1;
    if (rows_equal(rows + (int64_t)v * d1, q, d1)) return (int)v;
    s = (s + 1) & mask;
  }
}

__global__ void wide_clear_kernel(uint32_t* t, int64_t cap) {
  ::vp::pdl_begin();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap; i += (int64_t)gridDim.x * blockDim.x)
    t[i] = kWideEmpty;
}

__global__ void wide_insert_kernel(const int64_t* __restrict__ rows, int64_t n, int d1, uint32_t* t, uint32_t mask) {
  ::vp::pdl_begin();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    wide_insert(t, mask, rows, d1, (uint32_t)i);
}

// flags: 1 duplicate row, 2 negative batch, 4 axis not a multiple of the stride
__global__ void wide_check_kernel(const int64_t* __restrict__ rows, int64_t n, int d1, const uint32_t* __restrict__ t,
                                  uint32_t mask, const __grid_constant__ WideOffsets ts, int32_t* flags) {
  ::vp::pdl_begin();
  int f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t* r = rows + i * d1;
    if (r[0] < 0) f |= 2;
    for (int a = 1; a < d1; ++a)
      if (r[a] % ts.d[a - 1] != 0) f |= 4;
    if (wide_find(t, mask, rows, d1, r) != (int)i) f |= 1;
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

__device__ __forceinline__ int64_t floor_div64(int64_t a, int64_t b) {  // b > 0, Python //
  int64_t q = a / b;
  return (a % b != 0 && a < 0) ? q - 1 : q;
}

__global__ void wide_downsample_kernel(const int64_t* __restrict__ in, int64_t n, int d1,
                                       const __grid_constant__ WideOffsets step, int64_t* __restrict__ ds) {
  ::vp::pdl_begin();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * d1; e += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(e % d1);
    ds[e] = a == 0 ? in[e] : floor_div64(in[e], step.d[a - 1]) * step.d[a - 1];
  }
}

// keep[i] = row i is the first occurrence of its downsampled tuple; per-block counts
constexpr int kWideBlock = 1024;
__global__ void __launch_bounds__(kWideBlock)
wide_first_kernel(const int64_t* __restrict__ ds, int64_t n, int d1, const uint32_t* __restrict__ t, uint32_t mask,
                  int32_t* __restrict__ block_counts) {
  ::vp::pdl_begin();
  __shared__ int s_warp[kWideBlock / 32 + 1];
  const int64_t i = blockIdx.x * (int64_t)kWideBlock + threadIdx.x;
  const int keep = (i < n && wide_find(t, mask, ds, d1, ds + i * d1) == (int)i) ? 1 : 0;
  int tot;
  block_exclusive_scan<kWideBlock>(keep, s_warp, &tot);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = tot;
}

// single CTA: exclusive scan of the block counts -> block bases, n_out
__global__ void __launch_bounds__(kWideBlock)
wide_scan_kernel(int32_t* block_counts, int nblocks, int32_t* n_out_dev) {
  ::vp::pdl_begin();
  __shared__ int s_warp[kWideBlock / 32 + 1];
  __shared__ int s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < nblocks; base += kWideBlock) {
    const int i = base + threadIdx.x;
    const int v = i < nblocks ? block_counts[i] : 0;
    int tot;
    const int e = block_exclusive_scan<kWideBlock>(v, s_warp, &tot);
    if (i < nblocks) block_counts[i] = s_carry + e;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_out_dev = s_carry;
}

// ordered scatter of the kept rows (ascending first index = first-seen order)
__global__ void __launch_bounds__(kWideBlock)
wide_compact_kernel(const int64_t* __restrict__ ds, int64_t n, int d1, const uint32_t* __restrict__ t, uint32_t mask,
                    const int32_t* __restrict__ block_base, int64_t* __restrict__ out) {
  ::vp::pdl_begin();
  __shared__ int s_warp[kWideBlock / 32 + 1];
  const int64_t i = blockIdx.x * (int64_t)kWideBlock + threadIdx.x;
  const int keep = (i < n && wide_find(t, mask, ds, d1, ds + i * d1) == (int)i) ? 1 : 0;
  int tot;
  const int pos = block_exclusive_scan<kWideBlock>(keep, s_warp, &tot) + block_base[blockIdx.x];
  if (keep)
    for (int a = 0; a < d1; ++a) out[(int64_t)pos * d1 + a] = ds[i * d1 + a];
}

// one thread per output row: the K queries of the row, nbr + per-tile counts
__global__ void __launch_bounds__(kWideTile)
wide_probe_kernel(const int64_t* __restrict__ in, const int64_t* __restrict__ out, int64_t n_out, int d1,
                  const uint32_t* __restrict__ t, uint32_t mask, const __grid_constant__ WideOffsets offs, int K,
                  int32_t* __restrict__ nbr, int32_t* __restrict__ counts, int ntiles) {
  ::vp::pdl_begin();
  __shared__ int s_cnt[kWideTile / 32][VP_MAX_OFFSETS];
  const int tile = blockIdx.x;
  const int64_t u = (int64_t)tile * kWideTile + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool valid = u < n_out;
  int64_t r[kWideMaxD1], q[kWideMaxD1];
  for (int a = 0; a < d1; ++a) r[a] = valid ? out[u * d1 + a] : 0;
  for (int k = 0; k < K; ++k) {
    int v = -1;
    if (valid) {
      q[0] = r[0];
      for (int a = 1; a < d1; ++a) q[a] = r[a] + offs.d[k * (d1 - 1) + a - 1];
      v = wide_find(t, mask, in, d1, q);
      nbr[u * K + k] = v;
    }
    const unsigned m = __ballot_sync(0xffffffffu, v >= 0);
    if (lane == 0) s_cnt[warp][k] = __popc(m);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += kWideTile) {
    int c = 0;
#pragma unroll
    for (int w = 0; w < kWideTile / 32; ++w) c += s_cnt[w][k];
    counts[(int64_t)k * ntiles + tile] = c;
  }
}

static uint32_t wide_cap(int64_t n) {  // pow2 >= 2n + 2 (load <= 1/2)
  uint64_t c = 16;
  while (c < (uint64_t)(2 * n + 2)) c <<= 1;
  return (uint32_t)c;
}

static int wide_build(const int64_t* rows, int64_t n, int d1, uint32_t* t, uint32_t cap, cudaStream_t st) {
  ::vp::launch(wide_clear_kernel, (int)std::min<int64_t>(ceil_div(cap, 256), grid_cap(8)), 256, 0, st, t,
               (int64_t)cap);
  VP_CHECK_LAUNCH("wide_clear");
  if (n > 0) {
    ::vp::launch(wide_insert_kernel, (int)std::min<int64_t>(ceil_div(n, 256), grid_cap(8)), 256, 0, st, rows, n, d1,
                 t, cap - 1);
    VP_CHECK_LAUNCH("wide_insert");
  }
  return VP_OK;
}

}  // namespace vp

using namespace vp;

extern "C" {

size_t vp_wide_ws_bytes(int64_t n_in, int64_t n_out, int32_t D1, int32_t K) {
  Carver c(nullptr, 0);
  c.take<uint32_t>(wide_cap(std::max<int64_t>(n_in, 1)));
  c.take<int64_t>(std::max<int64_t>(n_in, 1) * std::max(D1, 1));  // downsampled rows
  c.take<int32_t>(ceil_div(std::max<int64_t>(n_in, 1), kWideBlock) + 1);
  const int64_t ntiles = ceil_div(std::max<int64_t>(n_out, 1), kWideTile);
  c.take<int32_t>(ntiles * std::max(K, 1));
  c.take<int32_t>(std::max(K, 1) + 1);
  return c.off;
}

int vp_wide_validate(const int64_t* rows, int64_t n, int32_t D1, const int64_t* tensor_stride, int32_t* flags,
                     void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(D1 >= 2 && D1 <= kWideMaxD1, VP_EVALIDATION, "wide coordinates: 1..7 axes");
  VP_REQUIRE(n < (1ll << 31) - 2, VP_EVALIDATION, "wide coordinates: too many rows");
  for (int a = 0; a + 1 < D1; ++a)
    VP_REQUIRE(tensor_stride[a] > 0, VP_EVALIDATION, "tensor_stride entries must be positive");
  if (n <= 0) return VP_OK;
  Carver c(ws, ws_bytes);
  const uint32_t cap = wide_cap(n);
  uint32_t* t = c.take<uint32_t>(cap);
  VP_REQUIRE(c.ok(), VP_EVALIDATION, "wide_validate: workspace too small");
  int r = wide_build(rows, n, D1, t, cap, st);
  if (r) return r;
  WideOffsets ts;
  for (int a = 0; a + 1 < D1; ++a) ts.d[a] = tensor_stride[a];
  ::vp::launch(wide_check_kernel, (int)std::min<int64_t>(ceil_div(n, 256), grid_cap(8)), 256, 0, st, rows, n, D1,
               (const uint32_t*)t, cap - 1, ts, flags);
  VP_CHECK_LAUNCH("wide_check");
  return VP_OK;
}

int vp_wide_output_coords(const int64_t* in, int64_t n, int32_t D1, const int64_t* step, int64_t* out,
                          int32_t* n_out_dev, void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(D1 >= 2 && D1 <= kWideMaxD1, VP_EVALIDATION, "wide coordinates: 1..7 axes");
  VP_REQUIRE(n < (1ll << 31) - 2, VP_EVALIDATION, "wide coordinates: too many rows");
  for (int a = 0; a + 1 < D1; ++a) VP_REQUIRE(step[a] > 0, VP_EVALIDATION, "stride entries must be positive");
  if (n <= 0) {
    cudaMemsetAsync(n_out_dev, 0, sizeof(int32_t), st);
    VP_CHECK_ASYNC("wide_output_coords(empty)");
    return VP_OK;
  }
  Carver c(ws, ws_bytes);
  const uint32_t cap = wide_cap(n);
  uint32_t* t = c.take<uint32_t>(cap);
  int64_t* ds = c.take<int64_t>(n * D1);
  const int nblocks = (int)ceil_div(n, kWideBlock);
  int32_t* bc = c.take<int32_t>(nblocks + 1);
  VP_REQUIRE(c.ok(), VP_EVALIDATION, "wide_output_coords: workspace too small");
  WideOffsets sd;
  for (int a = 0; a + 1 < D1; ++a) sd.d[a] = step[a];
  ::vp::launch(wide_downsample_kernel, (int)std::min<int64_t>(ceil_div(n * D1, 256), grid_cap(8)), 256, 0, st, in, n,
               D1, sd, ds);
  VP_CHECK_LAUNCH("wide_downsample");
  int r = wide_build(ds, n, D1, t, cap, st);
  if (r) return r;
  ::vp::launch(wide_first_kernel, nblocks, kWideBlock, 0, st, (const int64_t*)ds, n, D1, (const uint32_t*)t, cap - 1,
               bc);
  VP_CHECK_LAUNCH("wide_first");
  ::vp::launch(wide_scan_kernel, 1, kWideBlock, 0, st, bc, nblocks, n_out_dev);
  VP_CHECK_LAUNCH("wide_scan");
  ::vp::launch(wide_compact_kernel, nblocks, kWideBlock, 0, st, (const int64_t*)ds, n, D1, (const uint32_t*)t, cap - 1,
               (const int32_t*)bc, out);
  VP_CHECK_LAUNCH("wide_compact");
  return VP_OK;
}

int vp_wide_kernel_map(const int64_t* in, int64_t n_in, const int64_t* out, int64_t n_out, int32_t D1,
                       const int32_t* offsets_host, int32_t K, const int64_t* in_stride, int32_t* nbr,
                       int32_t* pair_in, int32_t* pair_out, int32_t* pair_ptr, void* ws, size_t ws_bytes,
                       vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(D1 >= 2 && D1 <= kWideMaxD1, VP_EVALIDATION, "wide coordinates: 1..7 axes");
  VP_REQUIRE(K >= 1 && K * (D1 - 1) <= VP_MAX_OFFSETS * (kWideMaxD1 - 1) && K <= VP_MAX_OFFSETS, VP_EVALIDATION,
             "kernel offset count out of range");
  VP_REQUIRE(pair_in && pair_out && pair_ptr, VP_EVALIDATION, "wide_kernel_map: pair outputs required");
  VP_REQUIRE(n_in < (1ll << 31) - 2 && n_out < (1ll << 31) - 2, VP_EVALIDATION, "wide coordinates: too many rows");
  Carver c(ws, ws_bytes);
  const uint32_t cap = wide_cap(std::max<int64_t>(n_in, 1));
  uint32_t* t = c.take<uint32_t>(cap);
  c.take<int64_t>(std::max<int64_t>(n_in, 1) * D1);
  c.take<int32_t>(ceil_div(std::max<int64_t>(n_in, 1), kWideBlock) + 1);
  const int ntiles = (int)ceil_div(std::max<int64_t>(n_out, 1), kWideTile);
  int32_t* counts = c.take<int32_t>((int64_t)ntiles * K);
  int32_t* totals = c.take<int32_t>(K + 1);
  VP_REQUIRE(c.ok(), VP_EVALIDATION, "wide_kernel_map: workspace too small");
  if (n_out <= 0) {
    cudaMemsetAsync(pair_ptr, 0, sizeof(int32_t) * (K + 1), st);
    VP_CHECK_ASYNC("wide_kernel_map(empty)");
    return VP_OK;
  }
  int r = wide_build(in, n_in, D1, t, cap, st);
  if (r) return r;
  WideOffsets offs;
  for (int k = 0; k < K; ++k)
    for (int a = 0; a + 1 < D1; ++a) offs.d[k * (D1 - 1) + a] = (int64_t)offsets_host[k * (D1 - 1) + a] * in_stride[a];
  ::vp::launch(wide_probe_kernel, ntiles, kWideTile, 0, st, in, out, n_out, D1, (const uint32_t*)t, cap - 1, offs, K,
               nbr, counts, ntiles);
  VP_CHECK_LAUNCH("wide_probe");
  return map_scan_emit(nbr, nullptr, n_out, K, counts, totals, ntiles, pair_in, pair_out, pair_ptr, nullptr, st);
}

}  // extern "C"
