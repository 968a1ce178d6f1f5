// Kernel-map construction (conv.py:149-183) on sm_100a.
//
//   1. hash over the input rows (rows are unique: SparseTensor invariant);
//   2. probe: every (output row u, offset k) pair, flat-indexed u*K+k so the
//      neighbour-table writes are fully coalesced; each tile of 256 output
//      rows also counts its hits per offset;
//   3. per-offset exclusive scan of the tile counts (one CTA per offset);
//   4. emit: per tile, per offset, warp-ballot compaction of the hit rows in
//      ASCENDING out-row order -> pair lists bit-exact with KernelMap.pairs
//      (conv.py:176-182: rows[hit], flatnonzero(hit)).
#include "common.cuh"

namespace vp {

constexpr int kMapTile = 256;  // output rows per tile (== threads per CTA)

struct Offsets {
  int32_t d[VP_MAX_OFFSETS * 3];
};

__global__ void map_insert_kernel(const int4* __restrict__ in, const int32_t* n_dev, int64_t cap_n,
                                  Slot* t, uint64_t cap) {
  int n = load_count(n_dev, cap_n);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int4 r = in[i];
    hash_insert(t, cap, pack_key(r.x, r.y, r.z, r.w), (int)i);
  }
}

// grid: one CTA per tile of kMapTile output rows.  counts[k * ntiles + tile].
__global__ void __launch_bounds__(kMapTile)
map_probe_kernel(const int4* __restrict__ out, const int32_t* n_out_dev, int64_t cap_out,
                 const Slot* __restrict__ t, uint64_t cap, const __grid_constant__ Offsets offs,
                 int K, int sx, int sy, int sz, int32_t* __restrict__ nbr, int32_t* counts,
                 int ntiles) {
  extern __shared__ int smem[];
  int4* s_rows = reinterpret_cast<int4*>(smem);         // kMapTile rows
  int* s_cnt = smem + kMapTile * 4;                     // K counters
  const int n_out = load_count(n_out_dev, cap_out);
  const int tile = blockIdx.x;
  const int64_t u0 = (int64_t)tile * kMapTile;
  if (u0 >= n_out) return;
  const int rows = (n_out - u0) < kMapTile ? (int)(n_out - u0) : kMapTile;
  if (threadIdx.x < rows) s_rows[threadIdx.x] = out[u0 + threadIdx.x];
  for (int k = threadIdx.x; k < K; k += kMapTile) s_cnt[k] = 0;
  __syncthreads();
  const int total = rows * K;
  int32_t* dst = nbr + u0 * K;
  for (int e = threadIdx.x; e < total; e += kMapTile) {
    int u = e / K, k = e - u * K;
    int4 r = s_rows[u];
    long long qx = (long long)r.y + (long long)offs.d[3 * k] * sx;
    long long qy = (long long)r.z + (long long)offs.d[3 * k + 1] * sy;
    long long qz = (long long)r.w + (long long)offs.d[3 * k + 2] * sz;
    int v = -1;
    // out-of-range queries are plain misses (kernels.py:135-148)
    if (packable64(r.x, qx, qy, qz)) v = hash_find(t, cap, pack_key(r.x, (int)qx, (int)qy, (int)qz));
    dst[e] = v;
    if (v >= 0) atomicAdd(&s_cnt[k], 1);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += kMapTile) counts[(int64_t)k * ntiles + tile] = s_cnt[k];
}

// one CTA per offset: exclusive scan over the tiles' counts, total[k].
__global__ void __launch_bounds__(1024)
map_scan_kernel(int32_t* counts, const int32_t* n_out_dev, int64_t cap_out, int ntiles_cap,
                int32_t* totals) {
  __shared__ int s_warp[1024 / 32 + 1];
  __shared__ int s_carry;
  const int n_out = load_count(n_out_dev, cap_out);
  const int ntiles = (int)((n_out + kMapTile - 1) / kMapTile);
  int32_t* c = counts + (int64_t)blockIdx.x * ntiles_cap;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < ntiles; base += 1024) {
    int i = base + threadIdx.x;
    int v = i < ntiles ? c[i] : 0, tot;
    int e = block_exclusive_scan<1024>(v, s_warp, &tot);
    if (i < ntiles) c[i] = s_carry + e;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = s_carry;
}

// per tile: for each offset, ordered compaction of hit rows.
__global__ void __launch_bounds__(kMapTile)
map_emit_kernel(const int32_t* __restrict__ nbr, const int32_t* n_out_dev, int64_t cap_out, int K,
                const int32_t* __restrict__ counts, const int32_t* __restrict__ totals, int ntiles_cap,
                int32_t* __restrict__ pair_in, int32_t* __restrict__ pair_out, int32_t* pair_ptr) {
  extern __shared__ int smem[];
  int* s_base = smem;                 // K+1 offset bases
  int* s_warp = smem + VP_MAX_OFFSETS + 1;  // kMapTile/32
  const int n_out = load_count(n_out_dev, cap_out);
  const int tile = blockIdx.x;
  const int64_t u0 = (int64_t)tile * kMapTile;
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int k = 0; k < K; ++k) {
      s_base[k] = acc;
      acc += totals[k];
    }
    s_base[K] = acc;
    if (tile == 0)
      for (int k = 0; k <= K; ++k) pair_ptr[k] = s_base[k];
  }
  __syncthreads();
  if (u0 >= n_out) return;
  const int64_t u = u0 + threadIdx.x;
  const bool valid = u < n_out;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int32_t* row = nbr + u * K;
  for (int k = 0; k < K; ++k) {
    int v = valid ? row[k] : -1;
    unsigned m = __ballot_sync(0xffffffffu, v >= 0);
    if (lane == 0) s_warp[warp] = __popc(m);
    __syncthreads();
    int before = 0;
#pragma unroll
    for (int w = 0; w < kMapTile / 32; ++w) before += (w < warp) ? s_warp[w] : 0;
    if (v >= 0) {
      int pos = s_base[k] + counts[(int64_t)k * ntiles_cap + tile] + before +
                __popc(m & ((1u << lane) - 1u));
      pair_in[pos] = v;
      pair_out[pos] = (int32_t)u;
    }
    __syncthreads();
  }
}

__global__ void map_inverse_kernel(const int32_t* __restrict__ nbr, const int32_t* n_out_dev,
                                   int64_t cap_out, int K, int32_t* __restrict__ inv) {
  const int n_out = load_count(n_out_dev, cap_out);
  const int64_t total = (int64_t)n_out * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int v = nbr[e];
    if (v >= 0) {
      int64_t u = e / K;
      int k = (int)(e - u * K);
      inv[(int64_t)v * K + k] = (int32_t)u;  // unique per (v,k): in rows unique per offset
    }
  }
}

}  // namespace vp

using namespace vp;

extern "C" {

size_t vp_kernel_map_ws_bytes(int64_t cap_in, int64_t cap_out, int32_t K) {
  Carver c(nullptr, 0);
  c.take<Slot>(hash_cap_for(cap_in) + 1);
  int64_t ntiles = ceil_div(std::max<int64_t>(cap_out, 1), kMapTile);
  c.take<int32_t>(ntiles * K);
  c.take<int32_t>(K + 1);
  return c.off;
}

int vp_kernel_map(const int32_t* in, const int32_t* n_in_dev, int64_t cap_in, const int32_t* out,
                  const int32_t* n_out_dev, int64_t cap_out, const int32_t* offsets_host, int32_t K,
                  const int32_t* in_stride, int32_t* nbr, int32_t* pair_in, int32_t* pair_out,
                  int32_t* pair_ptr, void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(K >= 1 && K <= VP_MAX_OFFSETS, VP_EVALIDATION, "kernel offset count out of range");
  VP_REQUIRE((pair_in == nullptr) == (pair_out == nullptr) && (pair_in == nullptr || pair_ptr),
             VP_EVALIDATION, "pair_in/pair_out/pair_ptr must be given together");
  Carver c(ws, ws_bytes);
  uint64_t cap = hash_cap_for(cap_in);
  Slot* t = c.take<Slot>(cap + 1);
  int ntiles = (int)ceil_div(std::max<int64_t>(cap_out, 1), kMapTile);
  int32_t* counts = c.take<int32_t>((int64_t)ntiles * K);
  int32_t* totals = c.take<int32_t>(K + 1);
  VP_REQUIRE(c.ok(), VP_EVALIDATION, "kernel_map: workspace too small");
  Offsets offs;
  memset(&offs, 0, sizeof(offs));
  memcpy(offs.d, offsets_host, sizeof(int32_t) * 3 * K);
  int r = hash_clear(t, cap, st);
  if (r) return r;
  if (cap_in > 0) {
    int blocks = (int)std::min<int64_t>(ceil_div(cap_in, 256), kNumSMs * 8);
    map_insert_kernel<<<blocks, 256, 0, st>>>((const int4*)in, n_in_dev, cap_in, t, cap);
    VP_CHECK_LAUNCH("map_insert");
  }
  if (cap_out <= 0) {
    if (pair_ptr) cudaMemsetAsync(pair_ptr, 0, sizeof(int32_t) * (K + 1), st);
    VP_CHECK_ASYNC("kernel_map(empty)");
    return VP_OK;
  }
  size_t smem = kMapTile * 16 + K * 4;
  map_probe_kernel<<<ntiles, kMapTile, smem, st>>>((const int4*)out, n_out_dev, cap_out, t, cap, offs, K,
                                                   in_stride[0], in_stride[1], in_stride[2], nbr, counts,
                                                   ntiles);
  VP_CHECK_LAUNCH("map_probe");
  if (pair_in) {
    map_scan_kernel<<<K, 1024, 0, st>>>(counts, n_out_dev, cap_out, ntiles, totals);
    VP_CHECK_LAUNCH("map_scan");
    size_t smem2 = (VP_MAX_OFFSETS + 1 + kMapTile / 32) * 4;
    map_emit_kernel<<<ntiles, kMapTile, smem2, st>>>(nbr, n_out_dev, cap_out, K, counts, totals, ntiles,
                                                     pair_in, pair_out, pair_ptr);
    VP_CHECK_LAUNCH("map_emit");
  }
  return VP_OK;
}

int vp_kernel_map_inverse(const int32_t* nbr, const int32_t* n_out_dev, int64_t cap_out, int32_t K,
                          int32_t* inv, int64_t cap_in, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (cap_in > 0) cudaMemsetAsync(inv, 0xff, sizeof(int32_t) * cap_in * K, st);
  VP_CHECK_ASYNC("kernel_map_inverse(memset)");
  if (cap_out > 0) {
    int blocks = (int)std::min<int64_t>(ceil_div(cap_out * K, 256), kNumSMs * 16);
    map_inverse_kernel<<<blocks, 256, 0, st>>>(nbr, n_out_dev, cap_out, K, inv);
    VP_CHECK_LAUNCH("kernel_map_inverse");
  }
  return VP_OK;
}

}  // extern "C"
