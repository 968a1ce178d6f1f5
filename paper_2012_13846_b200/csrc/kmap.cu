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

constexpr int kMapTile = 128;  // output rows per tile (== threads per CTA)
constexpr int kMapSmemK = 32;  // neighbour tile staged in smem when K <= 32

struct Offsets {
  int32_t d[VP_MAX_OFFSETS * 3];
};

// Dense-grid coordinate index for bounded lattices (the training engine's
// levels: batch < B, axes in [0, R*s) on multiples of s): cell ->
// row (INT_MAX = empty).  A lookup is one 4-byte load with no probing, and
// the 27 neighbours of a row fall in 9 z-runs of 3 adjacent cells.
struct GridSpec {
  int32_t* cells;
  int B, R, s;
};
constexpr int32_t kGridEmpty = 0x7fffffff;

// lattice cell of a row (per axis, in units of s) or false when off-lattice
__device__ __forceinline__ bool grid_coords(const GridSpec& g, int4 r, int& cx, int& cy, int& cz) {
  if (r.x < 0 || r.x >= g.B || r.y < 0 || r.z < 0 || r.w < 0) return false;
  cx = r.y / g.s;
  cy = r.z / g.s;
  cz = r.w / g.s;
  return cx < g.R && cy < g.R && cz < g.R && cx * g.s == r.y && cy * g.s == r.z && cz * g.s == r.w;
}

__device__ __forceinline__ int grid_linear(const GridSpec& g, int b, int cx, int cy, int cz) {
  return ((b * g.R + cx) * g.R + cy) * g.R + cz;  // < 2^31: host caps B*R^3
}

__global__ void grid_set_kernel(const int4* __restrict__ c, const int32_t* n_dev, int64_t cap, GridSpec g, int clear) {
  ::vp::pdl_begin();
  const int n = load_count(n_dev, cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int4 r = c[i];
    int cx, cy, cz;
    if (grid_coords(g, r, cx, cy, cz)) g.cells[grid_linear(g, r.x, cx, cy, cz)] = clear ? kGridEmpty : (int32_t)i;
  }
}

// Internal map hash.  The slot layout of the map's private table is not
// semantic (only the rows found are), so instead of splitmix64 on the 64-bit
// key it mixes the two 32-bit halves of the packed key (kernels.py:75-78
// fields) with 32-bit multiplies: a handful of instructions per probe
// instead of two emulated 64-bit multiplies.
__device__ __forceinline__ uint32_t map_slot(uint32_t hi, uint32_t lo, uint32_t mask) {
  uint32_t h = lo * 0x9E3779B1u ^ (hi * 0x85EBCA77u + 0x165667B1u);
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  return h & mask;
}

// packed key halves: hi = batch << 16 | (x + 32768), lo = (y + 32768) << 16 | (z + 32768)
__device__ __forceinline__ bool pack_halves(int b, int x, int y, int z, uint32_t& hi, uint32_t& lo) {
  const uint32_t ux = (uint32_t)(x + kAxisBias), uy = (uint32_t)(y + kAxisBias), uz = (uint32_t)(z + kAxisBias);
  if ((uint32_t)b > (uint32_t)kBatchMax || ux > 0xFFFFu || uy > 0xFFFFu || uz > 0xFFFFu) return false;
  hi = ((uint32_t)b << 16) | ux;
  lo = (uy << 16) | uz;
  return true;
}

__global__ void map_insert_kernel(const int4* __restrict__ in, const int32_t* n_dev, int64_t cap_n,
                                  Slot* t, uint64_t cap) {
  ::vp::pdl_begin();
  int n = load_count(n_dev, cap_n);
  const uint32_t mask = (uint32_t)(cap - 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int4 r = in[i];
    uint32_t hi, lo;
    if (!pack_halves(r.x, r.y, r.z, r.w, hi, lo)) continue;  // unpackable rows are never found
    const unsigned long long key = ((unsigned long long)hi << 32) | lo;
    const unsigned int nrow = ~(unsigned int)i;
    if (key == kEmptyKey) {
      atomicMax(&t[cap].nrow, nrow);
      continue;
    }
    uint32_t s = map_slot(hi, lo, mask);
    while (true) {
      const unsigned long long prev = atomicCAS(&t[s].key, (unsigned long long)kEmptyKey, key);
      if (prev == kEmptyKey || prev == key) {
        atomicMax(&t[s].nrow, nrow);  // rows are unique (SparseTensor), so this is the row
        break;
      }
      s = (s + 1) & mask;
    }
  }
}

// kMapTPR threads per output row split the K probes (k = j, j + 8, ...), so a
// thread's chain of dependent hash walks is short and 1024 independent walks
// are in flight per CTA; hits are counted per (warp, k) with ballots masked
// to the lanes owning k.  For K <= 32 the [128, K] neighbour tile is staged
// in shared memory and written back fully coalesced.  counts[k*ntiles+tile].
constexpr int kMapTPR = 8;
constexpr int kProbeThreads = kMapTile * kMapTPR;  // 1024
constexpr int kProbeWarps = kProbeThreads / 32;

__global__ void __launch_bounds__(kProbeThreads, 2)
map_probe_kernel(const int4* __restrict__ out, const int32_t* n_out_dev, int64_t cap_out,
                 const Slot* __restrict__ t, uint64_t cap, const __grid_constant__ Offsets offs,
                 int K, int32_t* __restrict__ nbr, int32_t* counts, int ntiles) {
  ::vp::pdl_begin();
  __shared__ int s_nbr[kMapTile * (kMapSmemK + 1)];
  __shared__ unsigned short s_cnt[kProbeWarps][VP_MAX_OFFSETS];
  const int n_out = load_count(n_out_dev, cap_out);
  const int tile = blockIdx.x;
  const int64_t u0 = (int64_t)tile * kMapTile;
  if (u0 >= n_out) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row = tid / kMapTPR, j = tid % kMapTPR;
  const int rows = (n_out - u0) < kMapTile ? (int)(n_out - u0) : kMapTile;
  const bool valid = row < rows;
  const bool staged = K <= kMapSmemK;
  const int4 r = valid ? out[u0 + row] : make_int4(-1, 0, 0, 0);
  // Probe kMapBatch offsets at once: the first probe step of every key is
  // issued before any result is inspected (memory-level parallelism); the
  // rare collision chains are finished afterwards.
  constexpr int kMapBatch = 2;
  const uint32_t mask = (uint32_t)(cap - 1);
  for (int kb = 0; kb < K; kb += kMapTPR * kMapBatch) {
    uint32_t khi[kMapBatch], klo[kMapBatch], slot[kMapBatch];
    int v[kMapBatch];
    bool live[kMapBatch];
#pragma unroll
    for (int b = 0; b < kMapBatch; ++b) {
      const int k = kb + b * kMapTPR + j;
      live[b] = false;
      v[b] = -1;
      khi[b] = klo[b] = slot[b] = 0;
      // offsets arrive pre-multiplied by the input stride and clamped, so
      // the query stays in int32; out-of-range queries are plain misses
      // (kernels.py:135-148)
      if (valid && k < K && pack_halves(r.x, r.y + offs.d[3 * k], r.z + offs.d[3 * k + 1],
                                        r.w + offs.d[3 * k + 2], khi[b], klo[b])) {
        if ((khi[b] & klo[b]) == 0xFFFFFFFFu) {
          v[b] = (int)~t[cap].nrow;  // the one key equal to the empty marker
        } else {
          live[b] = true;
          slot[b] = map_slot(khi[b], klo[b], mask);
        }
      }
    }
    uint4 sv[kMapBatch];
#pragma unroll
    for (int b = 0; b < kMapBatch; ++b)
      if (live[b]) sv[b] = __ldg(reinterpret_cast<const uint4*>(t + slot[b]));
#pragma unroll
    for (int b = 0; b < kMapBatch; ++b) {
      if (!live[b]) continue;
      uint4 s4 = sv[b];
      uint32_t s = slot[b];
      while (true) {
        if (s4.x == klo[b] && s4.y == khi[b]) { v[b] = (int)~s4.z; break; }
        if ((s4.x & s4.y) == 0xFFFFFFFFu) break;  // empty slot
        s = (s + 1) & mask;
        s4 = __ldg(reinterpret_cast<const uint4*>(t + s));
      }
    }
#pragma unroll
    for (int b = 0; b < kMapBatch; ++b) {
      const int k0 = kb + b * kMapTPR;
      if (k0 >= K) break;
      const int k = k0 + j;
      if (k < K) {
        if (staged) s_nbr[row * (kMapSmemK + 1) + k] = v[b];
        else if (valid) nbr[(u0 + row) * K + k] = v[b];
      }
      const unsigned m = __ballot_sync(0xffffffffu, v[b] >= 0);
      if (lane < kMapTPR && k0 + lane < K) s_cnt[warp][k0 + lane] = (unsigned short)__popc(m & (0x01010101u << lane));
    }
  }
  __syncthreads();
  if (staged) {  // warp per row: K <= 32 contiguous ints, no division
    int32_t* dst = nbr + u0 * K;
    for (int rr = warp; rr < rows; rr += kProbeWarps)
      if (lane < K) dst[rr * K + lane] = s_nbr[rr * (kMapSmemK + 1) + lane];
  }
  for (int k = tid; k < K; k += kProbeThreads) {
    int c = 0;
#pragma unroll 8
    for (int w = 0; w < kProbeWarps; ++w) c += s_cnt[w][k];
    counts[(int64_t)k * ntiles + tile] = c;
  }
}

// Dense-grid probe: one thread per output row, offsets in batches of 9
// independent 4-byte loads (a 3x3x3 kernel = 3 batches, each 3 z-runs of 3
// adjacent cells).  Offsets arrive pre-scaled to cells (off * in_stride / s)
// with their linear cell delta, so a probe is 3 unsigned compares + 1 load.
struct GridOffsets {
  int32_t d[VP_MAX_OFFSETS * 3];
  int32_t lin[VP_MAX_OFFSETS];
};

__global__ void __launch_bounds__(kMapTile)
map_probe_grid_kernel(const int4* __restrict__ out, const int32_t* n_out_dev, int64_t cap_out, GridSpec g,
                      const __grid_constant__ GridOffsets offs, int K, int32_t* __restrict__ nbr, int32_t* counts,
                      int ntiles) {
  ::vp::pdl_begin();
  __shared__ int s_nbr[kMapTile * (kMapSmemK + 1)];
  __shared__ int s_cnt[kMapTile / 32][VP_MAX_OFFSETS];
  const int n_out = load_count(n_out_dev, cap_out);
  const int tile = blockIdx.x;
  const int64_t u0 = (int64_t)tile * kMapTile;
  if (u0 >= n_out) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows = (n_out - u0) < kMapTile ? (int)(n_out - u0) : kMapTile;
  const bool valid = tid < rows;
  const bool staged = K <= kMapSmemK;
  int cx = 0, cy = 0, cz = 0, base = 0;
  bool on = false;
  if (valid) {
    const int4 r = out[u0 + tid];
    on = grid_coords(g, r, cx, cy, cz);
    if (on) base = grid_linear(g, r.x, cx, cy, cz);
  }
  const unsigned R = (unsigned)g.R;
  constexpr int KB = 27;  // a whole 3^3 kernel's loads in flight at once (larger K loops)
  for (int kb = 0; kb < K; kb += KB) {
    int v[KB];
#pragma unroll
    for (int b = 0; b < KB; ++b) {
      const int k = kb + b;
      v[b] = kGridEmpty;
      if (on && k < K && (unsigned)(cx + offs.d[3 * k]) < R && (unsigned)(cy + offs.d[3 * k + 1]) < R &&
          (unsigned)(cz + offs.d[3 * k + 2]) < R)
        v[b] = __ldg(g.cells + base + offs.lin[k]);
    }
#pragma unroll
    for (int b = 0; b < KB; ++b) {
      const int k = kb + b;
      if (k >= K) break;
      const int x = v[b] == kGridEmpty ? -1 : v[b];
      if (staged) s_nbr[tid * (kMapSmemK + 1) + k] = x;
      else if (valid) nbr[(u0 + tid) * K + k] = x;
      const unsigned m = __ballot_sync(0xffffffffu, x >= 0);
      if (lane == 0) s_cnt[warp][k] = __popc(m);
    }
  }
  __syncthreads();
  if (staged) {  // warp per row: K <= 32 contiguous ints, no division
    int32_t* dst = nbr + u0 * K;
    for (int rr = warp; rr < rows; rr += kMapTile / 32)
      if (lane < K) dst[rr * K + lane] = s_nbr[rr * (kMapSmemK + 1) + lane];
  }
  for (int k = tid; k < K; k += kMapTile) {
    int c = 0;
#pragma unroll
    for (int w = 0; w < kMapTile / 32; ++w) c += s_cnt[w][k];
    counts[(int64_t)k * ntiles + tile] = c;
  }
}

// one CTA per offset: exclusive scan over the tiles' counts, total[k].
__global__ void __launch_bounds__(1024)
map_scan_kernel(int32_t* counts, const int32_t* n_out_dev, int64_t cap_out, int ntiles_cap,
                int32_t* totals) {
  ::vp::pdl_begin();
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

// per tile: for each offset, ordered compaction of the hit rows (ascending
// out row == conv.py:181 flatnonzero order) with warp ballots; the per-warp
// hit counts of all offsets are gathered first so the loop has no barriers.
__global__ void __launch_bounds__(kMapTile)
map_emit_kernel(const int32_t* __restrict__ nbr, const int32_t* n_out_dev, int64_t cap_out, int K,
                const int32_t* __restrict__ counts, const int32_t* __restrict__ totals, int ntiles_cap,
                int32_t* __restrict__ pair_in, int32_t* __restrict__ pair_out, int32_t* pair_ptr) {
  ::vp::pdl_begin();
  __shared__ int s_nbr[kMapTile * (kMapSmemK + 1)];
  __shared__ int s_w[kMapTile / 32][VP_MAX_OFFSETS];
  __shared__ int s_base[VP_MAX_OFFSETS + 1];
  __shared__ int s_tot[VP_MAX_OFFSETS];
  const int n_out = load_count(n_out_dev, cap_out);
  const int tile = blockIdx.x;
  const int64_t u0 = (int64_t)tile * kMapTile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // all global loads of the offset bases issued in parallel, then a serial
  // prefix over K values in shared memory
  for (int k = tid; k < K; k += kMapTile) s_tot[k] = __ldg(totals + k);
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int k = 0; k < K; ++k) {
      s_base[k] = acc;
      acc += s_tot[k];
    }
    s_base[K] = acc;
    if (tile == 0)
      for (int k = 0; k <= K; ++k) pair_ptr[k] = s_base[k];
  }
  if (u0 >= n_out) return;
  for (int k = tid; k < K; k += kMapTile) s_w[0][k] = __ldg(counts + (int64_t)k * ntiles_cap + tile);
  __syncthreads();  // thread 0 is done reading s_tot (totals)
  for (int k = tid; k < K; k += kMapTile) s_tot[k] = s_w[0][k];
  const int rows = (n_out - u0) < kMapTile ? (int)(n_out - u0) : kMapTile;
  const bool staged = K <= kMapSmemK;
  if (staged) {
    const int32_t* src = nbr + u0 * K;
    for (int e = tid; e < rows * K; e += kMapTile) {
      const int rr = e / K, k = e - rr * K;
      s_nbr[rr * (kMapSmemK + 1) + k] = src[e];
    }
  }
  __syncthreads();
  const bool valid = tid < rows;
  auto nb = [&](int k) -> int {
    if (!valid) return -1;
    return staged ? s_nbr[tid * (kMapSmemK + 1) + k] : nbr[(u0 + tid) * K + k];
  };
  for (int k = 0; k < K; ++k) {
    const unsigned m = __ballot_sync(0xffffffffu, nb(k) >= 0);
    if (lane == 0) s_w[warp][k] = __popc(m);
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int k = 0; k < K; ++k) {
    const int v = nb(k);
    const unsigned m = __ballot_sync(0xffffffffu, v >= 0);
    if (v >= 0) {
      int before = 0;
#pragma unroll
      for (int w = 0; w < kMapTile / 32; ++w) before += (w < warp) ? s_w[w][k] : 0;
      const int pos = s_base[k] + s_tot[k] + before + __popc(m & lt);
      pair_in[pos] = v;
      pair_out[pos] = (int32_t)(u0 + tid);
    }
  }
}

__global__ void map_inverse_kernel(const int32_t* __restrict__ nbr, const int32_t* n_out_dev,
                                   int64_t cap_out, int K, int32_t* __restrict__ inv) {
  ::vp::pdl_begin();
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

namespace vp {
// per-offset scan of the tile counts + ordered pair emission (shared by the
// hash, dense-grid and brick probes)
int map_scan_emit(const int32_t* nbr, const int32_t* n_out_dev, int64_t cap_out, int K, int32_t* counts,
                  int32_t* totals, int ntiles, int32_t* pair_in, int32_t* pair_out, int32_t* pair_ptr,
                  cudaStream_t st) {
  ::vp::launch(map_scan_kernel, K, 1024, 0, st, counts, n_out_dev, cap_out, ntiles, totals);
  VP_CHECK_LAUNCH("map_scan");
  ::vp::launch(map_emit_kernel, ntiles, kMapTile, 0, st, nbr, n_out_dev, cap_out, K, (const int32_t*)counts,
               (const int32_t*)totals, ntiles, pair_in, pair_out, pair_ptr);
  VP_CHECK_LAUNCH("map_emit");
  return VP_OK;
}
}  // namespace vp

using namespace vp;

extern "C" {

size_t vp_kernel_map_ws_bytes(int64_t cap_in, int64_t cap_out, int32_t K) {
  Carver c(nullptr, 0);
  c.take<Slot>(hash_cap_internal(cap_in) + 1);
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
  uint64_t cap = hash_cap_internal(cap_in);
  Slot* t = c.take<Slot>(cap + 1);
  int ntiles = (int)ceil_div(std::max<int64_t>(cap_out, 1), kMapTile);
  int32_t* counts = c.take<int32_t>((int64_t)ntiles * K);
  int32_t* totals = c.take<int32_t>(K + 1);
  VP_REQUIRE(c.ok(), VP_EVALIDATION, "kernel_map: workspace too small");
  Offsets offs;
  memset(&offs, 0, sizeof(offs));
  for (int k = 0; k < K; ++k)
    for (int a = 0; a < 3; ++a) {
      // off * stride, clamped: anything beyond +-2^20 misses like +-2^20 does
      const int64_t d = (int64_t)offsets_host[3 * k + a] * in_stride[a];
      offs.d[3 * k + a] = (int32_t)std::max<int64_t>(std::min<int64_t>(d, 1 << 20), -(1 << 20));
    }
  int r = hash_clear(t, cap, st);
  if (r) return r;
  if (cap_in > 0) {
    int blocks = (int)std::min<int64_t>(ceil_div(cap_in, 256), grid_cap(8));
    ::vp::launch(map_insert_kernel, blocks, 256, 0, st, (const int4*)in, n_in_dev, cap_in, t, cap);
    VP_CHECK_LAUNCH("map_insert");
  }
  if (cap_out <= 0) {
    if (pair_ptr) cudaMemsetAsync(pair_ptr, 0, sizeof(int32_t) * (K + 1), st);
    VP_CHECK_ASYNC("kernel_map(empty)");
    return VP_OK;
  }
  ::vp::launch(map_probe_kernel, ntiles, kProbeThreads, 0, st, (const int4*)out, n_out_dev, cap_out, t, cap, offs, K,
                                                   nbr, counts, ntiles);
  VP_CHECK_LAUNCH("map_probe");
  if (pair_in) {
    ::vp::launch(map_scan_kernel, K, 1024, 0, st, counts, n_out_dev, cap_out, ntiles, totals);
    VP_CHECK_LAUNCH("map_scan");
    ::vp::launch(map_emit_kernel, ntiles, kMapTile, 0, st, nbr, n_out_dev, cap_out, K, counts, totals, ntiles,
                                                     pair_in, pair_out, pair_ptr);
    VP_CHECK_LAUNCH("map_emit");
  }
  return VP_OK;
}

int vp_grid_set(const int32_t* coords, const int32_t* n_dev, int64_t cap, int32_t* cells, int32_t B, int32_t R,
                int32_t s, int32_t clear, vp_stream_t stream) {
  VP_REQUIRE(B >= 1 && R >= 1 && s >= 1, VP_EVALIDATION, "grid: extents must be positive");
  VP_REQUIRE((int64_t)B * R * R * R < (1ll << 31), VP_EVALIDATION, "grid: B*R^3 must be < 2^31 cells");
  if (cap <= 0) return VP_OK;
  int blocks = (int)std::min<int64_t>(ceil_div(cap, 256), grid_cap(8));
  ::vp::launch(grid_set_kernel, blocks, 256, 0, (cudaStream_t)stream, (const int4*)coords, n_dev, cap, GridSpec{cells, B, R, s},
                                                          clear);
  VP_CHECK_LAUNCH("grid_set");
  return VP_OK;
}

size_t vp_kernel_map_grid_ws_bytes(int64_t cap_out, int32_t K) {
  Carver c(nullptr, 0);
  int64_t ntiles = ceil_div(std::max<int64_t>(cap_out, 1), kMapTile);
  c.take<int32_t>(ntiles * K);
  c.take<int32_t>(K + 1);
  return c.off;
}

int vp_kernel_map_grid(const int32_t* cells, int32_t B, int32_t R, int32_t s, const int32_t* out,
                       const int32_t* n_out_dev, int64_t cap_out, const int32_t* offsets_host, int32_t K,
                       const int32_t* in_stride, int32_t* nbr, int32_t* pair_in, int32_t* pair_out, int32_t* pair_ptr,
                       void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(K >= 1 && K <= VP_MAX_OFFSETS, VP_EVALIDATION, "kernel offset count out of range");
  VP_REQUIRE(pair_in && pair_out && pair_ptr, VP_EVALIDATION, "kernel_map_grid: pair outputs required");
  VP_REQUIRE(B >= 1 && R >= 1 && s >= 1, VP_EVALIDATION, "grid: extents must be positive");
  Carver c(ws, ws_bytes);
  int ntiles = (int)ceil_div(std::max<int64_t>(cap_out, 1), kMapTile);
  int32_t* counts = c.take<int32_t>((int64_t)ntiles * K);
  int32_t* totals = c.take<int32_t>(K + 1);
  VP_REQUIRE(c.ok(), VP_EVALIDATION, "kernel_map_grid: workspace too small");
  VP_REQUIRE((int64_t)B * R * R * R < (1ll << 31), VP_EVALIDATION, "grid: B*R^3 must be < 2^31 cells");
  for (int a = 0; a < 3; ++a)
    VP_REQUIRE(in_stride[a] >= 1 && in_stride[a] % s == 0, VP_EVALIDATION,
               "kernel_map_grid: in_stride must be a multiple of the grid spacing");
  GridOffsets offs;
  memset(&offs, 0, sizeof(offs));
  for (int k = 0; k < K; ++k) {
    int dc[3];
    for (int a = 0; a < 3; ++a) {
      const int64_t d = (int64_t)offsets_host[3 * k + a] * (in_stride[a] / s);
      // beyond the lattice in either direction: every query misses
      dc[a] = (int)std::max<int64_t>(std::min<int64_t>(d, R), -(int64_t)R);
      offs.d[3 * k + a] = dc[a];
    }
    offs.lin[k] = (dc[0] * R + dc[1]) * R + dc[2];
  }
  if (cap_out <= 0) {
    cudaMemsetAsync(pair_ptr, 0, sizeof(int32_t) * (K + 1), st);
    VP_CHECK_ASYNC("kernel_map_grid(empty)");
    return VP_OK;
  }
  ::vp::launch(map_probe_grid_kernel, ntiles, kMapTile, 0, st, (const int4*)out, n_out_dev, cap_out,
                                                     GridSpec{const_cast<int32_t*>(cells), B, R, s}, offs, K, nbr,
                                                     counts, ntiles);
  VP_CHECK_LAUNCH("map_probe_grid");
  return map_scan_emit(nbr, n_out_dev, cap_out, K, counts, totals, ntiles, pair_in, pair_out, pair_ptr, st);
}

int vp_kernel_map_inverse(const int32_t* nbr, const int32_t* n_out_dev, int64_t cap_out, int32_t K,
                          int32_t* inv, int64_t cap_in, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (cap_in > 0) cudaMemsetAsync(inv, 0xff, sizeof(int32_t) * cap_in * K, st);
  VP_CHECK_ASYNC("kernel_map_inverse(memset)");
  if (cap_out > 0) {
    int blocks = (int)std::min<int64_t>(ceil_div(cap_out * K, 256), grid_cap(16));
    ::vp::launch(map_inverse_kernel, blocks, 256, 0, st, nbr, n_out_dev, cap_out, K, inv);
    VP_CHECK_LAUNCH("kernel_map_inverse");
  }
  return VP_OK;
}

}  // extern "C"
