// Two-level ("brick") coordinate index for the kernel map (conv.py:149-183).
//
// The dense lattice (kmap.cu, vp_grid_set) spends 4 bytes on every cell of
// B * R^3; at C5 (256 clouds at 128^3: 2.1 GB) its random probes miss L2 and
// go to DRAM, ~12x the map's algorithmic bytes.  Surface clouds occupy a
// thin shell, so the lattice is cut into 4^3 bricks: a coarse table
// (B * ceil(R/4)^3 int32, 64x smaller) holds a brick id for occupied bricks
// only, and each brick is 64 int32 cells (256 B) in a pool.  A probe is one
// coarse load plus one cell load, both L2-resident at every config; a
// row's 27 neighbours touch at most 8 bricks.
//
// Build (no spin-waits): mark (atomicMin of the row index into the coarse
// cell) -> assign (the minimum row of each brick takes a pool slot,
// atomicAdd; ids are arbitrary but only the cells' row values are ever
// observed, so maps stay deterministic) -> fill (each row writes its cell).
// The clear pass walks the allocated bricks, empties their 64 cells and
// their coarse entry, and resets the pool counter: the index is reusable
// with no full-size memset.
#include <algorithm>
#include <cstring>

#include "common.cuh"

namespace vp {

constexpr int32_t kBrickEmpty = 0x7f7f7f7f;  // memset(0x7f)-able; above any row index

struct BrickSpec {
  int32_t* coarse;   // [B * Rc^3]: kBrickEmpty | min row (during build) | -(id + 1)
  int32_t* bricks;   // [pool * 64]: row or kBrickEmpty
  int32_t* owner;    // [pool]: coarse cell of each allocated brick (for the clear)
  int32_t* counter;  // [1]: allocated bricks
  int B, R, s, Rc;
};

struct BrickOffsets {
  int32_t d[VP_MAX_OFFSETS * 3];
};

__device__ __forceinline__ bool brick_cell(const BrickSpec& g, int4 r, int& cx, int& cy, int& cz) {
  if (r.x < 0 || r.x >= g.B || r.y < 0 || r.z < 0 || r.w < 0) return false;
  cx = r.y / g.s;
  cy = r.z / g.s;
  cz = r.w / g.s;
  return cx < g.R && cy < g.R && cz < g.R && cx * g.s == r.y && cy * g.s == r.z && cz * g.s == r.w;
}
__device__ __forceinline__ int brick_coarse(const BrickSpec& g, int b, int cx, int cy, int cz) {
  return ((b * g.Rc + (cx >> 2)) * g.Rc + (cy >> 2)) * g.Rc + (cz >> 2);
}
__device__ __forceinline__ int brick_local(int cx, int cy, int cz) { return ((cx & 3) * 4 + (cy & 3)) * 4 + (cz & 3); }

__global__ void brick_mark_kernel(const int4* __restrict__ c, const int32_t* n_dev, int64_t cap, BrickSpec g) {
  ::vp::pdl_begin();
  const int n = load_count(n_dev, cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int cx, cy, cz;
    if (brick_cell(g, c[i], cx, cy, cz)) atomicMin(&g.coarse[brick_coarse(g, c[i].x, cx, cy, cz)], (int32_t)i);
  }
}

__global__ void brick_assign_kernel(const int4* __restrict__ c, const int32_t* n_dev, int64_t cap, BrickSpec g) {
  ::vp::pdl_begin();
  const int n = load_count(n_dev, cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int cx, cy, cz;
    const int4 r = c[i];
    if (!brick_cell(g, r, cx, cy, cz)) continue;
    const int cl = brick_coarse(g, r.x, cx, cy, cz);
    if (g.coarse[cl] == (int32_t)i) {  // this brick's minimum row allocates it (one writer per brick)
      const int id = atomicAdd(g.counter, 1);
      g.owner[id] = cl;
      g.coarse[cl] = -(id + 1);
    }
  }
}

__global__ void brick_fill_kernel(const int4* __restrict__ c, const int32_t* n_dev, int64_t cap, BrickSpec g) {
  ::vp::pdl_begin();
  const int n = load_count(n_dev, cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int cx, cy, cz;
    const int4 r = c[i];
    if (!brick_cell(g, r, cx, cy, cz)) continue;
    const int id = -g.coarse[brick_coarse(g, r.x, cx, cy, cz)] - 1;
    g.bricks[(int64_t)id * 64 + brick_local(cx, cy, cz)] = (int32_t)i;
  }
}

// empty every allocated brick (64 cells, warp-wide) and its coarse entry
__global__ void brick_clear_kernel(BrickSpec g) {
  ::vp::pdl_begin();
  const int nb = *g.counter;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int id = warp; id < nb; id += nw) {
    g.bricks[(int64_t)id * 64 + lane] = kBrickEmpty;
    g.bricks[(int64_t)id * 64 + 32 + lane] = kBrickEmpty;
    if (lane == 0) g.coarse[g.owner[id]] = kBrickEmpty;
  }
}

__global__ void brick_reset_counter_kernel(int32_t* counter) {
  ::vp::pdl_begin();
  *counter = 0;
}

// Probe: one thread per output row; all K coarse loads are issued first,
// then all K cell loads (two rounds of independent L2 hits).  Same nbr /
// per-tile counts layout as map_probe_grid_kernel, so map_scan + map_emit
// follow unchanged.
constexpr int kBrickTile = 128;
constexpr int kBrickSmemK = 32;

__global__ void __launch_bounds__(kBrickTile)
map_probe_brick_kernel(const int4* __restrict__ out, const int32_t* n_out_dev, int64_t cap_out, BrickSpec g,
                       const __grid_constant__ BrickOffsets offs, int K, int32_t* __restrict__ nbr, int32_t* counts,
                       int ntiles, uint32_t* __restrict__ masks) {
  ::vp::pdl_begin();
  __shared__ int s_nbr[kBrickTile * (kBrickSmemK + 1)];
  __shared__ int s_cnt[kBrickTile / 32][VP_MAX_OFFSETS];
  const int n_out = load_count(n_out_dev, cap_out);
  const int tile = blockIdx.x;
  const int64_t u0 = (int64_t)tile * kBrickTile;
  if (u0 >= n_out) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows = (n_out - u0) < kBrickTile ? (int)(n_out - u0) : kBrickTile;
  const bool valid = tid < rows;
  const bool staged = K <= kBrickSmemK;
  int cx = 0, cy = 0, cz = 0, b = 0;
  bool on = false;
  if (valid) {
    const int4 r = out[u0 + tid];
    on = brick_cell(g, r, cx, cy, cz);
    b = r.x;
  }
  const unsigned R = (unsigned)g.R;
  constexpr int KB = 27;
  uint32_t hitm = 0;
  for (int kb = 0; kb < K; kb += KB) {
    int cid[KB], loc[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      const int k = kb + j;
      cid[j] = kBrickEmpty;
      loc[j] = 0;
      if (on && k < K) {
        const int qx = cx + offs.d[3 * k], qy = cy + offs.d[3 * k + 1], qz = cz + offs.d[3 * k + 2];
        if ((unsigned)qx < R && (unsigned)qy < R && (unsigned)qz < R) {
          cid[j] = __ldg(g.coarse + brick_coarse(g, b, qx, qy, qz));
          loc[j] = brick_local(qx, qy, qz);
        }
      }
    }
    int v[KB];
#pragma unroll
    for (int j = 0; j < KB; ++j)
      v[j] = cid[j] < 0 ? __ldg(g.bricks + (int64_t)(-cid[j] - 1) * 64 + loc[j]) : kBrickEmpty;
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      const int k = kb + j;
      if (k >= K) break;
      const int x = v[j] == kBrickEmpty ? -1 : v[j];
      if (k < 32 && x >= 0) hitm |= 1u << k;
      if (staged) s_nbr[tid * (kBrickSmemK + 1) + k] = x;
      else if (valid) nbr[(u0 + tid) * K + k] = x;
      const unsigned m = __ballot_sync(0xffffffffu, x >= 0);
      if (lane == 0) s_cnt[warp][k] = __popc(m);
    }
  }
  __syncthreads();
  if (staged) {  // warp per row: K <= 32 contiguous ints
    int32_t* dst = nbr + u0 * K;
    for (int rr = warp; rr < rows; rr += kBrickTile / 32)
      if (lane < K) dst[rr * K + lane] = s_nbr[rr * (kBrickSmemK + 1) + lane];
  }
  if (masks && valid) masks[u0 + tid] = hitm;
  for (int k = tid; k < K; k += kBrickTile) {
    int c = 0;
#pragma unroll
    for (int w = 0; w < kBrickTile / 32; ++w) c += s_cnt[w][k];
    counts[(int64_t)k * ntiles + tile] = c;
  }
}

// defined in kmap.cu (shared with the dense-grid and hash paths)
int map_scan_emit(const int32_t* nbr, const int32_t* n_out_dev, int64_t cap_out, int K, int32_t* counts,
                  int32_t* totals, int ntiles, int32_t* pair_in, int32_t* pair_out, int32_t* pair_ptr,
                  const uint32_t* masks, cudaStream_t st);

}  // namespace vp

using namespace vp;

extern "C" {

int64_t vp_brick_pool(int64_t cap, int32_t B, int32_t R) {
  const int64_t Rc = (R + 3) / 4;
  return std::max<int64_t>(1, std::min<int64_t>(cap, (int64_t)B * Rc * Rc * Rc));
}

size_t vp_brick_bytes(int64_t cap, int32_t B, int32_t R) {
  const int64_t Rc = (R + 3) / 4;
  Carver c(nullptr, 0);
  c.take<int32_t>((int64_t)B * Rc * Rc * Rc);
  c.take<int32_t>(vp_brick_pool(cap, B, R) * 64);
  c.take<int32_t>(vp_brick_pool(cap, B, R));
  c.take<int32_t>(1);
  return c.off;
}

static BrickSpec brick_spec(void* index, int64_t cap, int B, int R, int s) {
  const int Rc = (R + 3) / 4;
  Carver c(index, vp_brick_bytes(cap, B, R));
  BrickSpec g;
  g.coarse = c.take<int32_t>((int64_t)B * Rc * Rc * Rc);
  g.bricks = c.take<int32_t>(vp_brick_pool(cap, B, R) * 64);
  g.owner = c.take<int32_t>(vp_brick_pool(cap, B, R));
  g.counter = c.take<int32_t>(1);
  g.B = B;
  g.R = R;
  g.s = s;
  g.Rc = Rc;
  return g;
}

int vp_brick_init(void* index, int64_t cap, int32_t B, int32_t R, vp_stream_t stream) {
  VP_REQUIRE(B >= 1 && R >= 1, VP_EVALIDATION, "brick: extents must be positive");
  const int64_t Rc = (R + 3) / 4;
  VP_REQUIRE((int64_t)B * Rc * Rc * Rc < (1ll << 31), VP_EVALIDATION, "brick: too many coarse cells");
  BrickSpec g = brick_spec(index, cap, B, R, 1);
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(g.coarse, 0x7f, sizeof(int32_t) * (size_t)B * Rc * Rc * Rc, st);  // kBrickEmpty
  cudaMemsetAsync(g.bricks, 0x7f, sizeof(int32_t) * (size_t)vp_brick_pool(cap, B, R) * 64, st);
  cudaMemsetAsync(g.counter, 0, sizeof(int32_t), st);
  VP_CHECK_ASYNC("brick_init");
  return VP_OK;
}

int vp_brick_set(const int32_t* coords, const int32_t* n_dev, int64_t cap, void* index, int64_t index_cap, int32_t B,
                 int32_t R, int32_t s, int32_t clear, vp_stream_t stream) {
  VP_REQUIRE(B >= 1 && R >= 1 && s >= 1, VP_EVALIDATION, "brick: extents must be positive");
  VP_REQUIRE(cap <= index_cap, VP_EVALIDATION, "brick: more rows than the index pool");
  cudaStream_t st = (cudaStream_t)stream;
  BrickSpec g = brick_spec(index, index_cap, B, R, s);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cap, 256), grid_cap(8)));
  if (clear) {
    ::vp::launch(brick_clear_kernel, kNumSMs * 4, 256, 0, st, g);
    VP_CHECK_LAUNCH("brick_clear");
    ::vp::launch(brick_reset_counter_kernel, 1, 1, 0, st, g.counter);
    VP_CHECK_LAUNCH("brick_reset");
    return VP_OK;
  }
  if (cap <= 0) return VP_OK;
  ::vp::launch(brick_mark_kernel, blocks, 256, 0, st, (const int4*)coords, n_dev, cap, g);
  VP_CHECK_LAUNCH("brick_mark");
  ::vp::launch(brick_assign_kernel, blocks, 256, 0, st, (const int4*)coords, n_dev, cap, g);
  VP_CHECK_LAUNCH("brick_assign");
  ::vp::launch(brick_fill_kernel, blocks, 256, 0, st, (const int4*)coords, n_dev, cap, g);
  VP_CHECK_LAUNCH("brick_fill");
  return VP_OK;
}

int vp_kernel_map_brick(const void* index, int64_t index_cap, int32_t B, int32_t R, int32_t s, const int32_t* out,
                        const int32_t* n_out_dev, int64_t cap_out, const int32_t* offsets_host, int32_t K,
                        const int32_t* in_stride, int32_t* nbr, int32_t* pair_in, int32_t* pair_out,
                        int32_t* pair_ptr, void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(K >= 1 && K <= VP_MAX_OFFSETS, VP_EVALIDATION, "kernel offset count out of range");
  VP_REQUIRE(pair_in && pair_out && pair_ptr, VP_EVALIDATION, "kernel_map_brick: pair outputs required");
  VP_REQUIRE(B >= 1 && R >= 1 && s >= 1, VP_EVALIDATION, "brick: extents must be positive");
  Carver c(ws, ws_bytes);
  const int ntiles = (int)ceil_div(std::max<int64_t>(cap_out, 1), kBrickTile);
  int32_t* counts = c.take<int32_t>((int64_t)ntiles * K);
  int32_t* totals = c.take<int32_t>(K + 1);
  uint32_t* masks = c.take<uint32_t>(std::max<int64_t>(cap_out, 1));
  VP_REQUIRE(c.ok(), VP_EVALIDATION, "kernel_map_brick: workspace too small");
  for (int a = 0; a < 3; ++a)
    VP_REQUIRE(in_stride[a] >= 1 && in_stride[a] % s == 0, VP_EVALIDATION,
               "kernel_map_brick: in_stride must be a multiple of the lattice spacing");
  BrickOffsets offs;
  memset(&offs, 0, sizeof(offs));
  for (int k = 0; k < K; ++k)
    for (int a = 0; a < 3; ++a) {
      const int64_t d = (int64_t)offsets_host[3 * k + a] * (in_stride[a] / s);
      offs.d[3 * k + a] = (int32_t)std::max<int64_t>(std::min<int64_t>(d, R), -(int64_t)R);
    }
  if (cap_out <= 0) {
    cudaMemsetAsync(pair_ptr, 0, sizeof(int32_t) * (K + 1), st);
    VP_CHECK_ASYNC("kernel_map_brick(empty)");
    return VP_OK;
  }
  BrickSpec g = brick_spec(const_cast<void*>(index), index_cap, B, R, s);
  ::vp::launch(map_probe_brick_kernel, ntiles, kBrickTile, 0, st, (const int4*)out, n_out_dev, cap_out, g, offs, K, nbr,
               counts, ntiles, masks);
  VP_CHECK_LAUNCH("map_probe_brick");
  return map_scan_emit(nbr, n_out_dev, cap_out, K, counts, totals, ntiles, pair_in, pair_out, pair_ptr, masks, st);
}

size_t vp_kernel_map_brick_ws_bytes(int64_t cap_out, int32_t K) { return vp_kernel_map_grid_ws_bytes(cap_out, K); }

}  // extern "C"
