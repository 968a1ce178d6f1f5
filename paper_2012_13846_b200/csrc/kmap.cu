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
// levels: batch < B, axes in [0, R*s) on multiples of s): cells [B*R^3]
// (cell -> row) followed by an occupancy bitmap [ceil(B*R^3/32)] words.  A
// cell is meaningful only where its bit is set, so the probe reads the
// bitmap (B*R^3/8 bytes: 2 MB at C3 level 0, L2-resident) for all 27
// neighbours and loads cells only for the ~3 hits per row; empty lattice
// sectors are never fetched from DRAM, and a clear only zeroes bitmap words.
struct GridSpec {
  int32_t* cells;
  uint32_t* bits;
  int B, R, s;
  int ox, oy, oz;  // lattice origin (multiples of s): cell = (coord - origin) / s
};
inline int64_t grid_cells(int B, int R) { return (int64_t)B * R * R * R; }
// the bitmap starts 32-byte aligned after the cells (64-bit loads); 8 zero
// words of slack after it for the probe's line-crossing loads
inline int64_t grid_bits_offset(int B, int R) { return (grid_cells(B, R) + 7) & ~(int64_t)7; }
inline GridSpec grid_spec(int32_t* cells, int B, int R, int s) {
  return GridSpec{cells, reinterpret_cast<uint32_t*>(cells + grid_bits_offset(B, R)), B, R, s, 0, 0, 0};
}
constexpr int32_t kGridEmpty = 0x7fffffff;

// lattice cell of a row (per axis, in units of s) or false when off-lattice
__device__ __forceinline__ bool grid_coords(const GridSpec& g, int4 r, int& cx, int& cy, int& cz) {
  r.y -= g.ox;
  r.z -= g.oy;
  r.w -= g.oz;
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
    if (!grid_coords(g, r, cx, cy, cz)) continue;
    const int p = grid_linear(g, r.x, cx, cy, cz);
    if (clear) {
      g.bits[p >> 5] = 0u;  // every bit of the word belongs to a row of this (same) set
    } else {
      g.cells[p] = (int32_t)i;
      atomicOr(&g.bits[p >> 5], 1u << (p & 31));
    }
  }
}

// Internal map hash.  The slot layout of the map's private table is not
// semantic (only the rows found are), so instead of splitmix64 on the 64-bit
// key it mixes the two 32-bit halves of the packed key (kernels.py:75-78
// fields) with 32-bit multiplies: a handful of instructions per probe
// instead of two emulated 64-bit multiplies.
//
// z-grouped homes (zlg > 0): rows with the same (batch, x, y) and the same
// aligned run of 2^zlg lattice steps in z (q = biased z >> zsh, zsh = log2 of
// the input stride in z) hash together and take consecutive home slots
// (q & (2^zlg - 1)), so a row's 3 z-neighbours usually share one 64-128 B
// line of the table: ~9-12 distinct lines per 27-offset probe instead of 27.
__device__ __forceinline__ uint32_t map_slot(uint32_t hi, uint32_t lo, uint32_t mask, int zsh, int zlg) {
  const uint32_t q = (lo & 0xFFFFu) >> zsh;
  const uint32_t lg = (lo & 0xFFFF0000u) | (q >> zlg);
  uint32_t h = lg * 0x9E3779B1u ^ (hi * 0x85EBCA77u + 0x165667B1u);
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  return ((h << zlg) | (q & ((1u << zlg) - 1u))) & mask;
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
                                  Slot* t, uint64_t cap, int zsh, int zlg) {
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
    uint32_t s = map_slot(hi, lo, mask, zsh, zlg);
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
                 int K, int32_t* __restrict__ nbr, int32_t* counts, int ntiles, uint32_t* __restrict__ masks,
                 int zsh, int zlg, int stream_nbr) {
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
  uint32_t hitm = 0;  // the row's hit bits (k < 32), identical in its 8 lanes
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
          slot[b] = map_slot(khi[b], klo[b], mask, zsh, zlg);
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
      if (k0 < 32) hitm |= ((m >> ((row & 3) * kMapTPR)) & 0xFFu) << k0;  // the row's 8 lanes: k0..k0+7
      if (lane < kMapTPR && k0 + lane < K) s_cnt[warp][k0 + lane] = (unsigned short)__popc(m & (0x01010101u << lane));
    }
  }
  if (masks && valid && j == 0) masks[u0 + row] = hitm;
  __syncthreads();
  if (staged) {  // warp per row: K <= 32 contiguous ints, no division
    int32_t* dst = nbr + u0 * K;
    for (int rr = warp; rr < rows; rr += kProbeWarps)
      if (lane < K) {
        if (stream_nbr) __stcs(dst + rr * K + lane, s_nbr[rr * (kMapSmemK + 1) + lane]);
        else dst[rr * K + lane] = s_nbr[rr * (kMapSmemK + 1) + lane];
      }
  }
  for (int k = tid; k < K; k += kProbeThreads) {
    int c = 0;
#pragma unroll 8
    for (int w = 0; w < kProbeWarps; ++w) c += s_cnt[w][k];
    counts[(int64_t)k * ntiles + tile] = c;
  }
}

// Dense-grid probe: one thread per output row; the bitmap words of all 27
// neighbours are loaded at once (the 3 z-neighbours of a column share a
// word: L1 hits), then the cells of the set bits only.  Offsets arrive
// pre-scaled to cells (off * in_stride / s) with their linear cell delta, so
// a probe is 3 unsigned compares + 1 bitmap load (+ 1 cell load on a hit).
// masks[u] (K <= 32) gets the row's hit bits for the emit.
struct GridOffsets {
  int32_t d[VP_MAX_OFFSETS * 3];
  int32_t lin[VP_MAX_OFFSETS];
};

__global__ void __launch_bounds__(kMapTile)
map_probe_grid_kernel(const int4* __restrict__ out, const int32_t* n_out_dev, int64_t cap_out, GridSpec g,
                      const __grid_constant__ GridOffsets offs, int K, int32_t* __restrict__ nbr, int32_t* counts,
                      int ntiles, uint32_t* __restrict__ masks) {
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
  uint32_t hitm = 0;
  for (int kb = 0; kb < K; kb += KB) {
    uint32_t w[KB];
#pragma unroll
    for (int b = 0; b < KB; ++b) {
      const int k = kb + b;
      w[b] = 0u;
      if (on && k < K && (unsigned)(cx + offs.d[3 * k]) < R && (unsigned)(cy + offs.d[3 * k + 1]) < R &&
          (unsigned)(cz + offs.d[3 * k + 2]) < R) {
        const int p = base + offs.lin[k];
        w[b] = (__ldg(g.bits + (p >> 5)) >> (p & 31)) & 1u;
      }
    }
    int v[KB];
#pragma unroll
    for (int b = 0; b < KB; ++b) v[b] = w[b] ? __ldg(g.cells + base + offs.lin[kb + b]) : -1;
#pragma unroll
    for (int b = 0; b < KB; ++b) {
      const int k = kb + b;
      if (k >= K) break;
      const int x = v[b];
      if (k < 32 && x >= 0) hitm |= 1u << k;
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
  if (masks && valid) masks[u0 + tid] = hitm;
  for (int k = tid; k < K; k += kMapTile) {
    int c = 0;
#pragma unroll
    for (int w = 0; w < kMapTile / 32; ++w) c += s_cnt[w][k];
    counts[(int64_t)k * ntiles + tile] = c;
  }
}

// Unit-cube probe (the 3^3 offsets {-1,0,1}^3 in lattice steps, any order:
// every map the training engine builds).  A row's 27 neighbour bits are 9
// z-runs of 3 adjacent bits, one per (dx, dy) column of the bitmap: 9 64-bit
// loads (a second one only when the run crosses a 64-bit word) instead of 27
// scattered loads, then cell loads for the hits only.  cube.k maps
// ((dx+1)*3 + dy+1)*3 + dz+1 to the caller's offset index.
struct GridCube {
  int8_t k[27];
};

__global__ void __launch_bounds__(kMapTile)
map_probe_grid_cube_kernel(const int4* __restrict__ out, const int32_t* n_out_dev, int64_t cap_out, GridSpec g,
                           const __grid_constant__ GridOffsets offs, const __grid_constant__ GridCube cube,
                           int32_t* __restrict__ nbr, int32_t* counts, int ntiles, uint32_t* __restrict__ masks,
                           int32_t* __restrict__ own, int32_t* __restrict__ scratch) {
  ::vp::pdl_begin();
  constexpr int K = 27;
  __shared__ int s_nbr[kMapTile * (kMapSmemK + 1)];
  __shared__ int s_cnt[kMapTile / 32][K];
  __shared__ int s_koff[32];
  const int tile = blockIdx.x;
  const int64_t u0 = (int64_t)tile * kMapTile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the row's coordinates are loaded alongside the live count (one round trip)
  const int4 r = u0 + tid < cap_out ? __ldg(out + u0 + tid) : make_int4(-1, 0, 0, 0);
  const int n_out = load_count(n_out_dev, cap_out);
  if (u0 >= n_out) return;
  const int rows = (n_out - u0) < kMapTile ? (int)(n_out - u0) : kMapTile;
  const bool valid = tid < rows;
  int cx = 0, cy = 0, cz = 0, b = 0, base = 0;
  bool on = false;
  if (valid) {
    on = grid_coords(g, r, cx, cy, cz);
    b = r.x;
    if (on) base = grid_linear(g, b, cx, cy, cz);
  }
  const int R = g.R;
  const unsigned long long* __restrict__ b64 = reinterpret_cast<const unsigned long long*>(g.bits);
  uint32_t hit = 0;
  if (on) {
    const int zs = cz > 0 ? cz - 1 : 0;  // first bit of the run (dz = -1, or dz = 0 at the z = 0 face)
    unsigned long long lo[9];
    int q[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      const int qx = cx + c / 3 - 1, qy = cy + c % 3 - 1;
      q[c] = -1;
      lo[c] = 0ull;
      if ((unsigned)qx < (unsigned)R && (unsigned)qy < (unsigned)R) {
        q[c] = ((b * R + qx) * R + qy) * R + zs;
        lo[c] = __ldg(b64 + (q[c] >> 6));
      }
    }
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      if (q[c] < 0) continue;
      const int sh = q[c] & 63;
      unsigned long long v = lo[c] >> sh;
      if (sh > 61) v |= __ldg(b64 + (q[c] >> 6) + 1) << (64 - sh);
      uint32_t t3 = cz > 0 ? (uint32_t)v & 7u : ((uint32_t)v << 1) & 6u;
      if (cz + 1 >= R) t3 &= 3u;
#pragma unroll
      for (int dz = 0; dz < 3; ++dz)
        if ((t3 >> dz) & 1u) hit |= 1u << cube.k[c * 3 + dz];
    }
  }
  int v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = ((hit >> k) & 1u) ? __ldg(g.cells + base + offs.lin[k]) : -1;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    s_nbr[tid * (kMapSmemK + 1) + k] = v[k];
    const unsigned m = __ballot_sync(0xffffffffu, v[k] >= 0);
    if (lane == 0) s_cnt[warp][k] = __popc(m);
  }
  __syncthreads();
  int32_t* dst = nbr + u0 * K;
  for (int rr = warp; rr < rows; rr += kMapTile / 32)
    if (lane < K) dst[rr * K + lane] = s_nbr[rr * (kMapSmemK + 1) + lane];
  if (masks && valid) masks[u0 + tid] = hit;
  if (warp == 0) {  // the tile's per-offset counts: k-major for the scan, tile-major + offsets for the emit
    int c = 0;
    if (lane < K) {
#pragma unroll
      for (int w = 0; w < kMapTile / 32; ++w) c += s_cnt[w][lane];
      counts[(int64_t)lane * ntiles + tile] = c;
      if (own) own[(int64_t)tile * 32 + lane] = c;
    }
    int inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += y;
    }
    s_koff[lane] = inc - c;
  }
  if (!scratch) return;
  // The tile's pairs compacted in the final (offset, ascending row) order
  // into its private scratch slab [2][kMapTile*K]: the emit then copies 27
  // contiguous segments instead of re-reading nbr rows for the hits.
  __syncthreads();
  int32_t* sc_in = scratch + (int64_t)tile * 2 * kMapTile * K;
  int32_t* sc_out = sc_in + kMapTile * K;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const bool h = (hit >> k) & 1u;
    const unsigned m = __ballot_sync(0xffffffffu, h);
    if (h) {
      int before = s_koff[k];
#pragma unroll
      for (int w = 0; w < kMapTile / 32; ++w) before += (w < warp) ? s_cnt[w][k] : 0;
      const int pos = before + __popc(m & lt);
      sc_in[pos] = v[k];
      sc_out[pos] = (int32_t)(u0 + tid);
    }
  }
}

// Emit from the probe's compacted tile slabs: per offset, one contiguous
// segment of the slab goes to pair_in/pair_out at the offset base + the
// tile's scanned prefix.  Warps take offsets round-robin; lanes copy.
__global__ void __launch_bounds__(kMapTile)
map_emit_slab_kernel(const int32_t* __restrict__ scratch, const int32_t* __restrict__ own, const int32_t* n_out_dev,
                     int64_t cap_out, int K, const int32_t* __restrict__ counts, const int32_t* __restrict__ totals,
                     int ntiles_cap, int32_t* __restrict__ pair_in, int32_t* __restrict__ pair_out,
                     int32_t* pair_ptr) {
  ::vp::pdl_begin();
  __shared__ int s_base[33];
  __shared__ int s_pre[32];
  __shared__ int s_len[32];
  __shared__ int s_off[32];
  const int tile = blockIdx.x;
  const int64_t u0 = (int64_t)tile * kMapTile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_out = load_count(n_out_dev, cap_out);
  if (warp == 0) {  // offset bases (scan of the K totals)
    const int t = lane < K ? __ldg(totals + lane) : 0;
    int inc = t;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += y;
    }
    if (lane < K) s_base[lane] = inc - t;
    if (tile == 0 && lane < K) pair_ptr[lane] = inc - t;
    if (tile == 0 && lane == K - 1) pair_ptr[K] = inc;
  } else if (warp == 1 && u0 < n_out) {  // the tile's segment lengths / slab offsets / scanned prefixes
    const int c = lane < K ? __ldg(own + (int64_t)tile * 32 + lane) : 0;
    int inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += y;
    }
    s_len[lane] = c;
    s_off[lane] = inc - c;
    s_pre[lane] = lane < K ? __ldg(counts + (int64_t)lane * ntiles_cap + tile) : 0;
  }
  if (u0 >= n_out) return;
  __syncthreads();
  const int32_t* sc_in = scratch + (int64_t)tile * 2 * kMapTile * K;
  const int32_t* sc_out = sc_in + kMapTile * K;
  for (int k = warp; k < K; k += kMapTile / 32) {
    const int len = s_len[k], src = s_off[k], dst = s_base[k] + s_pre[k];
    for (int i = lane; i < len; i += 32) {
      pair_in[dst + i] = __ldg(sc_in + src + i);
      pair_out[dst + i] = __ldg(sc_out + src + i);
    }
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

// K <= 32 emit from the probe's per-row hit masks: the counting ballots need
// no loads, and only the hit entries of the tile's nbr rows are read (~3 of
// 27 per row) instead of staging the whole [128, K] tile.
__global__ void __launch_bounds__(kMapTile)
map_emit_mask_kernel(const int32_t* __restrict__ nbr, const uint32_t* __restrict__ masks, const int32_t* n_out_dev,
                     int64_t cap_out, int K, const int32_t* __restrict__ counts, const int32_t* __restrict__ totals,
                     int ntiles_cap, int32_t* __restrict__ pair_in, int32_t* __restrict__ pair_out,
                     int32_t* pair_ptr) {
  ::vp::pdl_begin();
  __shared__ int s_w[kMapTile / 32][32];
  __shared__ int s_base[33];
  __shared__ int s_tot[32];
  const int tile = blockIdx.x;
  const int64_t u0 = (int64_t)tile * kMapTile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t hm_raw = u0 + tid < cap_out ? __ldg(masks + u0 + tid) : 0u;  // beside the live count
  const int n_out = load_count(n_out_dev, cap_out);
  if (warp == 0) {  // offset bases: one warp-wide inclusive scan of the K totals
    const int t = lane < K ? __ldg(totals + lane) : 0;
    int inc = t;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += y;
    }
    if (lane < K) s_base[lane] = inc - t;
    if (lane == K - 1) s_base[K] = inc;
    if (tile == 0 && lane < K) pair_ptr[lane] = inc - t;
    if (tile == 0 && lane == K - 1) pair_ptr[K] = inc;
  }
  if (u0 >= n_out) return;
  const int rows = (n_out - u0) < kMapTile ? (int)(n_out - u0) : kMapTile;
  const bool valid = tid < rows;
  if (tid < K) s_tot[tid] = __ldg(counts + (int64_t)tid * ntiles_cap + tile);
  const uint32_t hm = valid ? hm_raw : 0u;
  // all hit values in flight at once (~3 of 32 per row), not one dependent
  // load per offset inside the ordered loop
  const int32_t* row = nbr + (u0 + tid) * K;
  int v[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = (k < K && ((hm >> k) & 1u)) ? __ldg(row + k) : -1;
  for (int k = 0; k < K; ++k) {
    const unsigned m = __ballot_sync(0xffffffffu, (hm >> k) & 1u);
    if (lane == 0) s_w[warp][k] = __popc(m);
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k >= K) break;
    const bool hit = (hm >> k) & 1u;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (hit) {
      int before = 0;
#pragma unroll
      for (int w = 0; w < kMapTile / 32; ++w) before += (w < warp) ? s_w[w][k] : 0;
      const int pos = s_base[k] + s_tot[k] + before + __popc(m & lt);
      pair_in[pos] = v[k];
      pair_out[pos] = (int32_t)(u0 + tid);
    }
  }
}

// Bounding box of two row sets for the operator API's lattice decision:
// bbox[0..8] = min over rows of (b, x, y, z, -b, -x, -y, -z) and of
// "on the spacing-s lattice" (1) / "off it" (0); memset 0x7f initialises
// every field to a value above any row's.
__global__ void coords_bbox_kernel(const int4* __restrict__ a, int64_t n_a, const int4* __restrict__ b, int64_t n_b,
                                   int s, int32_t* bbox) {
  ::vp::pdl_begin();
  int m[9];
#pragma unroll
  for (int f = 0; f < 9; ++f) m[f] = 0x7f7f7f7f;
  const int64_t n = n_a + n_b;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int4 r = i < n_a ? __ldg(a + i) : __ldg(b + (i - n_a));
    m[0] = min(m[0], r.x);
    m[1] = min(m[1], r.y);
    m[2] = min(m[2], r.z);
    m[3] = min(m[3], r.w);
    m[4] = min(m[4], -r.x);
    m[5] = min(m[5], -r.y);
    m[6] = min(m[6], -r.z);
    m[7] = min(m[7], -r.w);
    // sign-independent lattice test (a mask for power-of-two spacings)
    const bool on = (s & (s - 1)) == 0 ? ((r.y | r.z | r.w) & (s - 1)) == 0
                                       : (r.y % s) == 0 && (r.z % s) == 0 && (r.w % s) == 0;
    m[8] = min(m[8], on ? 1 : 0);
  }
  __shared__ int s_m[9];
  if (threadIdx.x < 9) s_m[threadIdx.x] = 0x7f7f7f7f;
  __syncthreads();
#pragma unroll
  for (int f = 0; f < 9; ++f) {
    int v = m[f];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, d));
    if ((threadIdx.x & 31) == 0) atomicMin(s_m + f, v);
  }
  __syncthreads();  // one global atomic per field per block (same-address atomics serialise in L2)
  if (threadIdx.x < 9 && s_m[threadIdx.x] != 0x7f7f7f7f) atomicMin(bbox + threadIdx.x, s_m[threadIdx.x]);
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
                  const uint32_t* masks, cudaStream_t st) {
  ::vp::launch(map_scan_kernel, K, 1024, 0, st, counts, n_out_dev, cap_out, ntiles, totals);
  VP_CHECK_LAUNCH("map_scan");
  if (masks && K <= 32) {
    ::vp::launch(map_emit_mask_kernel, ntiles, kMapTile, 0, st, nbr, masks, n_out_dev, cap_out, K,
                 (const int32_t*)counts, (const int32_t*)totals, ntiles, pair_in, pair_out, pair_ptr);
    VP_CHECK_LAUNCH("map_emit_mask");
    return VP_OK;
  }
  ::vp::launch(map_emit_kernel, ntiles, kMapTile, 0, st, nbr, n_out_dev, cap_out, K, (const int32_t*)counts,
               (const int32_t*)totals, ntiles, pair_in, pair_out, pair_ptr);
  VP_CHECK_LAUNCH("map_emit");
  return VP_OK;
}
}  // namespace vp

using namespace vp;

extern "C" {

// the map's private table: slots >= VP_MAP_LOADF * rows (power of two)
static uint64_t map_table_cap(int64_t n) {
  static const int f = getenv("VP_MAP_LOADF") ? std::max(2, atoi(getenv("VP_MAP_LOADF"))) : 4;
  uint64_t cap = 8;
  while (cap < (uint64_t)(f * n + 4)) cap <<= 1;
  return cap;
}
static int map_zgroup_log2() {
  static const int v = getenv("VP_MAP_ZG") ? std::min(4, std::max(0, atoi(getenv("VP_MAP_ZG")))) : 0;
  return v;
}

size_t vp_kernel_map_ws_bytes(int64_t cap_in, int64_t cap_out, int32_t K) {
  Carver c(nullptr, 0);
  c.take<Slot>(map_table_cap(cap_in) + 1);
  int64_t ntiles = ceil_div(std::max<int64_t>(cap_out, 1), kMapTile);
  c.take<int32_t>(ntiles * K);
  c.take<int32_t>(K + 1);
  c.take<uint32_t>(std::max<int64_t>(cap_out, 1));
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
  uint64_t cap = map_table_cap(cap_in);
  Slot* t = c.take<Slot>(cap + 1);
  int ntiles = (int)ceil_div(std::max<int64_t>(cap_out, 1), kMapTile);
  int32_t* counts = c.take<int32_t>((int64_t)ntiles * K);
  int32_t* totals = c.take<int32_t>(K + 1);
  uint32_t* masks = c.take<uint32_t>(std::max<int64_t>(cap_out, 1));
  VP_REQUIRE(c.ok(), VP_EVALIDATION, "kernel_map: workspace too small");
  Offsets offs;
  memset(&offs, 0, sizeof(offs));
  for (int k = 0; k < K; ++k)
    for (int a = 0; a < 3; ++a) {
      // off * stride, clamped: anything beyond +-2^20 misses like +-2^20 does
      const int64_t d = (int64_t)offsets_host[3 * k + a] * in_stride[a];
      offs.d[3 * k + a] = (int32_t)std::max<int64_t>(std::min<int64_t>(d, 1 << 20), -(1 << 20));
    }
  // z-grouped homes on the input lattice: zsh = log2(in_stride z) (0 when it
  // is not a power of two: grouping by raw z is still a valid hash)
  int zsh = 0;
  if (in_stride[2] > 0 && (in_stride[2] & (in_stride[2] - 1)) == 0)
    while ((1 << zsh) < in_stride[2]) ++zsh;
  const int zlg = map_zgroup_log2();
  int r = hash_clear(t, cap, st);
  if (r) return r;
  if (cap_in > 0) {
    int blocks = (int)std::min<int64_t>(ceil_div(cap_in, 256), grid_cap(8));
    ::vp::launch(map_insert_kernel, blocks, 256, 0, st, (const int4*)in, n_in_dev, cap_in, t, cap, zsh, zlg);
    VP_CHECK_LAUNCH("map_insert");
  }
  if (cap_out <= 0) {
    if (pair_ptr) cudaMemsetAsync(pair_ptr, 0, sizeof(int32_t) * (K + 1), st);
    VP_CHECK_ASYNC("kernel_map(empty)");
    return VP_OK;
  }
  ::vp::launch(map_probe_kernel, ntiles, kProbeThreads, 0, st, (const int4*)out, n_out_dev, cap_out, t, cap, offs, K,
                                                   nbr, counts, ntiles, masks, zsh, zlg,
                                                   getenv("VP_MAP_STREAM_NBR") ? atoi(getenv("VP_MAP_STREAM_NBR")) : 0);
  VP_CHECK_LAUNCH("map_probe");
  if (pair_in) return map_scan_emit(nbr, n_out_dev, cap_out, K, counts, totals, ntiles, pair_in, pair_out, pair_ptr,
                                    masks, st);
  return VP_OK;
}

static int grid_set_g(const int32_t* coords, const int32_t* n_dev, int64_t cap, GridSpec g, int clear,
                      cudaStream_t st) {
  VP_REQUIRE(g.B >= 1 && g.R >= 1 && g.s >= 1, VP_EVALIDATION, "grid: extents must be positive");
  VP_REQUIRE(grid_cells(g.B, g.R) < (1ll << 31), VP_EVALIDATION, "grid: B*R^3 must be < 2^31 cells");
  if (cap <= 0) return VP_OK;
  const int64_t bitmap_bytes = 4 * (vp_grid_words(g.B, g.R) - grid_bits_offset(g.B, g.R));
  if (clear && bitmap_bytes <= 32 * cap) {
    // the bitmap holds only this row set: zeroing it whole costs fewer bytes
    // than one scattered 32-byte sector store per row
    cudaMemsetAsync(g.bits, 0, bitmap_bytes, st);
    VP_CHECK_ASYNC("grid_clear(memset)");
    return VP_OK;
  }
  int blocks = (int)std::min<int64_t>(ceil_div(cap, 256), grid_cap(8));
  ::vp::launch(grid_set_kernel, blocks, 256, 0, st, (const int4*)coords, n_dev, cap, g, clear);
  VP_CHECK_LAUNCH("grid_set");
  return VP_OK;
}

int vp_grid_set(const int32_t* coords, const int32_t* n_dev, int64_t cap, int32_t* cells, int32_t B, int32_t R,
                int32_t s, int32_t clear, vp_stream_t stream) {
  VP_REQUIRE(B >= 1 && R >= 1 && s >= 1, VP_EVALIDATION, "grid: extents must be positive");
  VP_REQUIRE((int64_t)B * R * R * R < (1ll << 31), VP_EVALIDATION, "grid: B*R^3 must be < 2^31 cells");
  return grid_set_g(coords, n_dev, cap, grid_spec(cells, B, R, s), clear, (cudaStream_t)stream);
}

int64_t vp_grid_words(int32_t B, int32_t R) {
  if (B < 1 || R < 1) return 0;
  return grid_bits_offset(B, R) + ((ceil_div(grid_cells(B, R), 32) + 1) & ~(int64_t)1) + 8;
}

int vp_grid_init(int32_t* cells, int32_t B, int32_t R, vp_stream_t stream) {
  VP_REQUIRE(B >= 1 && R >= 1, VP_EVALIDATION, "grid: extents must be positive");
  VP_REQUIRE(grid_cells(B, R) < (1ll << 31), VP_EVALIDATION, "grid: B*R^3 must be < 2^31 cells");
  cudaMemsetAsync(grid_spec(cells, B, R, 1).bits, 0,
                  sizeof(uint32_t) * (vp_grid_words(B, R) - grid_bits_offset(B, R)), (cudaStream_t)stream);
  VP_CHECK_ASYNC("grid_init");
  return VP_OK;
}

size_t vp_kernel_map_grid_ws_bytes(int64_t cap_out, int32_t K) {
  Carver c(nullptr, 0);
  int64_t ntiles = ceil_div(std::max<int64_t>(cap_out, 1), kMapTile);
  c.take<int32_t>(ntiles * K);
  c.take<int32_t>(K + 1);
  c.take<uint32_t>(std::max<int64_t>(cap_out, 1));
  if (K == 27) {  // unit-cube probe: per-tile counts + compacted pair slabs
    c.take<int32_t>(ntiles * 32);
    c.take<int32_t>(ntiles * 2 * kMapTile * K);
  }
  return c.off;
}

static int map_grid_g(GridSpec g, const int32_t* out, const int32_t* n_out_dev, int64_t cap_out,
                      const int32_t* offsets_host, int32_t K, const int32_t* in_stride, int32_t* nbr, int32_t* pair_in,
                      int32_t* pair_out, int32_t* pair_ptr, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int B = g.B, R = g.R, s = g.s;
  VP_REQUIRE(K >= 1 && K <= VP_MAX_OFFSETS, VP_EVALIDATION, "kernel offset count out of range");
  VP_REQUIRE(pair_in && pair_out && pair_ptr, VP_EVALIDATION, "kernel_map_grid: pair outputs required");
  VP_REQUIRE(B >= 1 && R >= 1 && s >= 1, VP_EVALIDATION, "grid: extents must be positive");
  Carver c(ws, ws_bytes);
  int ntiles = (int)ceil_div(std::max<int64_t>(cap_out, 1), kMapTile);
  int32_t* counts = c.take<int32_t>((int64_t)ntiles * K);
  int32_t* totals = c.take<int32_t>(K + 1);
  uint32_t* masks = c.take<uint32_t>(std::max<int64_t>(cap_out, 1));
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
  // the 3^3 unit cube in lattice steps (any order) takes the column probe
  GridCube cube;
  memset(&cube, -1, sizeof(cube));
  bool unit = K == 27;
  for (int k = 0; unit && k < K; ++k) {
    const int* d = offs.d + 3 * k;
    if (d[0] < -1 || d[0] > 1 || d[1] < -1 || d[1] > 1 || d[2] < -1 || d[2] > 1) { unit = false; break; }
    int8_t& slot = cube.k[((d[0] + 1) * 3 + d[1] + 1) * 3 + d[2] + 1];
    if (slot >= 0) unit = false;
    slot = (int8_t)k;
  }
  static const bool cube_on = !getenv("VP_MAP_CUBE") || atoi(getenv("VP_MAP_CUBE")) != 0;
  if (unit && cube_on) {
    int32_t* own = c.take<int32_t>((int64_t)ntiles * 32);
    int32_t* slab = c.take<int32_t>((int64_t)ntiles * 2 * kMapTile * K);
    VP_REQUIRE(c.ok(), VP_EVALIDATION, "kernel_map_grid: workspace too small");
    static const bool slab_on = !getenv("VP_MAP_SLAB") || atoi(getenv("VP_MAP_SLAB")) != 0;
    ::vp::launch(map_probe_grid_cube_kernel, ntiles, kMapTile, 0, st, (const int4*)out, n_out_dev, cap_out,
                 g, offs, cube, nbr, counts, ntiles,
                 slab_on ? nullptr : masks, slab_on ? own : nullptr, slab_on ? slab : nullptr);
    VP_CHECK_LAUNCH("map_probe_grid_cube");
    if (!slab_on)
      return map_scan_emit(nbr, n_out_dev, cap_out, K, counts, totals, ntiles, pair_in, pair_out, pair_ptr, masks,
                           st);
    ::vp::launch(map_scan_kernel, K, 1024, 0, st, counts, n_out_dev, cap_out, ntiles, totals);
    VP_CHECK_LAUNCH("map_scan");
    ::vp::launch(map_emit_slab_kernel, ntiles, kMapTile, 0, st, (const int32_t*)slab, (const int32_t*)own, n_out_dev,
                 cap_out, K, (const int32_t*)counts, (const int32_t*)totals, ntiles, pair_in, pair_out, pair_ptr);
    VP_CHECK_LAUNCH("map_emit_slab");
    return VP_OK;
  }
  ::vp::launch(map_probe_grid_kernel, ntiles, kMapTile, 0, st, (const int4*)out, n_out_dev, cap_out,
                                                     g, offs, K, nbr, counts, ntiles, masks);
  VP_CHECK_LAUNCH("map_probe_grid");
  return map_scan_emit(nbr, n_out_dev, cap_out, K, counts, totals, ntiles, pair_in, pair_out, pair_ptr, masks, st);
}

int vp_kernel_map_grid(const int32_t* cells, int32_t B, int32_t R, int32_t s, const int32_t* out,
                       const int32_t* n_out_dev, int64_t cap_out, const int32_t* offsets_host, int32_t K,
                       const int32_t* in_stride, int32_t* nbr, int32_t* pair_in, int32_t* pair_out, int32_t* pair_ptr,
                       void* ws, size_t ws_bytes, vp_stream_t stream) {
  VP_REQUIRE(B >= 1 && R >= 1 && s >= 1, VP_EVALIDATION, "grid: extents must be positive");
  return map_grid_g(grid_spec(const_cast<int32_t*>(cells), B, R, s), out, n_out_dev, cap_out, offsets_host, K,
                    in_stride, nbr, pair_in, pair_out, pair_ptr, ws, ws_bytes, (cudaStream_t)stream);
}

int vp_coords_bbox(const int32_t* a, int64_t n_a, const int32_t* b, int64_t n_b, int32_t s, int32_t* bbox,
                   vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(s >= 1, VP_EVALIDATION, "coords_bbox: spacing must be positive");
  cudaMemsetAsync(bbox, 0x7f, sizeof(int32_t) * 9, st);
  VP_CHECK_ASYNC("coords_bbox(init)");
  const int64_t n = std::max<int64_t>(n_a, 0) + std::max<int64_t>(n_b, 0);
  if (n <= 0) return VP_OK;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 512), grid_cap(4)));
  ::vp::launch(coords_bbox_kernel, blocks, 512, 0, st, (const int4*)a, n_a, (const int4*)b, n_b, s, bbox);
  VP_CHECK_LAUNCH("coords_bbox");
  return VP_OK;
}

int vp_kernel_map_lattice(const int32_t* in, int64_t n_in, const int32_t* out, int64_t n_out,
                          const int32_t* offsets_host, int32_t K, int32_t s, const int32_t* lattice_host,
                          int32_t* grid, int64_t grid_words, int32_t* nbr, int32_t* pair_in, int32_t* pair_out,
                          int32_t* pair_ptr, void* ws, size_t ws_bytes, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int B = lattice_host[0], R = lattice_host[1];
  VP_REQUIRE(B >= 1 && R >= 1 && s >= 1, VP_EVALIDATION, "lattice: extents must be positive");
  VP_REQUIRE(grid_words >= vp_grid_words(B, R), VP_EVALIDATION, "lattice: grid buffer too small");
  GridSpec g = grid_spec(grid, B, R, s);
  g.ox = lattice_host[2];
  g.oy = lattice_host[3];
  g.oz = lattice_host[4];
  const int32_t st3[3] = {s, s, s};
  int r = grid_set_g(in, nullptr, n_in, g, 0, st);
  if (r) return r;
  r = map_grid_g(g, out, nullptr, n_out, offsets_host, K, st3, nbr, pair_in, pair_out, pair_ptr, ws, ws_bytes, st);
  if (r) return r;
  return grid_set_g(in, nullptr, n_in, g, 1, st);
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
