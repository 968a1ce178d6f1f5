// Neighbour-pattern row grouping for the output-stationary implicit GEMM.
//
// A 128-row tile of the conv kernels pays one gather stage (and one MMA) per
// kernel offset that ANY of its rows uses.  In voxelization (first-seen)
// order a tile's rows are scattered over the cloud, so almost all 27 offsets
// are active while each row has only ~3 neighbours (surface clouds).
// Grouping rows that use the same offsets shrinks a tile's active set; the
// conv kernels then read the permuted table and write output row perm[i]
// for table row i: every output row is still written exactly once with the
// same per-row accumulation order (skipped offsets only contributed exact
// zeros), deterministic, no atomics on the output.
//
// The grouping key is 9 bits of the 3^3 hit mask, measured on C3's maps to
// group as well as or better than a full 27-bit sort (active offsets per
// 128-row tile, level-1 stride-1 table: unsorted 26.7, 27-bit sort 15.9,
// column key 13.7; level-0->1 inverse table: 25.9, 2.0, plane key 2.2):
//   key 0 "columns": which of the 9 (dx, dy) columns hold a hit;
//   key 1 "planes" : which dx / dy / dz planes hold a hit (3 + 3 + 3 bits).
// Stable counting sort over the LIVE rows into 512 buckets, three kernels
// (block histograms; bucket-major look-back scan; per-warp ordered scatter
// with __match_any_sync ranks) plus a coalesced row permute.  key 2 "mask"
// runs three such stable passes over 9-bit digits of the full 27-bit mask
// (LSD) — the order of a stable sort by the whole mask, which groups best
// when levels hold ~1M rows (C2 / C5).  No library sort; the order depends
// only on the table -> deterministic.
#include "common.cuh"

namespace vp {

constexpr int kGroupBuckets = 512;
constexpr int kGroupTile = 2048;      // rows per block
constexpr int kGroupThreads = 256;    // 8 warps x 256 rows each in the scatter

__device__ __forceinline__ int group_key(const int32_t* __restrict__ t, int K, int mode) {
  if (K != 27) {  // generic shapes: the first 9 offsets' hits
    int m = 0;
    for (int k = 0; k < K && k < 9; ++k) m |= (__ldg(t + k) >= 0) << k;
    return m;
  }
  int hit[27];
#pragma unroll
  for (int k = 0; k < 27; ++k) hit[k] = __ldg(t + k) >= 0;  // offset k = (dx, dy, dz) in product order
  int key = 0;
  if (mode == 0) {
#pragma unroll
    for (int c = 0; c < 9; ++c) key |= (hit[3 * c] | hit[3 * c + 1] | hit[3 * c + 2]) << c;
  } else {
#pragma unroll
    for (int k = 0; k < 27; ++k) {
      const int dx = k / 9, dy = (k / 3) % 3, dz = k % 3;
      key |= (hit[k] << dx) | (hit[k] << (3 + dy)) | (hit[k] << (6 + dz));
    }
  }
  return key;
}

constexpr int kScanTile = 4096;  // hist entries per block of the look-back scan (4 per thread)

// keys of the block's live rows + the block's bucket histogram (bucket-major);
// block 0 also zeroes the scan's look-back state for the next kernel
// full-mask mode (key_mode 2): masks[r] = the row's 27-bit hit mask, and the
// key of pass p is bits [9p, 9p + 9) of the mask of the row at position i of
// the previous pass's order (LSD radix: three stable passes = the order of a
// stable sort by the whole mask)
__device__ __forceinline__ uint32_t full_mask(const int32_t* __restrict__ t, int K) {
  uint32_t m = 0;
  for (int k = 0; k < K && k < 27; ++k) m |= (uint32_t)(__ldg(t + k) >= 0) << k;
  return m;
}

// group_key of a 3^3 row from its 27-bit hit mask (bit k = offset k)
__device__ __forceinline__ int key_of_mask27(uint32_t m, int mode) {
  int key = 0;
  if (mode == 0) {
#pragma unroll
    for (int c = 0; c < 9; ++c) key |= (((m >> (3 * c)) & 7u) != 0u) << c;
  } else {
    // planes: dx = k / 9, dy = (k / 3) % 3, dz = k % 3
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const uint32_t mx = 0x1FFu << (9 * d);
      const uint32_t my = (0x7u << (3 * d)) | (0x7u << (9 + 3 * d)) | (0x7u << (18 + 3 * d));
      const uint32_t mz = 0x1249249u << d;  // bits d, d + 3, ..., d + 24
      key |= ((m & mx) != 0u) << d;
      key |= ((m & my) != 0u) << (3 + d);
      key |= ((m & mz) != 0u) << (6 + d);
    }
  }
  return key;
}

constexpr int kHistThreads = 1024;  // 32 warps: two 32-row groups each, their loads in flight together

__global__ void __launch_bounds__(kHistThreads)
group_hist_kernel(const int32_t* __restrict__ table, const int32_t* n_dev, int64_t cap, int K, int mode,
                  uint16_t* __restrict__ keys, int32_t* __restrict__ hist, int nblocks, ScanState ss, int scan_tiles,
                  uint32_t* __restrict__ masks, const int32_t* __restrict__ order_in, int shift, int desc) {
  ::vp::pdl_begin();
  __shared__ int s_h[kGroupBuckets];
  const int n = load_count(n_dev, cap);
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < scan_tiles; i += blockDim.x) ss.status[i] = 0ull;
    if (threadIdx.x == 0) *ss.counter = 0u;
  }
  for (int b = threadIdx.x; b < kGroupBuckets; b += blockDim.x) s_h[b] = 0;
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * kGroupTile;
  if (K == 27 && !(mode == 2 && order_in != nullptr)) {
    // 3^3 tables: a warp reads 32 consecutive rows (864 contiguous words) with
    // 27 coalesced loads; ballot j holds the hit bits of words 32 j .. 32 j + 31,
    // so the 864-bit stream is the rows' 27-bit hit masks back to back
    __shared__ uint32_t s_bal[kHistThreads / 32][27];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t words = cap * 27;
    for (int g = warp * 32; g < kGroupTile; g += blockDim.x) {
      const int64_t rb = r0 + g;
      if (rb >= n) break;  // warp-uniform
      // all 27 loads in flight before the first ballot (clamped, unconditional)
      int32_t v[27];
#pragma unroll
      for (int j = 0; j < 27; ++j) v[j] = __ldg(table + min(rb * 27 + j * 32 + lane, words - 1));
#pragma unroll
      for (int j = 0; j < 27; ++j) {
        const bool hit = rb * 27 + j * 32 + lane < words && v[j] >= 0;
        const uint32_t b = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) s_bal[warp][j] = b;
      }
      __syncwarp();
      const int64_t r = rb + lane;
      int key = kGroupBuckets + lane;  // dead lanes: unique dummy keys
      if (r < n) {
        const int st = 27 * lane, wi = st >> 5, off = st & 31;
        uint32_t m = s_bal[warp][wi] >> off;
        if (off > 5) m |= s_bal[warp][wi + 1] << (32 - off);
        m &= (1u << 27) - 1u;
        if (mode == 2) {
          masks[r] = m;
          key = (int)((m >> shift) & (kGroupBuckets - 1));
        } else {
          key = key_of_mask27(m, mode);
          if (masks != nullptr) masks[r] = m;  // the tile schedule's costs
        }
        if (desc) key = kGroupBuckets - 1 - key;
        keys[r] = (uint16_t)key;
      }
      // neighbouring rows share keys: one shared atomic per distinct key in the warp (a count)
      const unsigned same = __match_any_sync(0xffffffffu, key);
      if (key < kGroupBuckets && (same & ((1u << lane) - 1u)) == 0) atomicAdd(&s_h[key], __popc(same));
      __syncwarp();
    }
  } else
  for (int i = threadIdx.x; i < kGroupTile; i += blockDim.x) {
    const int64_t r = r0 + i;
    if (r < n) {
      int key;
      if (mode == 2) {  // position r of the previous pass's order
        uint32_t m;
        if (order_in == nullptr) {
          m = full_mask(table + r * K, K);
          masks[r] = m;
        } else {
          m = masks[order_in[r]];
        }
        key = (int)((m >> shift) & (kGroupBuckets - 1));
      } else {
        key = group_key(table + r * K, K, mode);
        if (masks != nullptr) masks[r] = full_mask(table + r * K, K);  // the tile schedule's costs
      }
      if (desc) key = kGroupBuckets - 1 - key;  // descending key order (every digit of the mask in mode 2)
      keys[r] = (uint16_t)key;
      atomicAdd(&s_h[key], 1);  // a count: order-independent
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kGroupBuckets; b += blockDim.x) hist[(int64_t)b * nblocks + blockIdx.x] = s_h[b];
}

// exclusive scan of hist in place (bucket-major: bucket b's rows of block j
// start at the sum over all (bucket < b) plus (bucket b, block < j)):
// single pass, kScanTile entries per block, decoupled look-back across tiles
__global__ void __launch_bounds__(1024) group_scan_kernel(int32_t* hist, int total, ScanState ss) {
  ::vp::pdl_begin();
  __shared__ int s_warp[1024 / 32 + 1];
  __shared__ int s_tile;
  __shared__ long long s_prefix;
  if (threadIdx.x == 0) s_tile = scan_next_tile(ss);
  __syncthreads();
  const int tile = s_tile;
  const int i0 = tile * kScanTile + threadIdx.x * 4;
  int v[4], sum = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    v[j] = i0 + j < total ? hist[i0 + j] : 0;
    sum += v[j];
  }
  int tot;
  const int excl = block_exclusive_scan<1024>(sum, s_warp, &tot);
  if (threadIdx.x < 32) {
    const long long p = scan_lookback_warp(ss, tile, tot);
    if (threadIdx.x == 0) s_prefix = p;
  }
  __syncthreads();
  int run = (int)s_prefix + excl;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (i0 + j < total) hist[i0 + j] = run;
    run += v[j];
  }
}

// stable scatter: warp w walks rows [w*256, w*256+256) of the block tile in
// order; ranks within a 32-row group from __match_any_sync; per-(warp,
// bucket) bases = the block's scanned base + the earlier warps' counts
__global__ void __launch_bounds__(kGroupThreads)
group_scatter_kernel(const uint16_t* __restrict__ keys, const int32_t* n_dev, int64_t cap,
                     const int32_t* __restrict__ offs, int nblocks, int32_t* __restrict__ perm,
                     const int32_t* __restrict__ order_in) {
  ::vp::pdl_begin();
  constexpr int W = kGroupThreads / 32, RW = kGroupTile / W;
  __shared__ int s_cnt[W][kGroupBuckets];
  const int n = load_count(n_dev, cap);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < W * kGroupBuckets; e += blockDim.x) (&s_cnt[0][0])[e] = 0;
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * kGroupTile + warp * RW;
  for (int g = 0; g < RW; g += 32) {  // per-warp counts (shared atomics: counts only)
    const int64_t r = r0 + g + lane;
    if (r < n) atomicAdd(&s_cnt[warp][keys[r]], 1);
  }
  __syncthreads();
  // base[w][b] = offs[b][block] + sum_{w' < w} cnt[w'][b]  (in place)
  for (int b = threadIdx.x; b < kGroupBuckets; b += blockDim.x) {
    int acc = offs[(int64_t)b * nblocks + blockIdx.x];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const int c = s_cnt[w][b];
      s_cnt[w][b] = acc;
      acc += c;
    }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int g = 0; g < RW; g += 32) {
    const int64_t r = r0 + g + lane;
    const bool live = r < n;
    const int key = live ? (int)keys[r] : kGroupBuckets + lane;  // dead lanes: unique dummy keys
    const unsigned m = __match_any_sync(0xffffffffu, key);
    if (live) {
      const int pos = s_cnt[warp][key] + __popc(m & lt);
      perm[pos] = order_in ? order_in[r] : (int32_t)r;
    }
    __syncwarp();
    if (live && (m & lt) == 0) s_cnt[warp][key] += __popc(m);  // the group's leader advances the base
    __syncwarp();
  }
}

// ---------------------------------------------------------------- tile schedule
// The conv kernels hand 128-row tiles to CTAs round-robin (tile p -> CTA
// p % G, G = the launch's CTA count) and a tile costs one gather stage per
// offset any of its rows uses, so after the grouping tile costs range 2..27
// active offsets and, with 2-4 tiles per CTA, the CTA that drew the heavy
// ones sets the kernel's duration (C3 level 1: slowest CTA 28 stages against
// a mean of 15.5, tools/cta_probe.py).  The schedule moves whole 128-row
// tiles: every row keeps its tile mates and so its exact accumulation; only
// which CTA runs the tile (and the order of the per-CTA BN partial sums)
// changes.  LPT by rounds with the round-robin slot counts (below); the
// ragged last tile keeps the last position, so a scheduled grouping sorts by
// DESCENDING key: the partial tile then holds the rows with the fewest
// neighbour columns (with ascending keys it held the densest rows and its
// CTA, one with the most slots, set the duration).  Applied when G < tiles
// <= kSchedRounds G (the regime where a few heavy tiles per CTA decide the
// duration); outside it the order is the descending-key grouping.
constexpr int kSchedRounds = 4;
constexpr int kSchedOvh = 3;  // per-item overhead in active-offset units (~1 us vs ~0.22-0.45 us per offset)

__device__ __forceinline__ bool sched_on(int ntiles, int G) {
  return G > 0 && G <= 1024 && ntiles > G && ntiles <= kSchedRounds * G && ntiles <= kSchedRounds * 1024;
}

// active offsets of each 128-row tile of the grouped order: OR of its rows'
// hit masks (written by the hist kernel), one warp per tile
__global__ void __launch_bounds__(256)
tile_cost_kernel(const uint32_t* __restrict__ masks, const int32_t* __restrict__ order, const int32_t* n_dev,
                 int64_t cap, int K, int G, int32_t* __restrict__ cost) {
  ::vp::pdl_begin();
  const int n = load_count(n_dev, cap);
  const int ntiles = (n + 127) / 128;
  if (!sched_on(ntiles, G) || K > 27) return;
  const int lane = threadIdx.x & 31;
  for (int t = blockIdx.x * 8 + (threadIdx.x >> 5); t < ntiles; t += gridDim.x * 8) {
    uint32_t m = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t r = (int64_t)t * 128 + q * 32 + lane;
      if (r < n) m |= __ldg(masks + __ldg(order + r));
    }
    m = __reduce_or_sync(0xffffffffu, m);
    if (lane == 0) cost[t] = __popc(m);
  }
}

// tile_at[position] = grouped tile placed there (identity when off).  One
// block of 32 ceil(G / 32) threads: a stable counting sort of the full tiles
// by descending cost (per-warp counts, ordered per-warp scatter), then LPT
// by rounds (2-4): in each round every CTA with a free slot takes one tile;
// the CTAs ranked by (load, free slots, index) ascending take the next tiles
// in descending cost (heaviest tile -> least-loaded CTA; among equal loads
// the CTA with fewer slots takes the heavier tile).  Thread b is CTA b; its
// rank is a count over the broadcast keys.
constexpr int kSchedMaxTiles = kSchedRounds * 1024;

__global__ void __launch_bounds__(1024)
tile_assign_kernel(const int32_t* __restrict__ cost, const int32_t* n_dev, int64_t cap, int K, int G,
                   int32_t* __restrict__ tile_at) {
  ::vp::pdl_begin();
  __shared__ int s_cnt[32][28];
  __shared__ int16_t s_sorted[kSchedMaxTiles];
  __shared__ uint32_t s_key[1024];
  const int n = load_count(n_dev, cap);
  const int ntiles = (n + 127) / 128;
  if (!sched_on(ntiles, G) || K > 27) {
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) tile_at[t] = t;
    return;
  }
  const int nfull = n / 128;  // tiles of 128 live rows; a ragged tile keeps position ntiles - 1
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  // -- stable sort of tiles [0, nfull) by key K - cost (descending cost)
  for (int e = threadIdx.x; e < 32 * 28; e += blockDim.x) (&s_cnt[0][0])[e] = 0;
  __syncthreads();
  const int chunk = (nfull + nwarps - 1) / nwarps;  // tiles per warp, contiguous
  const int t0 = min(nfull, warp * chunk), t1 = min(nfull, t0 + chunk);
  for (int t = t0 + lane; t < t1; t += 32) atomicAdd(&s_cnt[warp][K - __ldg(cost + t)], 1);  // counts only
  __syncthreads();
  if (warp == 0) {  // exclusive scan, key-major then warp order
    int base = 0;
    for (int key = 0; key <= K; ++key) {
      const int v = lane < nwarps ? s_cnt[lane][key] : 0;
      int inc = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += u;
      }
      if (lane < nwarps) s_cnt[lane][key] = base + inc - v;
      base += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int g = t0; g < t1; g += 32) {
    const int t = g + lane;
    const bool live = t < t1;
    const int key = live ? K - __ldg(cost + t) : 64 + lane;  // dead lanes: unique dummy keys
    const unsigned m = __match_any_sync(0xffffffffu, key);
    if (live) s_sorted[s_cnt[warp][key] + __popc(m & lt)] = (int16_t)t;
    __syncwarp();
    if (live && (m & lt) == 0) s_cnt[warp][key] += __popc(m);
    __syncwarp();
  }
  __syncthreads();
  // -- LPT by rounds over CTA b's round-robin positions b, b + G, ...
  const int R = ntiles / G, rem = ntiles % G;
  const int b = threadIdx.x;
  int slots = b < G ? R + (b < rem ? 1 : 0) : 0;
  int used = 0, load = 0;
  if (nfull < ntiles && b == (ntiles - 1) % G) {  // the ragged tile holds this CTA's last slot
    load = __ldg(cost + ntiles - 1) + kSchedOvh;
    --slots;
    tile_at[ntiles - 1] = ntiles - 1;
  }
  int next = 0;  // sorted tiles assigned so far
  while (next < nfull) {
    // load < 2^8 (<= 4 tiles of <= 27 + kSchedOvh), free slots < 8, b < 1024
    const uint32_t mine = used < slots ? ((uint32_t)load << 13) | ((uint32_t)(slots - used) << 10) | (uint32_t)b
                                       : 0xffffffffu;
    s_key[b] = mine;
    __syncthreads();
    int rank = 0, navail = 0;
    for (int j = 0; j < G; ++j) {
      const uint32_t kj = s_key[j];  // broadcast
      rank += kj < mine;
      navail += kj != 0xffffffffu;
    }
    const int take = min(navail, nfull - next);
    if (mine != 0xffffffffu && rank < take) {
      const int t = s_sorted[next + rank];
      tile_at[b + used * G] = t;
      ++used;
      load += __ldg(cost + t) + kSchedOvh;
    }
    next += take;
    __syncthreads();
  }
}

// table_sorted[i, :] = table[perm[i], :] (coalesced writes); with a tile
// schedule, position i reads grouped row tile_at[i / 128] * 128 + i % 128 and
// perm_out receives the composed permutation
__global__ void permute_rows_kernel(const int32_t* __restrict__ table, const int32_t* __restrict__ perm,
                                    const int32_t* n_dev, int64_t cap, int K, int32_t* __restrict__ out,
                                    const int32_t* __restrict__ tile_at, int32_t* __restrict__ perm_out) {
  ::vp::pdl_begin();
  const int n = load_count(n_dev, cap);
  if (K == 27) {
    // a warp writes 32 output rows (864 contiguous words): one perm load per
    // lane, the source rows by shuffle, then 27 independent gathered loads in
    // flight and 27 coalesced stores
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t rb = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; rb < n; rb += nwarps * 32) {
      const int64_t i = rb + lane;
      int32_t row = 0;
      if (i < n) {
        const int64_t src = tile_at ? (int64_t)__ldg(tile_at + (i >> 7)) * 128 + (i & 127) : i;
        row = __ldg(perm + src);
        if (perm_out != nullptr) perm_out[i] = row;
      }
      const int live = (int)(n - rb < 32 ? n - rb : 32) * 27;
      int32_t v[27];
#pragma unroll
      for (int j = 0; j < 27; ++j) {
        const int w = j * 32 + lane;
        const int r = __shfl_sync(0xffffffffu, row, w / 27);
        v[j] = w < live ? __ldg(table + (int64_t)r * 27 + (w - (w / 27) * 27)) : 0;
      }
#pragma unroll
      for (int j = 0; j < 27; ++j) {
        const int w = j * 32 + lane;
        if (w < live) out[rb * 27 + w] = v[j];
      }
    }
    return;
  }
  const int64_t total = (int64_t)n * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / K;
    const int k = (int)(e - i * K);
    const int64_t src = tile_at ? (int64_t)__ldg(tile_at + (i >> 7)) * 128 + (i & 127) : i;
    const int32_t row = __ldg(perm + src);
    out[e] = __ldg(table + (int64_t)row * K + k);
    if (perm_out != nullptr && k == 0) perm_out[i] = row;
  }
}

}  // namespace vp

using namespace vp;

extern "C" {

size_t vp_kernel_map_sort_ws_bytes(int64_t cap, int32_t K) {
  (void)K;
  const int64_t nblocks = ceil_div(std::max<int64_t>(cap, 1), kGroupTile);
  Carver c(nullptr, 0);
  c.take<uint16_t>(std::max<int64_t>(cap, 1));
  c.take<int32_t>(nblocks * kGroupBuckets);
  c.take<unsigned int>(4);
  c.take<unsigned long long>(ceil_div(nblocks * kGroupBuckets, kScanTile));
  c.take<uint32_t>(std::max<int64_t>(cap, 1));  // full-mask mode: masks + an order buffer
  c.take<int32_t>(std::max<int64_t>(cap, 1));
  c.take<int32_t>(ceil_div(std::max<int64_t>(cap, 1), 128));  // tile schedule: costs + placement
  c.take<int32_t>(ceil_div(std::max<int64_t>(cap, 1), 128));
  return c.off;
}

int vp_kernel_map_group_sched(const int32_t* table, const int32_t* n_dev, int64_t cap, int32_t K, int32_t key_mode,
                              int32_t sched_grid, int32_t* perm, int32_t* table_sorted, void* ws, size_t ws_bytes,
                              vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(sched_grid >= 0, VP_EVALIDATION, "kernel_map_group: schedule grid must be >= 0");
  VP_REQUIRE(K >= 1 && K <= VP_MAX_OFFSETS, VP_EVALIDATION, "kernel offset count out of range");
  VP_REQUIRE(key_mode >= 0 && key_mode <= 2, VP_EVALIDATION, "kernel_map_group: key mode must be 0, 1 or 2");
  if (cap <= 0) return VP_OK;
  VP_REQUIRE(cap < (1ll << 31), VP_EVALIDATION, "kernel_map_group: too many rows");
  const int nblocks = (int)ceil_div(cap, kGroupTile);
  Carver c(ws, ws_bytes);
  uint16_t* keys = c.take<uint16_t>(cap);
  int32_t* hist = c.take<int32_t>((int64_t)nblocks * kGroupBuckets);
  const int total = nblocks * kGroupBuckets;
  const int scan_tiles = (int)ceil_div(total, kScanTile);
  ScanState ss{c.take<unsigned int>(4), nullptr};
  ss.status = c.take<unsigned long long>(scan_tiles);
  uint32_t* masks = c.take<uint32_t>(cap);
  int32_t* order = c.take<int32_t>(cap);
  const int64_t tiles_cap = ceil_div(cap, 128);
  int32_t* tcost = c.take<int32_t>(tiles_cap);
  int32_t* tile_at = c.take<int32_t>(tiles_cap);
  VP_REQUIRE(c.ok(), VP_EVALIDATION, "kernel_map_group: workspace too small");
  const bool sched = sched_grid > 0;
  // one pass (9-bit key) or three stable LSD passes over the 27-bit mask,
  // alternating between `order` and `perm` so the last pass lands in perm
  // (with a tile schedule: in `order`, and the permute writes perm)
  const int passes = key_mode == 2 ? 3 : 1;
  int32_t* bufs[2] = {sched ? order : perm, sched ? perm : order};  // pass p writes bufs[p % 2]
  for (int ps = 0; ps < passes; ++ps) {
    const int32_t* in = ps == 0 ? nullptr : bufs[(ps - 1) % 2];
    int32_t* out = bufs[ps % 2];
    ::vp::launch(group_hist_kernel, nblocks, kHistThreads, 0, st, table, n_dev, cap, K, key_mode, keys, hist, nblocks,
                 ss, scan_tiles, (key_mode == 2 || (sched && ps == 0)) ? masks : nullptr, in, 9 * ps, (int)sched);
    VP_CHECK_LAUNCH("map_group: hist");
    ::vp::launch(group_scan_kernel, scan_tiles, 1024, 0, st, hist, total, ss);
    VP_CHECK_LAUNCH("map_group: scan");
    ::vp::launch(group_scatter_kernel, nblocks, kGroupThreads, 0, st, (const uint16_t*)keys, n_dev, cap,
                 (const int32_t*)hist, nblocks, out, in);
    VP_CHECK_LAUNCH("map_group: scatter");
  }
  const int pblocks = (int)std::min<int64_t>(ceil_div(cap * K, 256), grid_cap(16));
  if (!sched) {
    ::vp::launch(permute_rows_kernel, pblocks, 256, 0, st, table, (const int32_t*)perm, n_dev, cap, K, table_sorted,
                 (const int32_t*)nullptr, (int32_t*)nullptr);
    VP_CHECK_LAUNCH("map_group: permute");
    return VP_OK;
  }
  if (tiles_cap <= sched_grid || sched_grid > 1024 || K > 27) {  // no tile moves possible: descending order only
    ::vp::launch(permute_rows_kernel, pblocks, 256, 0, st, table, (const int32_t*)order, n_dev, cap, K, table_sorted,
                 (const int32_t*)nullptr, perm);
    VP_CHECK_LAUNCH("map_group: permute");
    return VP_OK;
  }
  ::vp::launch(tile_cost_kernel, (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(tiles_cap, 8), grid_cap(8))), 256,
               0, st, (const uint32_t*)masks, (const int32_t*)order, n_dev, cap, K, (int)sched_grid, tcost);
  VP_CHECK_LAUNCH("map_group: tile cost");
  const int athreads = (int)std::min<int64_t>(1024, ceil_div(std::max<int32_t>(sched_grid, 32), 32) * 32);
  ::vp::launch(tile_assign_kernel, 1, athreads, 0, st, (const int32_t*)tcost, n_dev, cap, K, (int)sched_grid, tile_at);
  VP_CHECK_LAUNCH("map_group: tile assign");
  ::vp::launch(permute_rows_kernel, pblocks, 256, 0, st, table, (const int32_t*)order, n_dev, cap, K, table_sorted,
               (const int32_t*)tile_at, perm);
  VP_CHECK_LAUNCH("map_group: permute");
  return VP_OK;
}

int vp_kernel_map_group(const int32_t* table, const int32_t* n_dev, int64_t cap, int32_t K, int32_t key_mode,
                        int32_t* perm, int32_t* table_sorted, void* ws, size_t ws_bytes, vp_stream_t stream) {
  return vp_kernel_map_group_sched(table, n_dev, cap, K, key_mode, 0, perm, table_sorted, ws, ws_bytes, stream);
}

// the operator-API entry point: plane key (good for stride-1 and strided tables alike)
int vp_kernel_map_sort(const int32_t* table, const int32_t* n_dev, int64_t cap, int32_t K, int32_t* perm,
                       int32_t* table_sorted, void* ws, size_t ws_bytes, vp_stream_t stream) {
  return vp_kernel_map_group(table, n_dev, cap, K, 1, perm, table_sorted, ws, ws_bytes, stream);
}

}  // extern "C"
