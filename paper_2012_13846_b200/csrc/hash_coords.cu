// Coordinate hash, packing, validation, strided output coordinates and
// voxelization — the integer stage that precedes the kernel map.
//
// Reference anchors: _kernels.pyx:16-73 (hash), kernels.py:53-79 (packing),
// tensor.py:28-78 (SparseTensor invariants), conv.py:124-146 (output
// coordinates), tensor.py:132-229 (voxelize + batch).
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace vp {

static thread_local std::string g_last_error;
static thread_local long long g_kernel_launches = 0;  // diagnostic: kernels enqueued by this thread

void set_error(const std::string& msg) { g_last_error = msg; }

int check_launch(const char* what, int kernels) {
  g_kernel_launches += kernels;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return VP_EINTERNAL;
  }
  return VP_OK;
}

uint64_t hash_cap_for(int64_t n) {
  // _kernels.pyx:27-29 — pow2 >= 2n+2, min 8
  uint64_t cap = 8;
  while (cap < (uint64_t)(2 * n + 2)) cap <<= 1;
  return cap;
}

uint64_t hash_cap_internal(int64_t n) {
  // internal tables (maps, coordinates): load factor <= 1/4 so most probes
  // resolve in the first 4-slot group (the slot layout is not semantic)
  uint64_t cap = 8;
  while (cap < (uint64_t)(4 * n + 4)) cap <<= 1;
  return cap;
}

__global__ void hash_clear_kernel(Slot* t, uint64_t cap) {
  ::vp::pdl_begin();
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (; i <= cap; i += stride) {
    uint4 v;
    v.x = 0xffffffffu;
    v.y = 0xffffffffu;
    v.z = 0u;
    v.w = 0u;
    reinterpret_cast<uint4*>(t)[i] = v;
  }
}

int hash_clear(Slot* t, uint64_t cap, cudaStream_t st) {
  int blocks = (int)std::min<uint64_t>((cap + 1 + 255) / 256, (uint64_t)grid_cap(8));
  ::vp::launch(hash_clear_kernel, blocks, 256, 0, st, t, cap);
  VP_CHECK_LAUNCH("hash_clear");
  return VP_OK;
}

// ------------------------------------------------------------------ raw key hash
__global__ void hash_build_keys_kernel(const int64_t* __restrict__ keys, const int32_t* n_dev,
                                       int64_t cap_n, Slot* t, uint64_t cap) {
  ::vp::pdl_begin();
  int n = load_count(n_dev, cap_n);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    hash_insert(t, cap, (uint64_t)keys[i], (int)i);
}

__global__ void hash_lookup_keys_kernel(const Slot* __restrict__ t, uint64_t cap,
                                        const int64_t* __restrict__ q, int64_t m,
                                        int64_t* __restrict__ rows) {
  ::vp::pdl_begin();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    rows[i] = hash_find(t, cap, (uint64_t)q[i]);
}

// ------------------------------------------------------------------ packing
__global__ void pack_coords_kernel(const int4* __restrict__ c, int64_t n, int64_t* keys,
                                   int32_t* bad) {
  ::vp::pdl_begin();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int4 r = c[i];
    if (!packable(r.x, r.y, r.z, r.w)) {
      if (bad) atomicOr(bad, 1);
      keys[i] = 0;
    } else {
      keys[i] = (int64_t)pack_key(r.x, r.y, r.z, r.w);
    }
  }
}

// ------------------------------------------------------------------ validation
// tensor.py:49-78 invariants. Duplicates via a hash insert where the second
// occurrence of a key sees a different first row.
__global__ void validate_insert_kernel(const int4* __restrict__ c, const int32_t* n_dev,
                                       int64_t cap_n, int sx, int sy, int sz, Slot* t,
                                       uint64_t cap, int32_t* flags) {
  ::vp::pdl_begin();
  int n = load_count(n_dev, cap_n);
  int f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int4 r = c[i];
    if (r.x < 0) f |= 2;
    if ((r.y % sx) || (r.z % sy) || (r.w % sz)) f |= 4;
    if (!packable(r.x, r.y, r.z, r.w)) {
      f |= 8;
      continue;
    }
    hash_insert(t, cap, pack_key(r.x, r.y, r.z, r.w), (int)i);
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

__global__ void validate_dup_kernel(const int4* __restrict__ c, const int32_t* n_dev, int64_t cap_n,
                                    const Slot* __restrict__ t, uint64_t cap, int32_t* flags) {
  ::vp::pdl_begin();
  int n = load_count(n_dev, cap_n);
  int f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int4 r = c[i];
    if (!packable(r.x, r.y, r.z, r.w)) continue;
    if (hash_find(t, cap, pack_key(r.x, r.y, r.z, r.w)) != (int)i) f |= 1;
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

__global__ void finite_kernel(const void* p, int dtype, int64_t count, int32_t* flags) {
  ::vp::pdl_begin();
  int f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = ldf(p, dtype, i);
    if (dtype == VP_F64) {
      double d = reinterpret_cast<const double*>(p)[i];
      if (!isfinite(d)) f = 16;
    } else if (!isfinite(v)) {
      f = 16;
    }
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

// ------------------------------------------------------------------ output coords
// conv.py:142-146: rows[:,1:] = floor(rows[:,1:] / step) * step, unique in
// first-seen order.  Pass 1 inserts every downsampled row keyed to its first
// input row; pass 2 keeps row i iff it is that first row and compacts with a
// single-pass decoupled look-back scan (ascending i == first-seen order).
__device__ __forceinline__ int floordiv_mul(int a, int s) {
  int q = a / s;
  if ((a % s) != 0 && ((a < 0) != (s < 0))) --q;
  return q * s;
}

// a downsampled row that leaves the 16-bit packed range (e.g. x = -32768
// floored to a multiple of 3) cannot be keyed: flag it, and the compaction
// reports n_out = -1 so the caller takes the wide-row path (vp_wide_*),
// instead of merging rows whose packed keys collide
__device__ __forceinline__ bool axis_packable(int v) { return v >= kAxisMin && v <= kAxisMax; }

__global__ void oc_insert_kernel(const int4* __restrict__ in, const int32_t* n_dev, int64_t cap_n,
                                 int sx, int sy, int sz, Slot* t, uint64_t cap, unsigned int* unpackable) {
  ::vp::pdl_begin();
  int n = load_count(n_dev, cap_n);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int4 r = in[i];
    const int x = floordiv_mul(r.y, sx), y = floordiv_mul(r.z, sy), z = floordiv_mul(r.w, sz);
    if (!(axis_packable(x) && axis_packable(y) && axis_packable(z))) *unpackable = 1u;
    hash_insert(t, cap, pack_key(r.x, x, y, z), (int)i);
  }
}

constexpr int kCompactBlock = 256;
constexpr int kCompactItems = 16;  // rows per thread (tile 4096 -> short look-back chains)
constexpr int kCompactTile = kCompactBlock * kCompactItems;

// first_of[i] = first (minimum) input row whose (downsampled) key equals row
// i's; one row per thread so every lookup is an independent memory request.
__global__ void first_of_kernel(const int4* __restrict__ rows, const int32_t* n_dev, int64_t cap_n, int sx, int sy,
                                int sz, const Slot* __restrict__ t, uint64_t cap, int32_t* __restrict__ first_of) {
  ::vp::pdl_begin();
  const int n = load_count(n_dev, cap_n);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int4 r = rows[i];
    first_of[i] = hash_find(t, cap, pack_key(r.x, floordiv_mul(r.y, sx), floordiv_mul(r.z, sy), floordiv_mul(r.w, sz)));
  }
}

// Ordered compaction of the first-occurrence rows (first_of[i] == i) with a
// single-pass decoupled look-back scan: out keeps ascending i == first-seen
// order (conv.py:145-146, tensor.py:138-144).  rank_of_first (nullable)
// receives each kept row's output position.
__global__ void __launch_bounds__(kCompactBlock)
compact_first_kernel(const int4* __restrict__ rows, const int32_t* n_dev, int64_t cap_n, int sx, int sy, int sz,
                     const int32_t* __restrict__ first_of, ScanState ss, int4* __restrict__ out, int32_t* n_out,
                     int32_t* rank_of_first, const unsigned int* unpackable) {
  ::vp::pdl_begin();
  __shared__ int s_tile;
  __shared__ int s_warp[kCompactBlock / 32 + 1];
  __shared__ long long s_prefix;
  const int n = load_count(n_dev, cap_n);
  if (threadIdx.x == 0) s_tile = scan_next_tile(ss);
  __syncthreads();
  const int tile = s_tile;
  const int64_t base = (int64_t)tile * kCompactTile;
  if (base >= n && tile > 0) return;  // past the end: nobody waits on us
  const int64_t i0 = base + (int64_t)threadIdx.x * kCompactItems;
  int flags = 0;
#pragma unroll
  for (int j = 0; j < kCompactItems; ++j) {
    const int64_t i = i0 + j;
    if (i < n && __ldg(first_of + i) == (int)i) flags |= 1 << j;
  }
  int cnt = __popc(flags), total;
  int excl = block_exclusive_scan<kCompactBlock>(cnt, s_warp, &total);
  if (threadIdx.x < 32) {
    long long p = scan_lookback_warp(ss, tile, total);
    if (threadIdx.x == 0) s_prefix = p;
  }
  __syncthreads();
  long long pos = s_prefix + excl;
#pragma unroll
  for (int j = 0; j < kCompactItems; ++j) {
    if (flags & (1 << j)) {
      int4 r = rows[i0 + j];
      r.y = floordiv_mul(r.y, sx);
      r.z = floordiv_mul(r.z, sy);
      r.w = floordiv_mul(r.w, sz);
      if (rank_of_first) rank_of_first[i0 + j] = (int)pos;
      out[pos++] = r;
    }
  }
  if (n == 0 && tile == 0 && threadIdx.x == 0) *n_out = 0;
  const int64_t last = (int64_t)n - 1;
  if (last >= base && last < base + kCompactTile && threadIdx.x == 0)
    *n_out = (unpackable && *unpackable) ? -1 : (int)(s_prefix + total);
}

// parent[i] = output row of input row i = rank of its first row
__global__ void oc_parent_kernel(const int32_t* n_dev, int64_t cap_n, const int32_t* first_of,
                                 const int32_t* rank_of_first, int32_t* parent) {
  ::vp::pdl_begin();
  int n = load_count(n_dev, cap_n);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    parent[i] = rank_of_first[first_of[i]];
}

// ------------------------------------------------------------------ voxelize
// tensor.py:171-175: floor(p / voxel_size) (f64), clip [0, res-1], prepend
// batch index; tensor.py:205-221: batch index = cloud position.
__device__ __forceinline__ int cloud_of(const int64_t* offs, int nc, int64_t i) {
  int lo = 0, hi = nc;  // offs[lo] <= i < offs[hi]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (offs[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int4 voxel_of(const void* pts, int dtype, int64_t i, double vs, int rx,
                                         int ry, int rz, int b) {
  double p0, p1, p2;
  if (dtype == VP_F64) {
    const double* q = reinterpret_cast<const double*>(pts) + 3 * i;
    p0 = q[0]; p1 = q[1]; p2 = q[2];
  } else {
    const float* q = reinterpret_cast<const float*>(pts) + 3 * i;
    p0 = (double)q[0]; p1 = (double)q[1]; p2 = (double)q[2];
  }
  // np.floor(points / voxel_size).astype(int64) then clip
  double f0 = floor(p0 / vs), f1 = floor(p1 / vs), f2 = floor(p2 / vs);
  long long v0 = f0 < 0 ? 0 : (f0 > rx - 1 ? rx - 1 : (long long)f0);
  long long v1 = f1 < 0 ? 0 : (f1 > ry - 1 ? ry - 1 : (long long)f1);
  long long v2 = f2 < 0 ? 0 : (f2 > rz - 1 ? rz - 1 : (long long)f2);
  return make_int4(b, (int)v0, (int)v1, (int)v2);
}

__global__ void vox_insert_kernel(const void* pts, int dtype, int64_t n, const int64_t* offs, int nc,
                                  double vs, int rx, int ry, int rz, Slot* t, uint64_t cap,
                                  int4* vox_tmp) {
  ::vp::pdl_begin();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int b = cloud_of(offs, nc, i);
    int4 v = voxel_of(pts, dtype, i, vs, rx, ry, rz, b);
    vox_tmp[i] = v;
    hash_insert(t, cap, pack_key(v.x, v.y, v.z, v.w), (int)i);
  }
}

__global__ void fill_kernel(void* p, int dtype, const int32_t* n_dev, int64_t cap, float v) {
  ::vp::pdl_begin();
  int n = load_count(n_dev, cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    stf(p, dtype, i, v);
}

// ------------------------------------------------------------------ voxel mean
// tensor.py:180-183: np.add.at(feats, group, features) accumulates in point
// order, then divides by the counts.  Deterministic restatement: count points
// per voxel (integer atomics are order-independent), scan to segment starts,
// drop point ids into their voxel's segment (slot order arbitrary), then each
// voxel sorts its own segment ascending (restoring point order) and sums in
// f64 in that order — the same summation order as np.add.at.
__global__ void vm_count_kernel(const int32_t* p2v, int64_t n, int32_t* counts) {
  ::vp::pdl_begin();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&counts[p2v[i]], 1);
}
__global__ void vm_scan_kernel(const int32_t* counts, const int32_t* n_vox_dev, int64_t cap_vox,
                               int32_t* starts, int32_t* cursor) {
  ::vp::pdl_begin();
  __shared__ int s_warp[1024 / 32 + 1];
  __shared__ int s_carry;
  int nv = load_count(n_vox_dev, cap_vox);
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nv; base += 1024) {
    int64_t i = base + threadIdx.x;
    int v = i < nv ? counts[i] : 0, tot;
    int e = block_exclusive_scan<1024>(v, s_warp, &tot);
    if (i < nv) {
      starts[i] = s_carry + e;
      cursor[i] = s_carry + e;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_carry += tot;
    __syncthreads();
  }
}
__global__ void vm_place_kernel(const int32_t* p2v, int64_t n, int32_t* cursor, int32_t* order) {
  ::vp::pdl_begin();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    order[atomicAdd(&cursor[p2v[i]], 1)] = (int32_t)i;
}
__global__ void vm_sum_kernel(const void* f, int dtype, int F, int32_t* order, const int32_t* starts,
                              const int32_t* counts, const int32_t* n_vox_dev, int64_t cap_vox,
                              float* out) {
  ::vp::pdl_begin();
  int nv = load_count(n_vox_dev, cap_vox);
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < nv;
       g += (int64_t)gridDim.x * blockDim.x) {
    int s = starts[g], c = counts[g];
    int32_t* seg = order + s;
    // restore point order inside the voxel (the sums run in point order,
    // tensor.py:171-184): insertion sort for the usual handful of points,
    // in-place heapsort (O(c log c)) when clipping piles many points into
    // one boundary voxel
    if (c <= 32) {
      for (int a = 1; a < c; ++a) {
        int32_t key = seg[a];
        int b = a - 1;
        while (b >= 0 && seg[b] > key) {
          seg[b + 1] = seg[b];
          --b;
        }
        seg[b + 1] = key;
      }
    } else {
      auto sift = [&](int root, int end) {
        while (2 * root + 1 < end) {
          int ch = 2 * root + 1;
          if (ch + 1 < end && seg[ch + 1] > seg[ch]) ++ch;
          if (seg[root] >= seg[ch]) break;
          const int32_t tmp = seg[root];
          seg[root] = seg[ch];
          seg[ch] = tmp;
          root = ch;
        }
      };
      for (int r = c / 2 - 1; r >= 0; --r) sift(r, c);
      for (int end = c - 1; end > 0; --end) {
        const int32_t tmp = seg[0];
        seg[0] = seg[end];
        seg[end] = tmp;
        sift(0, end);
      }
    }
    for (int j = 0; j < F; ++j) {
      double acc = 0.0;
      for (int k = 0; k < c; ++k) {
        int64_t i = seg[k];
        acc += dtype == VP_F64 ? reinterpret_cast<const double*>(f)[i * F + j]
                               : (double)reinterpret_cast<const float*>(f)[i * F + j];
      }
      out[g * F + j] = (float)(acc / (double)c);
    }
  }
}

}  // namespace vp

using namespace vp;

extern "C" {

const char* vp_last_error(void) { return g_last_error.c_str(); }
const char* vp_version(void) { return "voxpipe_b200 0.1.0 sm_100a"; }
long long vp_kernel_launches(void) { return g_kernel_launches; }

int64_t vp_hash_capacity(int64_t n) { return (int64_t)hash_cap_for(n); }
size_t vp_hash_bytes(int64_t cap) { return (size_t)(cap + 1) * sizeof(Slot); }

int vp_hash_build(const int64_t* keys, const int32_t* n_dev, int64_t cap_n, void* table,
                  int64_t table_cap, vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(table_cap >= 8 && (table_cap & (table_cap - 1)) == 0, VP_EVALIDATION,
             "table capacity must be a power of two >= 8");
  int r = hash_clear((Slot*)table, table_cap, st);
  if (r) return r;
  if (cap_n > 0) {
    int blocks = (int)std::min<int64_t>(ceil_div(cap_n, 256), grid_cap(8));
    ::vp::launch(hash_build_keys_kernel, blocks, 256, 0, st, keys, n_dev, cap_n, (Slot*)table, table_cap);
    VP_CHECK_LAUNCH("hash_build");
  }
  return VP_OK;
}

int vp_hash_lookup(const void* table, int64_t table_cap, const int64_t* q, int64_t m,
                   int64_t* rows, vp_stream_t stream) {
  if (m <= 0) return VP_OK;
  int blocks = (int)std::min<int64_t>(ceil_div(m, 256), grid_cap(8));
  ::vp::launch(hash_lookup_keys_kernel, blocks, 256, 0, (cudaStream_t)stream, (const Slot*)table, table_cap, q,
                                                                     m, rows);
  VP_CHECK_LAUNCH("hash_lookup");
  return VP_OK;
}

int vp_pack_coords(const int32_t* coords, int64_t n, int64_t* keys, int32_t* bad_dev,
                   vp_stream_t stream) {
  if (n <= 0) return VP_OK;
  int blocks = (int)std::min<int64_t>(ceil_div(n, 256), grid_cap(8));
  ::vp::launch(pack_coords_kernel, blocks, 256, 0, (cudaStream_t)stream, (const int4*)coords, n, keys, bad_dev);
  VP_CHECK_LAUNCH("pack_coords");
  return VP_OK;
}

size_t vp_validate_coords_ws_bytes(int64_t cap_n) {
  Carver c(nullptr, 0);
  c.take<Slot>(hash_cap_internal(cap_n) + 1);
  return c.off;
}

int vp_validate_coords(const int32_t* coords, const int32_t* n_dev, int64_t cap_n,
                       const int32_t* ts, int32_t* flags, void* ws, size_t ws_bytes,
                       vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  Carver c(ws, ws_bytes);
  uint64_t cap = hash_cap_internal(cap_n);
  Slot* t = c.take<Slot>(cap + 1);
  VP_REQUIRE(c.ok(), VP_EVALIDATION, "validate_coords: workspace too small");
  VP_REQUIRE(ts[0] > 0 && ts[1] > 0 && ts[2] > 0, VP_EVALIDATION, "tensor_stride entries must be positive");
  if (cap_n <= 0) return VP_OK;
  int r = hash_clear(t, cap, st);
  if (r) return r;
  int blocks = (int)std::min<int64_t>(ceil_div(cap_n, 256), grid_cap(8));
  ::vp::launch(validate_insert_kernel, blocks, 256, 0, st, (const int4*)coords, n_dev, cap_n, ts[0], ts[1], ts[2],
                                                 t, cap, flags);
  VP_CHECK_LAUNCH("validate_insert");
  ::vp::launch(validate_dup_kernel, blocks, 256, 0, st, (const int4*)coords, n_dev, cap_n, t, cap, flags);
  VP_CHECK_LAUNCH("validate_dup");
  return VP_OK;
}

int vp_check_finite(const void* feats, int32_t dtype, int64_t count, int32_t* flags,
                    vp_stream_t stream) {
  if (count <= 0) return VP_OK;
  int blocks = (int)std::min<int64_t>(ceil_div(count, 256), grid_cap(8));
  ::vp::launch(finite_kernel, blocks, 256, 0, (cudaStream_t)stream, feats, dtype, count, flags);
  VP_CHECK_LAUNCH("check_finite");
  return VP_OK;
}

size_t vp_output_coords_ws_bytes(int64_t cap_in) {
  Carver c(nullptr, 0);
  c.take<Slot>(hash_cap_internal(cap_in) + 1);
  int64_t tiles = ceil_div(std::max<int64_t>(cap_in, 1), kCompactTile);
  c.take<unsigned int>(4);
  c.take<unsigned long long>(tiles);
  c.take<unsigned int>(4);
  c.take<unsigned long long>(tiles);
  c.take<int32_t>(cap_in);  // first_of
  c.take<int32_t>(cap_in);  // rank_of_first
  return c.off;
}

int vp_output_coords(const int32_t* in, const int32_t* n_in_dev, int64_t cap_in, const int32_t* step,
                     int32_t* out, int32_t* n_out_dev, int32_t* parent, void* ws, size_t ws_bytes,
                     vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(step[0] > 0 && step[1] > 0 && step[2] > 0, VP_EVALIDATION,
             "stride must list D positive integers");
  Carver c(ws, ws_bytes);
  uint64_t cap = hash_cap_internal(cap_in);
  Slot* t = c.take<Slot>(cap + 1);
  int64_t tiles = ceil_div(std::max<int64_t>(cap_in, 1), kCompactTile);
  ScanState s1{c.take<unsigned int>(4), nullptr};
  s1.status = c.take<unsigned long long>(tiles);
  ScanState s2{c.take<unsigned int>(4), nullptr};
  s2.status = c.take<unsigned long long>(tiles);
  int32_t* first_of = c.take<int32_t>(cap_in);
  int32_t* rank_of_first = c.take<int32_t>(cap_in);
  VP_REQUIRE(c.ok(), VP_EVALIDATION, "output_coords: workspace too small");
  if (cap_in <= 0) {
    cudaMemsetAsync(n_out_dev, 0, sizeof(int32_t), st);
    VP_CHECK_ASYNC("output_coords(empty)");
    return VP_OK;
  }
  int r = hash_clear(t, cap, st);
  if (r) return r;
  cudaMemsetAsync(s1.counter, 0, 256 + tiles * 8, st);
  int blocks = (int)std::min<int64_t>(ceil_div(cap_in, 256), grid_cap(8));
  unsigned int* unpackable = s1.counter + 2;  // zeroed with the scan state above
  ::vp::launch(oc_insert_kernel, blocks, 256, 0, st, (const int4*)in, n_in_dev, cap_in, step[0], step[1], step[2],
                                           t, cap, unpackable);
  VP_CHECK_LAUNCH("oc_insert");
  (void)s2;
  ::vp::launch(first_of_kernel, (int)ceil_div(cap_in, 256), 256, 0, st, (const int4*)in, n_in_dev, cap_in, step[0], step[1],
                                                               step[2], t, cap, first_of);
  VP_CHECK_LAUNCH("oc_first_of");
  ::vp::launch(compact_first_kernel, (int)tiles, kCompactBlock, 0, st, (const int4*)in, n_in_dev, cap_in, step[0], step[1],
                                                             step[2], first_of, s1, (int4*)out, n_out_dev,
                                                             parent ? rank_of_first : nullptr,
                                                             (const unsigned int*)unpackable);
  VP_CHECK_LAUNCH("oc_compact");
  if (parent) {
    ::vp::launch(oc_parent_kernel, blocks, 256, 0, st, n_in_dev, cap_in, first_of, rank_of_first, parent);
    VP_CHECK_LAUNCH("oc_parent");
  }
  return VP_OK;
}

size_t vp_voxelize_ws_bytes(int64_t n) {
  Carver c(nullptr, 0);
  c.take<Slot>(hash_cap_internal(n) + 1);
  int64_t tiles = ceil_div(std::max<int64_t>(n, 1), kCompactTile);
  c.take<unsigned int>(4);
  c.take<unsigned long long>(tiles);
  c.take<int4>(n);
  c.take<int32_t>(n);
  c.take<int32_t>(n);
  return c.off;
}

int vp_voxelize(const void* points, int32_t pts_dtype, int64_t n, const int64_t* offs, int32_t nc,
                double vs, const int32_t* res, int32_t* coords_out, int32_t* n_out_dev,
                int32_t* p2v, void* feats_out, int32_t feat_dtype, void* ws, size_t ws_bytes,
                vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(vs > 0, VP_EVALIDATION, "voxel_size must be positive");
  VP_REQUIRE(res[0] >= 1 && res[1] >= 1 && res[2] >= 1, VP_EVALIDATION,
             "resolution must list D positive integers");
  VP_REQUIRE(res[0] <= 32768 && res[1] <= 32768 && res[2] <= 32768 && nc <= 65536, VP_EVALIDATION,
             "resolution / batch exceed the packable coordinate range");
  VP_REQUIRE(pts_dtype == VP_F32 || pts_dtype == VP_F64, VP_EVALIDATION, "points must be f32 or f64");
  Carver c(ws, ws_bytes);
  uint64_t cap = hash_cap_internal(n);
  Slot* t = c.take<Slot>(cap + 1);
  int64_t tiles = ceil_div(std::max<int64_t>(n, 1), kCompactTile);
  ScanState s1{c.take<unsigned int>(4), nullptr};
  s1.status = c.take<unsigned long long>(tiles);
  int4* vox = c.take<int4>(n);
  int32_t* first_of = c.take<int32_t>(n);
  int32_t* rank_of_first = c.take<int32_t>(n);
  VP_REQUIRE(c.ok(), VP_EVALIDATION, "voxelize: workspace too small");
  if (n <= 0) {
    cudaMemsetAsync(n_out_dev, 0, sizeof(int32_t), st);
    VP_CHECK_ASYNC("voxelize(empty)");
    return VP_OK;
  }
  int r = hash_clear(t, cap, st);
  if (r) return r;
  cudaMemsetAsync(s1.counter, 0, 256 + tiles * 8, st);
  int blocks = (int)std::min<int64_t>(ceil_div(n, 256), grid_cap(8));
  ::vp::launch(vox_insert_kernel, blocks, 256, 0, st, points, pts_dtype, n, offs, nc, vs, res[0], res[1], res[2],
                                            t, cap, vox);
  VP_CHECK_LAUNCH("vox_insert");
  ::vp::launch(first_of_kernel, (int)ceil_div(n, 256), 256, 0, st, vox, nullptr, n, 1, 1, 1, t, cap, first_of);
  VP_CHECK_LAUNCH("vox_first_of");
  ::vp::launch(compact_first_kernel, (int)tiles, kCompactBlock, 0, st, vox, nullptr, n, 1, 1, 1, first_of, s1,
                                                             (int4*)coords_out, n_out_dev,
                                                             p2v ? rank_of_first : nullptr, (const unsigned int*)nullptr);
  VP_CHECK_LAUNCH("vox_compact");
  if (p2v) {
    ::vp::launch(oc_parent_kernel, blocks, 256, 0, st, nullptr, n, first_of, rank_of_first, p2v);
    VP_CHECK_LAUNCH("vox_p2v");
  }
  if (feats_out) {
    ::vp::launch(fill_kernel, blocks, 256, 0, st, feats_out, feat_dtype, n_out_dev, n, 1.0f);
    VP_CHECK_LAUNCH("vox_fill");
  }
  return VP_OK;
}

size_t vp_voxel_mean_ws_bytes(int64_t n, int64_t cap_vox) {
  Carver c(nullptr, 0);
  c.take<int32_t>(cap_vox);  // counts
  c.take<int32_t>(cap_vox);  // starts
  c.take<int32_t>(cap_vox);  // cursor
  c.take<int32_t>(n);        // order
  return c.off;
}

int vp_voxel_mean(const void* feats_in, int32_t in_dtype, int64_t n, int32_t F, const int32_t* p2v,
                  const int32_t* n_vox_dev, int64_t cap_vox, float* out, void* ws, size_t ws_bytes,
                  vp_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  VP_REQUIRE(in_dtype == VP_F32 || in_dtype == VP_F64, VP_EVALIDATION, "features must be f32 or f64");
  Carver c(ws, ws_bytes);
  int32_t* counts = c.take<int32_t>(cap_vox);
  int32_t* starts = c.take<int32_t>(cap_vox);
  int32_t* cursor = c.take<int32_t>(cap_vox);
  int32_t* order = c.take<int32_t>(n);
  VP_REQUIRE(c.ok(), VP_EVALIDATION, "voxel_mean: workspace too small");
  if (n <= 0 || cap_vox <= 0) return VP_OK;
  cudaMemsetAsync(counts, 0, cap_vox * sizeof(int32_t), st);
  int blocks = (int)std::min<int64_t>(ceil_div(n, 256), grid_cap(8));
  ::vp::launch(vm_count_kernel, blocks, 256, 0, st, p2v, n, counts);
  VP_CHECK_LAUNCH("vm_count");
  ::vp::launch(vm_scan_kernel, 1, 1024, 0, st, counts, n_vox_dev, cap_vox, starts, cursor);
  VP_CHECK_LAUNCH("vm_scan");
  ::vp::launch(vm_place_kernel, blocks, 256, 0, st, p2v, n, cursor, order);
  VP_CHECK_LAUNCH("vm_place");
  int vblocks = (int)std::min<int64_t>(ceil_div(cap_vox, 128), grid_cap(8));
  ::vp::launch(vm_sum_kernel, vblocks, 128, 0, st, feats_in, in_dtype, F, order, starts, counts, n_vox_dev,
                                         cap_vox, out);
  VP_CHECK_LAUNCH("vm_sum");
  return VP_OK;
}

}  // extern "C"
