// Shared device helpers for the voxpipe_b200 sm_100a kernels.
#pragma once
#include <cstdlib>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>

#include "../../include/voxpipe_b200.h"

namespace vp {

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
int check_launch(const char* what, int kernels);

// after a kernel launch: counts it (vp_kernel_launches) and checks errors
#define VP_CHECK_LAUNCH(what)                    \
  do {                                           \
    int _st = ::vp::check_launch(what, 1);       \
    if (_st != VP_OK) return _st;                \
  } while (0)
// after a memset/memcpy: checks errors only
#define VP_CHECK_ASYNC(what)                     \
  do {                                           \
    int _st = ::vp::check_launch(what, 0);       \
    if (_st != VP_OK) return _st;                \
  } while (0)

#define VP_REQUIRE(cond, code, msg)              \
  do {                                           \
    if (!(cond)) {                               \
      ::vp::set_error(msg);                      \
      return code;                               \
    }                                            \
  } while (0)

constexpr int kNumSMs = 148;

// Block cap of the grid-stride kernels: per_sm blocks per SM, lowered by
// VP_GRID_PER_SM (tuning: in the training step these kernels share the GPU
// with the critical-path stream, where small grids interfere less).
inline int grid_cap(int per_sm) {
  static const int lim = getenv("VP_GRID_PER_SM") ? (atoi(getenv("VP_GRID_PER_SM")) > 0 ? atoi(getenv("VP_GRID_PER_SM")) : 1)
                                                  : (1 << 20);
  return kNumSMs * (per_sm < lim ? per_sm : lim);
}

// ------------------------------------------------------------------ launch
// Every kernel of the library is launched with Programmatic Dependent Launch
// (programmatic stream serialization): inside a captured step the next
// kernel's launch and scheduling overlap the current kernel's tail instead of
// paying a full launch gap on each of the ~200 dependent kernels.  Each
// kernel starts with pdl_begin(): griddepcontrol.wait (the previous grid has
// completed and its writes are visible) and only then launch_dependents, so
// at most two grids overlap and no kernel reads anything early.
template <typename... KArgs, typename... Args>
inline void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// launch() with a thread-block cluster of `cluster` CTAs along x (grid.x
// must be a multiple of it): CTAs of a cluster can combine their shared
// memory results (distributed shared memory) before one of them writes.
template <typename... KArgs, typename... Args>
inline void launch_cluster(void (*kernel)(KArgs...), int cluster, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                           Args... args) {
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cluster;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Cooperative launch (every block co-resident: grid-wide waits are safe);
// returns the launch status so the caller can fall back.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_coop(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                               Args... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef VP_PDL_EARLY_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Carve a caller workspace into aligned sub-buffers.
struct Carver {
  char* base;
  size_t off = 0;
  size_t cap;
  Carver(void* b, size_t c) : base((char*)b), cap(c) {}
  template <class T>
  T* take(size_t count) {
    off = align_up(off, 256);
    T* p = (T*)(base ? base + off : nullptr);
    off += count * sizeof(T);
    return p;
  }
  bool ok() const { return off <= cap; }
};

// ------------------------------------------------------------------ keys
// kernels.py:40-46 field layout
constexpr int64_t kAxisBias = 32768;
constexpr int64_t kAxisMin = -32768;
constexpr int64_t kAxisMax = 32767;
constexpr int64_t kBatchMax = 65535;
constexpr uint64_t kEmptyKey = ~0ull;

__device__ __forceinline__ bool packable(int b, int x, int y, int z) {
  return b >= 0 && b <= kBatchMax && x >= kAxisMin && x <= kAxisMax && y >= kAxisMin &&
         y <= kAxisMax && z >= kAxisMin && z <= kAxisMax;
}
__device__ __forceinline__ bool packable64(long long b, long long x, long long y, long long z) {
  return b >= 0 && b <= kBatchMax && x >= kAxisMin && x <= kAxisMax && y >= kAxisMin &&
         y <= kAxisMax && z >= kAxisMin && z <= kAxisMax;
}

// kernels.py:75-78 — batch<<48 | (x+bias)<<32 | (y+bias)<<16 | (z+bias)
__device__ __forceinline__ uint64_t pack_key(int b, int x, int y, int z) {
  return ((uint64_t)(uint32_t)b << 48) | ((uint64_t)(uint32_t)(x + kAxisBias) << 32) |
         ((uint64_t)(uint32_t)(y + kAxisBias) << 16) | (uint64_t)(uint32_t)(z + kAxisBias);
}

// _kernels.pyx:16-21 — splitmix64 finalizer
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// ------------------------------------------------------------------ hash table
// 16-byte slots: {key, ~row}. ~row == 0 means "no row" (row -1). The key
// kEmptyKey marks an unused slot; the one valid key equal to kEmptyKey
// (batch 65535, all axes 32767) lives in the extra slot `cap`.
struct alignas(16) Slot {
  unsigned long long key;
  unsigned int nrow;  // ~row
  unsigned int pad;
};

__device__ __forceinline__ void hash_insert(Slot* t, uint64_t cap, uint64_t key, int row) {
  unsigned int nrow = ~(unsigned int)row;
  if (key == kEmptyKey) {
    atomicMax(&t[cap].nrow, nrow);
    return;
  }
  uint64_t mask = cap - 1;
  uint64_t s = mix64(key) & mask;
  while (true) {
    unsigned long long prev = atomicCAS(&t[s].key, (unsigned long long)kEmptyKey,
                                        (unsigned long long)key);
    if (prev == kEmptyKey || prev == key) {
      // FIRST occurrence wins (_kernels.pyx:44-46): keep the minimum row
      atomicMax(&t[s].nrow, nrow);
      return;
    }
    s = (s + 1) & mask;
  }
}

// One 16-byte load per probe step (a random probe costs one L1 wavefront;
// at load factor <= 1/4 a lookup averages ~1.2-1.4 steps).
__device__ __forceinline__ int hash_find(const Slot* __restrict__ t, uint64_t cap, uint64_t key) {
  if (key == kEmptyKey) return (int)~t[cap].nrow;
  const uint64_t mask = cap - 1;
  uint64_t s = mix64(key) & mask;
  while (true) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(t + s));
    const unsigned long long k = ((unsigned long long)v.y << 32) | v.x;
    if (k == key) return (int)~v.z;
    if (k == kEmptyKey) return -1;
    s = (s + 1) & mask;
  }
}

__global__ void hash_clear_kernel(Slot* t, uint64_t cap);
int hash_clear(Slot* t, uint64_t cap, cudaStream_t st);
uint64_t hash_cap_for(int64_t n);
uint64_t hash_cap_internal(int64_t n);

// ------------------------------------------------------------------ counts
__device__ __forceinline__ int load_count(const int32_t* n_dev, int64_t cap) {
  return n_dev ? *n_dev : (int)cap;
}

// ------------------------------------------------------------------ scan
// Single-pass decoupled look-back scan state: a dynamic tile counter and a
// status word per tile (2-bit flag | 62-bit value). Zeroed before each use.
struct ScanState {
  unsigned int* counter;
  unsigned long long* status;
};
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPre = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Get a dynamic tile id (in launch order) — thread 0 only; broadcast by caller.
__device__ __forceinline__ int scan_next_tile(ScanState s) { return (int)atomicAdd(s.counter, 1u); }

// Warp-0 look-back: returns the exclusive prefix of `tile` given its
// aggregate. Must be called by all lanes of warp 0 (same args).
__device__ __forceinline__ long long scan_lookback_warp(ScanState s, int tile, long long agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_release(&s.status[0], kFlagPre | (unsigned long long)agg);
    return 0;
  }
  if (lane == 0) st_release(&s.status[tile], kFlagAgg | (unsigned long long)agg);
  long long excl = 0;
  int base = tile - 1;
  while (true) {
    int j = base - lane;
    unsigned long long v = 0;
    if (j >= 0) {
      do {
        v = ld_acquire(&s.status[j]);
      } while ((v >> 62) == 0);
    } else {
      v = kFlagPre;  // virtual prefix 0 before tile 0
    }
    unsigned pre = __ballot_sync(0xffffffffu, (v >> 62) == 2);
    long long val = (long long)(v & kValMask);
    if (pre) {
      int first = __ffs(pre) - 1;  // nearest predecessor with an inclusive prefix
      long long contrib = lane <= first ? val : 0;
      for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
      excl += contrib;
      break;
    }
    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
    excl += val;
    base -= 32;
  }
  if (lane == 0) st_release(&s.status[tile], kFlagPre | (unsigned long long)(excl + agg));
  return excl;
}

// Block-wide exclusive scan of one int per thread (BLOCK threads);
// returns exclusive prefix, writes block total to *total.
template <int BLOCK>
__device__ __forceinline__ int block_exclusive_scan(int v, int* smem_warp /*BLOCK/32+1*/, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < BLOCK / 32 ? smem_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < BLOCK / 32) smem_warp[lane] = w;  // inclusive per-warp prefix
    if (lane == BLOCK / 32 - 1) smem_warp[BLOCK / 32] = w;
  }
  __syncthreads();
  int warp_excl = warp ? smem_warp[warp - 1] : 0;
  *total = smem_warp[BLOCK / 32];
  int r = warp_excl + x - v;
  __syncthreads();
  return r;
}

// bf16 helpers
__device__ __forceinline__ float ldf(const void* p, int dtype, int64_t i) {
  if (dtype == VP_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  if (dtype == VP_F64) return (float)reinterpret_cast<const double*>(p)[i];
  return reinterpret_cast<const float*>(p)[i];
}
__device__ __forceinline__ void stf(void* p, int dtype, int64_t i, float v) {
  if (dtype == VP_BF16)
    reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
  else
    reinterpret_cast<float*>(p)[i] = v;
}

}  // namespace vp
