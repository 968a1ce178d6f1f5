/*
 * voxpipe_b200 — C-ABI of the B200-native sparse-convolution hot path.
 *
 * Drop-in boundary for the reference voxpipe 0.1.0 (arXiv 2012.13846,
 * "SparsePipe"): every entry point below replaces one reference function or
 * loop of its hot path (cited per function).  Conventions:
 *
 *   - plain pointers and sizes only (no torch types); all array pointers are
 *     DEVICE pointers unless the parameter says "host";
 *   - stream-ordered: every call only enqueues work on `stream` (no host
 *     synchronisation), so calls are CUDA-graph capturable;
 *   - data-dependent counts live in device memory (`int32_t* n_*_dev`); a
 *     NULL count pointer means "the count equals the capacity argument";
 *     capacities (`cap_*`, host) size grids and buffers;
 *   - no global mutable state: scratch comes from the caller (`ws`, sized by
 *     the matching *_ws_bytes query), so calls are re-entrant across
 *     streams and threads (one workspace per concurrent call).  Workspaces
 *     must be ZERO-FILLED before their first use: the fused BN statistics
 *     keep a self-re-arming ticket counter in theirs, and every call leaves
 *     it at zero again;
 *   - status codes mirror voxpipe/errors.py:3-5 exit codes:
 *       VP_OK = 0, VP_EVALIDATION = 2 (ValidationError/StructuralError),
 *       VP_EINTERNAL = 3 (InternalError, e.g. a CUDA launch failure).
 *     vp_last_error() returns a per-thread message for the last failure.
 *
 * Coordinates are int32 rows [batch, x, y, z] (16 B, D <= 3 with unused axes
 * zero); hash keys use the reference packing (kernels.py:53-79): 16-bit
 * fields batch<<48 | (x+32768)<<32 | (y+32768)<<16 | (z+32768).
 * Features are bf16 (dtype 1) or fp32 (dtype 0) row-major [rows, channels].
 * Weights are [K, C_out, C_in] (conv.py:77-105 layout).
 */
#ifndef VOXPIPE_B200_H
#define VOXPIPE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* vp_stream_t; /* == cudaStream_t */

enum { VP_OK = 0, VP_EVALIDATION = 2, VP_EINTERNAL = 3 };
/* VP_TF32: fp32 storage with tf32 tensor-core math — accepted as the
 * feature dtype of vp_conv_fwd / vp_conv_dgrad (fp32 accumulation, error
 * <= 2e-3 * sum|W||x|); everywhere else it means VP_F32. */
enum { VP_F32 = 0, VP_BF16 = 1, VP_F64 = 2, VP_TF32 = 3 };
#define VP_MAX_OFFSETS 343 /* 7^3 */

const char* vp_last_error(void);
const char* vp_version(void);
/* diagnostic: number of kernels this thread has enqueued through the library
 * (bench.py's gpu_launches claim; a CUDA graph capture counts each node once) */
long long vp_kernel_launches(void);
/* diagnostics: record a clock64 timeline of CTA 0 of the conv kernels into
 * buf (device, >= 1280 int64; null disables) — see conv_fwd_tc.cuh */
int vp_debug_conv_trace(long long* buf);

/* ---------------------------------------------------------------- hash
 * Replaces _kernels.pyx:24-47 `build_table` and :50-73 `lookup` (the
 * VOXPIPE_BACKEND seam, kernels.py:21-32,82-92).  Open addressing with
 * linear probing on splitmix64 (_kernels.pyx:16-21); capacity = pow2 >=
 * 2n+2 (min 8) (_kernels.pyx:27-29); FIRST occurrence of a duplicated key
 * wins (_kernels.pyx:44-46); lookup returns the row or -1.  `table` holds
 * (cap + 1) 16-byte slots (vp_hash_bytes). */
int64_t vp_hash_capacity(int64_t n);
size_t vp_hash_bytes(int64_t cap);
int vp_hash_build(const int64_t* keys, const int32_t* n_dev, int64_t cap_n,
                  void* table, int64_t table_cap, vp_stream_t stream);
int vp_hash_lookup(const void* table, int64_t table_cap, const int64_t* queries,
                   int64_t m, int64_t* rows_out, vp_stream_t stream);

/* pack_rows (kernels.py:53-79) for int32 [n,4] rows; bad_dev (nullable)
 * receives 1 if any row is out of the packable range (ValidationError). */
int vp_pack_coords(const int32_t* coords, int64_t n, int64_t* keys, int32_t* bad_dev,
                   vp_stream_t stream);

/* ---------------------------------------------------------------- coords
 * SparseTensor invariants (tensor.py:49-78): flags_dev[0] |= 1 duplicate
 * row, |= 2 negative batch, |= 4 axis not a multiple of the stride, |= 8
 * unpackable coordinate.  Replaces the np.unique dedupe (tensor.py:28-33). */
size_t vp_validate_coords_ws_bytes(int64_t cap_n);
int vp_validate_coords(const int32_t* coords, const int32_t* n_dev, int64_t cap_n,
                       const int32_t* tensor_stride_host3, int32_t* flags_dev,
                       void* ws, size_t ws_bytes, vp_stream_t stream);
/* finite check of features (tensor.py:71-72): flags_dev[0] |= 16 if any
 * non-finite value. */
int vp_check_finite(const void* feats, int32_t dtype, int64_t count, int32_t* flags_dev,
                    vp_stream_t stream);

/* generate_output_coords (conv.py:124-146) for stride > 1: floor-div by
 * the NEW tensor stride `step` (= tensor_stride * stride), rescale, unique
 * rows in FIRST-SEEN order.  out needs cap_in rows; *n_out_dev receives
 * N_out, or -1 when a downsampled row leaves the packed 16-bit axis range
 * (e.g. -32768 floored to a multiple of 3): such rows cannot be keyed, so
 * the caller uses vp_wide_output_coords instead.  parent (nullable, int32
 * [cap_in]) receives the output row of each input row (pooling glue). */
size_t vp_output_coords_ws_bytes(int64_t cap_in);
int vp_output_coords(const int32_t* in, const int32_t* n_in_dev, int64_t cap_in,
                     const int32_t* step_host3, int32_t* out, int32_t* n_out_dev,
                     int32_t* parent, void* ws, size_t ws_bytes, vp_stream_t stream);

/* voxelize (tensor.py:147-184) + batch (tensor.py:205-229) fused: points
 * [n,3] (f32 or f64) of B clouds delimited by cloud_offsets_dev[B+1]
 * (int64); voxel = clip(floor(p / voxel_size), 0, res-1) in f64; batch index
 * = cloud position; rows in first-seen order per cloud, clouds
 * concatenated.  coords_out needs n rows; point2voxel (nullable) receives
 * each point's output row; feats_out (nullable, dtype feat_dtype, [n,1])
 * receives the occupancy feature 1.0. */
size_t vp_voxelize_ws_bytes(int64_t n_points);
int vp_voxelize(const void* points, int32_t pts_dtype, int64_t n_points,
                const int64_t* cloud_offsets_dev, int32_t n_clouds, double voxel_size,
                const int32_t* res_host3, int32_t* coords_out, int32_t* n_out_dev,
                int32_t* point2voxel, void* feats_out, int32_t feat_dtype,
                void* ws, size_t ws_bytes, vp_stream_t stream);
/* mean-merged features (tensor.py:178-183, np.add.at order = point order,
 * deterministic): feats_in [n, F] f32/f64 -> feats_out [n_vox, F] f32. */
size_t vp_voxel_mean_ws_bytes(int64_t n_points, int64_t cap_vox);
int vp_voxel_mean(const void* feats_in, int32_t in_dtype, int64_t n_points, int32_t F,
                  const int32_t* point2voxel, const int32_t* n_vox_dev, int64_t cap_vox,
                  float* feats_out, void* ws, size_t ws_bytes, vp_stream_t stream);

/* ---------------------------------------------------------------- kernel map
 * build_kernel_map (conv.py:149-183): one hash over the input rows, then
 * for every output row u and offset k (shape order) probe
 * out[u] + off_k * in_stride (batch untouched, conv.py:173-174);
 * out-of-packable-range queries are misses (kernels.py:131-148).
 *   nbr      [cap_out, K] int32 : input row or -1 (dense neighbour table)
 *   pair_in / pair_out [cap_out*K] (nullable): per-offset pair lists in
 *            CSR order — offset-major, out rows ASCENDING within an offset
 *            (bit-exact with KernelMap.pairs);
 *   pair_ptr [K+1] int32 device (nullable iff pair_in is NULL). */
size_t vp_kernel_map_ws_bytes(int64_t cap_in, int64_t cap_out, int32_t K);
int vp_kernel_map(const int32_t* in, const int32_t* n_in_dev, int64_t cap_in,
                  const int32_t* out, const int32_t* n_out_dev, int64_t cap_out,
                  const int32_t* offsets_host, int32_t K, const int32_t* in_stride_host3,
                  int32_t* nbr, int32_t* pair_in, int32_t* pair_out, int32_t* pair_ptr,
                  void* ws, size_t ws_bytes, vp_stream_t stream);
/* Dense-grid index for bounded lattices (batch < B, every axis a multiple
 * of s in [0, R*s)): `cells` is vp_grid_words(B, R) int32 words — the cell
 * table [B*R^3] (cell -> row) followed by an occupancy bitmap
 * [ceil(B*R^3/32)] — initialised once with vp_grid_init (zeroes the bitmap;
 * cell values are meaningful only where their bit is set).  vp_grid_set
 * writes each row's cell and bit (clear=0) or zeroes exactly the bitmap
 * words of those rows (clear=1), so the grid is reusable.  The probe reads
 * the bitmap for every neighbour and the cell only for hits.
 * vp_kernel_map_grid is build_kernel_map with the grid as the index: the
 * same nbr / pair outputs, bit-exact with the hash path on such lattices. */
int64_t vp_grid_words(int32_t B, int32_t R);
int vp_grid_init(int32_t* cells, int32_t B, int32_t R, vp_stream_t stream);
int vp_grid_set(const int32_t* coords, const int32_t* n_dev, int64_t cap, int32_t* cells, int32_t B,
                int32_t R, int32_t s, int32_t clear, vp_stream_t stream);
size_t vp_kernel_map_grid_ws_bytes(int64_t cap_out, int32_t K);
/* Lattice kernel map for the operator API (build_kernel_map on rows that
 * sit on one bounded lattice of spacing s; conv.py:149-183):
 * vp_coords_bbox writes bbox[9] (device int32) = the minimum over both row
 * sets of (b, x, y, z, -b, -x, -y, -z) and 1 if every row is on the spacing
 * lattice else 0; the caller reads it back, picks lattice_host =
 * {B, R, ox, oy, oz} (origin a multiple of s, R^3 cells per batch) and calls
 * vp_kernel_map_lattice: grid set + probe + scan + emit + clear on `grid`
 * (vp_grid_words(B, R) int32 words, bitmap zero on entry and on return).
 * Outputs and ws (vp_kernel_map_grid_ws_bytes) as vp_kernel_map_grid;
 * results identical to vp_kernel_map. */
int vp_coords_bbox(const int32_t* a, int64_t n_a, const int32_t* b, int64_t n_b, int32_t s, int32_t* bbox,
                   vp_stream_t stream);
int vp_kernel_map_lattice(const int32_t* in, int64_t n_in, const int32_t* out, int64_t n_out,
                          const int32_t* offsets_host, int32_t K, int32_t s, const int32_t* lattice_host,
                          int32_t* grid, int64_t grid_words, int32_t* nbr, int32_t* pair_in, int32_t* pair_out,
                          int32_t* pair_ptr, void* ws, size_t ws_bytes, vp_stream_t stream);
int vp_kernel_map_grid(const int32_t* cells, int32_t B, int32_t R, int32_t s, const int32_t* out,
                       const int32_t* n_out_dev, int64_t cap_out, const int32_t* offsets_host, int32_t K,
                       const int32_t* in_stride_host3, int32_t* nbr, int32_t* pair_in, int32_t* pair_out,
                       int32_t* pair_ptr, void* ws, size_t ws_bytes, vp_stream_t stream);
/* Neighbour-pattern row grouping (kmap_sort.cu): stable counting sort of
 * the live table rows by a 9-bit key of their 3^3 hit mask — key_mode 0:
 * which (dx, dy) columns hold a hit (stride-1 tables), 1: which dx / dy /
 * dz planes hold a hit (strided inverse tables), 2: the whole 27-bit mask
 * (three stable 9-bit passes; ~1M-row levels) — into perm [n] (table row
 * order -> row id) and table_sorted [n, K] = table[perm].  Passing
 * (table_sorted, perm) to vp_conv_fwd / vp_conv_dgrad gives results
 * identical to (table, NULL) with far fewer active offsets per 128-row tile.
 * vp_kernel_map_sort = key mode 1.  No library sort; deterministic. */
size_t vp_kernel_map_sort_ws_bytes(int64_t cap, int32_t K);
int vp_kernel_map_sort(const int32_t* table, const int32_t* n_dev, int64_t cap, int32_t K, int32_t* perm,
                       int32_t* table_sorted, void* ws, size_t ws_bytes, vp_stream_t stream);
int vp_kernel_map_group(const int32_t* table, const int32_t* n_dev, int64_t cap, int32_t K, int32_t key_mode,
                        int32_t* perm, int32_t* table_sorted, void* ws, size_t ws_bytes, vp_stream_t stream);
/* vp_kernel_map_group with a tile schedule for a conv launched with
 * sched_grid CTAs (vp_conv_tc_grid; 0 = plain vp_kernel_map_group): rows are
 * grouped in DESCENDING key order (the partial last tile gets the sparsest
 * rows), then whole 128-row tiles are placed so that the conv's round-robin
 * tile -> CTA assignment approximates longest-processing-time-first (tile
 * cost = its active offsets; the ragged last tile stays last).  The moves
 * apply when sched_grid < tiles <= 4 sched_grid and K <= 32; every row keeps
 * its tile mates, so per-row conv results are bitwise those of the
 * descending grouping without moves (e.g. sched_grid = 1). */
int vp_kernel_map_group_sched(const int32_t* table, const int32_t* n_dev, int64_t cap, int32_t K, int32_t key_mode,
                              int32_t sched_grid, int32_t* perm, int32_t* table_sorted, void* ws, size_t ws_bytes,
                              vp_stream_t stream);
/* CTA count of the default tensor-core conv config writing nd-wide rows into
 * cap_out rows (0 when nd takes no tensor-core path). */
int32_t vp_conv_tc_grid(int64_t nd, int64_t cap_out);
/* Two-level ("brick") index for bounded lattices, the same contract as the
 * dense grid with ~64x less memory: a coarse table over 4^3 bricks plus a
 * pool of 256 B bricks allocated only where rows exist (kmap_brick.cu).
 * `index` (vp_brick_bytes(cap, B, R) bytes) is initialised once with
 * vp_brick_init; vp_brick_set(clear=0) indexes the rows, vp_brick_set(clear=1)
 * empties exactly what was set so the index is reusable.  cap <= the cap the
 * index was sized for.  vp_kernel_map_brick == vp_kernel_map_grid on it. */
int64_t vp_brick_pool(int64_t cap, int32_t B, int32_t R);
size_t vp_brick_bytes(int64_t cap, int32_t B, int32_t R);
int vp_brick_init(void* index, int64_t cap, int32_t B, int32_t R, vp_stream_t stream);
int vp_brick_set(const int32_t* coords, const int32_t* n_dev, int64_t cap, void* index, int64_t index_cap,
                 int32_t B, int32_t R, int32_t s, int32_t clear, vp_stream_t stream);
size_t vp_kernel_map_brick_ws_bytes(int64_t cap_out, int32_t K);
int vp_kernel_map_brick(const void* index, int64_t index_cap, int32_t B, int32_t R, int32_t s, const int32_t* out,
                        const int32_t* n_out_dev, int64_t cap_out, const int32_t* offsets_host, int32_t K,
                        const int32_t* in_stride_host3, int32_t* nbr, int32_t* pair_in, int32_t* pair_out,
                        int32_t* pair_ptr, void* ws, size_t ws_bytes, vp_stream_t stream);
/* inverse neighbour table inv[v, k] = u for every pair (v,u) of offset k
 * (the dgrad gather table; conv.py:238-240 iterates the same pairs). */
int vp_kernel_map_inverse(const int32_t* nbr, const int32_t* n_out_dev, int64_t cap_out,
                          int32_t K, int32_t* inv, int64_t cap_in, vp_stream_t stream);

/* ---------------------------------------------------------------- sparse conv
 * Forward (conv.py:186-208, Eq. 3): y[u] = sum_k W_k x[nbr[u,k]], summed per
 * output row in offset order; output-stationary implicit GEMM on tcgen05
 * (bf16 in, fp32 TMEM accumulate) when x is bf16 and C_in, C_out are
 * multiples of 8 up to 256 (tiles of 32/64/128/256, the padding zero-filled
 * on load and never stored); tf32 math on the same tiles when x_dtype is
 * VP_TF32 (C_in <= 128); a SIMT kernel otherwise (exact fp32 / f64).
 * Deterministic, no atomics.
 *   table  : nbr [cap_out, K] (or inv for dgrad); flip != 0 reads column
 *            K-1-k (stride-1 symmetric kernels: inv[v,k] == nbr[v,K-1-k]).
 *   perm   : nullable; table row i holds the neighbours of output row
 *            perm[i] (vp_kernel_map_sort), which is where its result goes.
 *   w      : [K, c_out, c_in] in w_dtype.
 *   x_rows : rows allocated in x (every table entry is < x_rows); checked
 *            by the shim only.  The tensor-core path gathers rows with
 *            16-byte cp.async (8 lanes per 128 B row) and zero-fills a
 *            missing neighbour (table entry -1) with a 0-byte source; the
 *            per-tile [128, K] table slab is staged with one bulk copy
 *            (cp.async.bulk, SASS UBLKCP), not TMA tensor maps. */
int vp_conv_fwd(const void* x, int32_t x_dtype, int64_t x_rows, int64_t c_in, const void* w, int32_t w_dtype,
                int64_t c_out, int32_t K, const int32_t* table, int32_t flip, const int32_t* perm,
                const int32_t* n_out_dev, int64_t cap_out, void* y, int32_t y_dtype,
                void* ws, size_t ws_bytes, vp_stream_t stream);
size_t vp_conv_fwd_ws_bytes(int64_t c_in, int64_t c_out, int32_t K);
/* dgrad (conv.py:240): grad_in[v] = sum_k W_k^T g[inv[v,k]]; same kernel as
 * the forward with W transposed into ws.  table = inv (or nbr with flip). */
size_t vp_conv_dgrad_ws_bytes(int64_t c_in, int64_t c_out, int32_t K);
int vp_conv_dgrad(const void* g, int32_t g_dtype, int64_t g_rows, int64_t c_out, const void* w, int32_t w_dtype,
                  int64_t c_in, int32_t K, const int32_t* table, int32_t flip, const int32_t* perm,
                  const int32_t* n_in_dev, int64_t cap_in, void* grad_in, int32_t gi_dtype,
                  void* ws, size_t ws_bytes, vp_stream_t stream);
/* wgrad (conv.py:241): grad_w[k] = sum_{(v,u) in pairs_k} g[u] x[v]^T into
 * fp32 [K, c_out, c_in]; deterministic fixed-order chunked reduction. */
size_t vp_conv_wgrad_ws_bytes(int64_t c_in, int64_t c_out, int32_t K, int64_t cap_pairs);
int vp_conv_wgrad(const void* x, int32_t x_dtype, int64_t c_in, const void* g, int32_t g_dtype,
                  int64_t c_out, int32_t K, const int32_t* pair_in, const int32_t* pair_out,
                  const int32_t* pair_ptr, int64_t cap_pairs, void* grad_w,
                  void* ws, size_t ws_bytes, vp_stream_t stream);
/* vp_conv_wgrad for a weight gradient that runs on a side stream beside a
 * critical path (the data-parallel training step): the persistent grid is
 * capped like vp_conv_wgrad_sgd's (VP_WGRAD_SMS, 96 of 148 SMs, for pair
 * capacities <= 4M); results identical to vp_conv_wgrad. */
int vp_conv_wgrad_side(const void* x, int32_t x_dtype, int64_t c_in, const void* g, int32_t g_dtype,
                       int64_t c_out, int32_t K, const int32_t* pair_in, const int32_t* pair_out,
                       const int32_t* pair_ptr, int64_t cap_pairs, void* grad_w, void* ws, size_t ws_bytes,
                       vp_stream_t stream);

/* vp_conv_wgrad + momentum SGD of W in the reduction kernel (the training
 * step's per-layer update without a separate pass): m = momentum*m + grad_w,
 * p -= lr*m, p_bf16 (nullable) = bf16(p); grad_w is still written.
 * phase 0: everything; 1: the chunk partials only (no parameter access);
 * 2: the reduction + SGD over the partials phase 1 left in ws — so the
 * caller can start the partials early and order phase 2 after every reader
 * of p / p_bf16 (the layer's dgrad). */
int vp_conv_wgrad_sgd(const void* x, int32_t x_dtype, int64_t c_in, const void* g, int32_t g_dtype,
                      int64_t c_out, int32_t K, const int32_t* pair_in, const int32_t* pair_out,
                      const int32_t* pair_ptr, int64_t cap_pairs, void* grad_w, void* ws, size_t ws_bytes,
                      float* p, float* m, void* p_bf16, float lr, float momentum, int32_t phase,
                      vp_stream_t stream);

/* ---------------------------------------------------------------- glue
 * Model glue for the SparseResNet training step (no reference
 * implementation: SPEC.md:185 non-goal — parity self-defined). */
/* per-channel batch statistics over rows: mean/rstd [C] fp32.  One launch:
 * the last block to finish reduces every block's partials in block order.
 * ws (vp_bn_stats_ws_bytes) ends in a ticket word that must be ZERO before
 * the first call with that workspace; every call leaves it zero again (so a
 * zero-filled workspace can be reused, also under CUDA-graph replay).  The
 * same holds for vp_bn_backward's workspace. */
size_t vp_bn_stats_ws_bytes(int64_t cap_n, int64_t C);
int vp_bn_stats(const void* x, int32_t x_dtype, const int32_t* n_dev, int64_t cap_n, int64_t C,
                float eps, float* mean, float* rstd, void* ws, size_t ws_bytes, vp_stream_t stream);
/* vp_bn_stats + vp_bn_apply in ONE cooperative launch: the blocks reduce
 * their partial sums, the last one writes mean/rstd, and every block then
 * normalises its rows when VP_BN_FUSED=1; by default (faster inside the
 * concurrent training step) it issues the two launches.
 * ws: vp_bn_stats_ws_bytes, zero-filled before first use. */
int vp_bn_forward(const void* x, int32_t x_dtype, const int32_t* n_dev, int64_t cap_n, int64_t C, float eps,
                  float* mean, float* rstd, const float* gamma, const float* beta, const void* res,
                  int32_t res_dtype, int32_t relu, void* y, int32_t y_dtype, void* ws, size_t ws_bytes,
                  vp_stream_t stream);
/* y = act((x - mean) * rstd * gamma + beta [+ res]) ; act = relu if relu */
int vp_bn_apply(const void* x, int32_t x_dtype, const int32_t* n_dev, int64_t cap_n, int64_t C,
                const float* mean, const float* rstd, const float* gamma, const float* beta,
                const void* res, int32_t res_dtype, int32_t relu, void* y, int32_t y_dtype,
                vp_stream_t stream);
/* backward of bn_apply: the incoming gradient is gy (+ gy2 when non-null,
 * same dtype: the residual-branch sum), masked by (y > 0) when relu; writes
 * grad_x (and grad_res = masked gradient when non-null), ggamma/gbeta [C]. */
size_t vp_bn_backward_ws_bytes(int64_t cap_n, int64_t C);
int vp_bn_backward(const void* gy, const void* gy2, int32_t gy_dtype, const void* y, int32_t y_dtype,
                   const void* x, int32_t x_dtype, const int32_t* n_dev, int64_t cap_n, int64_t C,
                   const float* mean, const float* rstd, const float* gamma, int32_t relu,
                   void* grad_x, int32_t gx_dtype, void* grad_res, float* ggamma, float* gbeta,
                   void* ws, size_t ws_bytes, vp_stream_t stream);
/* ---- BN statistics fused into the producing conv (no reference code:
 * SPEC.md:184-185 non-goal).  The conv forward (or the dgrad of the NEXT
 * conv) writes per-CTA fp32 partial sums of the BN statistics from its
 * epilogue, so the critical path runs conv -> apply instead of conv ->
 * statistics pass -> apply.
 *   bn_part : vp_bn_part_bytes(C) bytes, device; int header (rows written,
 *             set on the device by the producer) + [rows][2][C] fp32.
 *   bn_mode : 0 off (plain vp_conv_fwd / vp_conv_dgrad);
 *             1 forward: partials (sum y, sum y^2) of the stored output;
 *             2 backward: the output becomes g = round(y) [+ bn_add],
 *               zeroed where bn_act <= 0 (ReLU mask; bn_act nullable),
 *               stored rounded; partials (sum g, sum g*(bn_pre - bn_mean)).
 *   bn_add/bn_act/bn_pre: same dtype and shape as the conv output.
 *   bn_out_a/bn_out_b (nullable together): also finalize the statistics in
 *             the producer chain — mode 1: mean / rstd (biased variance,
 *             bn_eps); mode 2: ggamma = bn_rstd * sum g*(pre-mean), gbeta =
 *             sum g — so the BN apply follows the conv directly.
 * bn_part must be ZERO-FILLED before its first use (a self-re-arming ticket
 * lives in the header).  A bf16 tensor-core conv fuses the statistics into
 * its epilogue and the finalize into its split-K reduction kernel; every
 * other path runs one extra pass over the output. */
size_t vp_bn_part_bytes(int64_t C);
int vp_conv_fwd_bn(const void* x, int32_t x_dtype, int64_t x_rows, int64_t c_in, const void* w, int32_t w_dtype,
                   int64_t c_out, int32_t K, const int32_t* table, int32_t flip, const int32_t* perm,
                   const int32_t* n_out_dev, int64_t cap_out, void* y, int32_t y_dtype, void* ws, size_t ws_bytes,
                   int32_t bn_mode, void* bn_part, const void* bn_add, const void* bn_act, const void* bn_pre,
                   const float* bn_mean, float bn_eps, float* bn_out_a, float* bn_out_b, const float* bn_rstd,
                   vp_stream_t stream);
int vp_conv_dgrad_bn(const void* g, int32_t g_dtype, int64_t g_rows, int64_t c_out, const void* w, int32_t w_dtype,
                     int64_t c_in, int32_t K, const int32_t* table, int32_t flip, const int32_t* perm,
                     const int32_t* n_in_dev, int64_t cap_in, void* grad_in, int32_t gi_dtype, void* ws,
                     size_t ws_bytes, int32_t bn_mode, void* bn_part, const void* bn_add, const void* bn_act,
                     const void* bn_pre, const float* bn_mean, float bn_eps, float* bn_out_a, float* bn_out_b,
                     const float* bn_rstd, vp_stream_t stream);
/* BN backward apply from finished (ggamma, gbeta) and the stored masked
 * gradient gm: grad_x = gamma*rstd*(gm - gbeta/n - xhat*ggamma/n). */
int vp_bn_backward_apply(const void* gm, int32_t gm_dtype, const void* x, int32_t x_dtype, const int32_t* n_dev,
                         int64_t cap_n, int64_t C, const float* mean, const float* rstd, const float* gamma,
                         const float* ggamma, const float* gbeta, void* grad_x, int32_t gx_dtype, vp_stream_t stream);
/* vp_bn_apply with the statistics reduced from a mode-1 bn_part (fixed
 * order); also stores mean/rstd for the backward. */
int vp_bn_apply_part(const void* x, int32_t x_dtype, const int32_t* n_dev, int64_t cap_n, int64_t C, float eps,
                     const void* bn_part, float* mean, float* rstd, const float* gamma, const float* beta,
                     const void* res, int32_t res_dtype, int32_t relu, void* y, int32_t y_dtype, vp_stream_t stream);
/* BN backward from a mode-2 bn_part: gm is the masked gradient the producer
 * stored; writes grad_x and ggamma/gbeta [C]. */
int vp_bn_backward_part(const void* gm, int32_t gm_dtype, const void* x, int32_t x_dtype, const int32_t* n_dev,
                        int64_t cap_n, int64_t C, const float* mean, const float* rstd, const float* gamma,
                        const void* bn_part, void* grad_x, int32_t gx_dtype, float* ggamma, float* gbeta,
                        vp_stream_t stream);
/* per-batch-index row segments of batch-contiguous rows: seg[0:B] =
 * counts, seg[B:2B] = starts (int32, device) */
int vp_batch_segments(const int32_t* coords, const int32_t* n_dev, int64_t cap_n, int32_t B, int32_t* seg,
                      vp_stream_t stream);
/* The classifier head of the training step, fused (two launches): per-cloud
 * mean pool of a [n, C], logits = pooled W^T + bias, softmax cross entropy
 * (mean over B) and its gradients (g_w, g_b fp32), and the gradient of every
 * row of a (pool backward) — masked by bn_act > 0 and stored in gm (a's
 * dtype); with bn_pre (the last BN's input) also that BN's backward
 * statistics, finalized to ggamma / gbeta (bn_rstd) so its backward apply
 * (vp_bn_backward_apply) follows directly.  bn_part: vp_bn_part_bytes(C),
 * zero-filled before first use.  Same arithmetic and summation order as
 * vp_global_pool + vp_linear_xent + vp_global_pool_backward. */
size_t vp_sparse_head_ws_bytes(int32_t B, int64_t C, int32_t classes);
int vp_sparse_head(const void* a, int32_t a_dtype, const int32_t* seg, int32_t B, int64_t C, const float* w,
                   const float* bias, int32_t classes, const int32_t* labels, float* pooled, float* logits, float* loss,
                   float* g_w, float* g_b, const void* bn_act, const void* bn_pre, const float* bn_mean,
                   const float* bn_rstd, void* gm, void* bn_part, float* ggamma, float* gbeta, void* ws,
                   size_t ws_bytes, vp_stream_t stream);
/* global average pool per batch index (rows batch-contiguous):
 * out [B, C] fp32, counts [B] int32 */
int vp_global_pool(const void* x, int32_t x_dtype, const int32_t* coords, const int32_t* n_dev,
                   int64_t cap_n, int64_t C, int32_t B, float* out, int32_t* counts,
                   void* ws, size_t ws_bytes, vp_stream_t stream);
size_t vp_global_pool_ws_bytes(int32_t B);
int vp_global_pool_backward(const float* gout, const int32_t* coords, const int32_t* counts,
                            const int32_t* n_dev, int64_t cap_n, int64_t C, void* gx,
                            int32_t gx_dtype, vp_stream_t stream);
/* linear + softmax cross entropy (mean over B); writes loss [1] fp32,
 * logits [B, classes], grad wrt pooled [B, C] and fc grads (fixed-order
 * reductions over the batch).  ws: vp_linear_xent_ws_bytes. */
size_t vp_linear_xent_ws_bytes(int32_t B, int32_t classes);
int vp_linear_xent(const float* pooled, int32_t B, int32_t C, const float* fc_w, const float* fc_b,
                   int32_t classes, const int32_t* labels, float* logits, float* loss,
                   float* g_pooled, float* g_fc_w, float* g_fc_b, void* ws, size_t ws_bytes,
                   vp_stream_t stream);
/* SGD with momentum over a flat fp32 parameter buffer (p, m, g of n):
 * m = momentum*m + g; p -= lr*m; and refresh the bf16 shadow copy of the
 * first n_bf16 entries (p_bf16 nullable). */
int vp_sgd_momentum(float* p, float* m, const float* g, int64_t n, float lr, float momentum,
                    void* p_bf16, int64_t n_bf16, vp_stream_t stream);
/* dtype conversion f32 <-> bf16 */
int vp_cast(const void* src, int32_t src_dtype, void* dst, int32_t dst_dtype, int64_t count,
            vp_stream_t stream);

/* ---------------------------------------------------------------- wide rows
 * Coordinates the packed 64-bit key cannot hold (kernels.py:40-78: more than
 * 3 axes, or axes beyond the 16-bit fields) — the reference's TupleCoordIndex
 * fallback (kernels.py:95-122).  Rows are int64 [n, D1] = [batch, x1..xD]
 * (2 <= D1 <= 8); the index is an open-addressing table of row numbers whose
 * probe compares whole tuples (first occurrence wins).  Host arrays:
 * tensor_stride / step / in_stride int64 [D1-1], offsets int32 [K, D1-1]. */
size_t vp_wide_ws_bytes(int64_t n_in, int64_t n_out, int32_t D1, int32_t K);
/* tensor.py:49-78 on wide rows: flags |= 1 duplicate, 2 negative batch,
 * 4 axis not a multiple of the tensor stride. */
int vp_wide_validate(const int64_t* rows, int64_t n, int32_t D1, const int64_t* tensor_stride,
                     int32_t* flags_dev, void* ws, size_t ws_bytes, vp_stream_t stream);
/* conv.py:124-146: out rows = unique(floor(in / step) * step) in first-seen
 * order; *n_out_dev = count.  out holds n rows. */
int vp_wide_output_coords(const int64_t* in, int64_t n, int32_t D1, const int64_t* step, int64_t* out,
                          int32_t* n_out_dev, void* ws, size_t ws_bytes, vp_stream_t stream);
/* conv.py:149-183 on wide rows: nbr [n_out, K] + CSR pairs in the reference
 * order (offset-major, ascending out row). */
int vp_wide_kernel_map(const int64_t* in, int64_t n_in, const int64_t* out, int64_t n_out, int32_t D1,
                       const int32_t* offsets, int32_t K, const int64_t* in_stride, int32_t* nbr,
                       int32_t* pair_in, int32_t* pair_out, int32_t* pair_ptr, void* ws, size_t ws_bytes,
                       vp_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* VOXPIPE_B200_H */
