// Warp-specialized output-stationary implicit GEMM for the sparse conv
// forward (conv.py:186-208) and dgrad (conv.py:240) on sm_100a tcgen05.
//
//   out[r, n] = sum_{k active} sum_{c} A_k[r, c] * B_k[n, c]
//   forward: A_k[r] = x[table[r, k]] (C_in wide), B_k = W_k        (K-major)
//   dgrad  : A_k[r] = g[table[r, k]] (C_out wide), B_k = W_k^T     (W read
//            directly as an MN-major operand: no transposed copy)
//
// CTA = 9 warps: warps 0-3 produce (cp.async gathers of 128 neighbour rows +
// the weight slice into a 128B-swizzled stage ring, completion signalled per
// stage on an mbarrier; 8 lanes per row so one warp instruction moves 4 whole
// 128 B lines), warp 8 issues tcgen05.mma from
// one elected lane into a double-buffered TMEM accumulator, warps 4-7 drain
// TMEM (tcgen05.ld) and store each output row exactly once.  Work items are
// (128-row tile, split) pairs; when the tile count cannot fill the grid the
// active offsets of a tile are split across CTAs (fp32 partials, reduced in a
// fixed order afterwards) -> deterministic with no atomics on the output.
// Each item's offset-activity scan (which offsets any of its rows hits) runs
// in the epilogue warps one item ahead, so the producers only publish at a
// tile boundary.
// C_in = 32 packs two offsets into one 64-wide K stage.  CPS CTAs share an SM
// (smem ring and TMEM sized to fit): random-row gather throughput scales with
// independent CTAs per SM far more than with ring depth (tools/gather_probe2).
#pragma once
#include "bn_epi.cuh"
#include "common.cuh"
#include "tc.cuh"

namespace vp {

using bf16 = __nv_bfloat16;

struct FwdParams {
  const bf16* x;
  const bf16* w;
  int K;
  const int32_t* table;
  int flip;
  const int32_t* perm;  // table row i holds output row perm[i] (null = identity; kmap_sort.cu)
  const int32_t* n_out_dev;
  int64_t cap_out;
  void* y;
  int y_dtype;
  float* part;    // split-K partials (grid * 128 * ND floats), may be null if max_split == 1
  int max_split;  // >= 1
  int stage_tbl;  // stage table tiles in smem (K <= kTblK, 16 B-aligned table); set by the launcher
  int dbg;        // experiments only: bit0 no MMA, bit1 no B copies, bit2 no A copies, bit3 plain arrive for empty, bit4 every offset active (no mask scan)
  BnEpi epi;      // BN statistics of the output (bn_epi.cuh); mode 0 = off.  Needs a bf16 output.
  long long* trace;  // debug timeline of CTA 0 (null = off)
  // real widths in 2-byte units (the kernel's KD / ND are the padded tile
  // widths): gathered row length (C_in, or 2 C_in for tf32) and output
  // columns.  Chunks past kreal load zeros, columns past nreal are not stored.
  int kreal;
  int nreal;
};

constexpr int kTcProd = 128, kTcEpi = 128, kTcThreads = kTcProd + kTcEpi + 32;
constexpr int kNbrSmemK = 32;  // (wgrad) neighbour table cached in smem when K <= 32
constexpr int kTcMaskWords = (VP_MAX_OFFSETS + 31) / 32;
constexpr int kTblK = 32;  // K <= kTblK: each tile's [128, K] table is staged in smem by TMA

// Debug timeline of CTA 0 (clock64), off unless vp_debug_conv_trace() set a
// buffer: stage events [g][4] at slot g < 256 (producer slot acquired,
// producer issued, MMA saw full, MMA committed), tile events at 1024 + 4*ii
// (prologue start, work published, epilogue got accumulator, epilogue done).
// (the buffer travels in FwdParams::trace; vp_debug_conv_trace sets it)
extern long long* g_conv_trace_host;
#define trace_ev(idx, on)                           \
  do {                                              \
    if (trc != nullptr && (on)) trc[idx] = clock64(); \
  } while (0)

constexpr int tmem_cols_pow2(int c) {
  return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : c <= 512 ? 512 : 1024;  // 1024: does not fit
}

// A stage holds RB "atoms": one unit each (a 128-row x 64-element bf16 A
// slab, 128 B swizzled rows, plus the matching [ND x 64] weight slab).  Big
// stages amortise the per-stage cost (barrier round trip, row lookups) that
// bounds small-row gathers (tools/gather_probe2: ~2x per 16 KB at RB=2).
// TT = 128-row tiles per work item sharing each weight (B) stage: the B
// slab is fetched once and feeds TT MMAs into TT TMEM accumulators, so at
// large N (no split-K needed) the L2->SMEM traffic of the weights, 1/2 to
// 2/3 of all staged bytes at C >= 128, is divided by TT.
// MODE: 0 = bf16 at exact tile widths (compile-time strides, the hot path);
// 1 = bf16 padded to the tile widths (runtime kreal / nreal); 2 = tf32
// (fp32 storage, padded like 1)
template <int KD, int ND, bool BMN, int CPS, int RB, int TT = 1, int MODE = 0>
struct FwdTC {
  static constexpr bool TF32 = MODE == 2;
  static constexpr bool PAIR = (KD == 32);
  static constexpr int NCH = PAIR ? 1 : KD / 64;
  static constexpr int A_BYTES = 128 * 128;
  static constexpr int NPAD = (BMN && ND < 64) ? 64 : ND;
  static constexpr int B_BYTES = NPAD * 128;
  static constexpr int STAGE = RB * (TT * A_BYTES + B_BYTES);
  static constexpr int BOOK = 4096;
  // two [128, K <= kTblK] neighbour-table tiles (double buffer)
  static constexpr int TBL_RESERVE = 2 * TT * 128 * kTblK * 4;
  // 228 KB of shared memory per SM, 1 KB reserved per CTA, 1 KB alignment slack
  static constexpr int BUDGET = (228 * 1024) / CPS - 2048 - BOOK - TBL_RESERVE;
  static constexpr int STAGES_RAW = BUDGET / STAGE;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : (STAGES_RAW < 2 ? 2 : STAGES_RAW);
  static constexpr bool FITS = STAGES_RAW >= 2 && tmem_cols_pow2(TT * ND) * CPS <= 512;
  static constexpr int ACC = (tmem_cols_pow2(2 * TT * ND) * CPS <= 512) ? 2 : 1;
  static constexpr int COLS = ACC * TT * ND;
  static constexpr int TMEM_COLS = tmem_cols_pow2(COLS);
  static constexpr uint32_t IDESC = TF32 ? tc::idesc_tf32(128, ND, 0, BMN ? 1 : 0) : tc::idesc_bf16(128, ND, 0, BMN ? 1 : 0);
  static constexpr int SMEM_BASE = STAGES * STAGE + 1024 + BOOK;
  static constexpr int SMEM_MAX = SMEM_BASE + 2 * TT * 128 * kTblK * 4;
  static int smem_bytes(int K, bool tbl) { return SMEM_BASE + (tbl ? 2 * TT * 128 * K * 4 : 0); }
};

// split-K work items the partial buffer holds (two per SM: the grid of the
// 2-CTA/SM configurations)
constexpr int kSplitItems = 2 * kNumSMs;

__device__ __forceinline__ int split_count(int ntiles, int grid, int max_split) {
  if (ntiles <= 0 || max_split <= 1 || ntiles * 2 > grid) return 1;
  int s = grid / ntiles;
  return s > max_split ? max_split : s;
}

// PW producer warps (4, or 8 for the small-row tiles: the gathers are bound
// by cp.async issue per warp); then 4 epilogue warps and the MMA warp
template <int PW>
constexpr int tc_threads() { return 32 * PW + kTcEpi + 32; }

template <int KD, int ND, bool BMN, int CPS, int RB, bool TBL, int TT = 1, int MODE = 0, int PW = 4>
__global__ void __launch_bounds__(tc_threads<PW>(), CPS) conv_tc_kernel(const __grid_constant__ FwdParams p) {
  constexpr int PROD = 32 * PW, RPT = 32 / PW;  // producer threads; rows per thread per 128-row tile
  ::vp::pdl_begin();
  using C = FwdTC<KD, ND, BMN, CPS, RB, TT, MODE>;
  constexpr bool TF32 = C::TF32;
  static_assert(!(TF32 && BMN), "tf32: dgrad reads a K-major transposed weight copy");
  const int kreal = MODE == 0 ? KD : p.kreal, nreal = MODE == 0 ? ND : p.nreal;
  constexpr int TR = 128 * TT;  // rows per work item
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* book = smem + C::STAGES * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(book);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + C::ACC;
  uint64_t* ifull = tempty + C::ACC;
  uint64_t* iempty = ifull + 2;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(iempty + 2);
  uint64_t* tbar = reinterpret_cast<uint64_t*>(book + 256);   // [2] table-tile arrivals
  int* s_info = reinterpret_cast<int*>(book + 512);          // [2] units per work item (for MMA)
  int* s_work = s_info + 4;                                  // u0, n_units, n_act (producers)
  uint32_t* s_mask = reinterpret_cast<uint32_t*>(book + 640);  // [2][16] per item parity
  int* s_na = reinterpret_cast<int*>(book + 800);              // [2] active offsets per parity
  uint64_t* sready = reinterpret_cast<uint64_t*>(book + 272);  // [2] item scan done (epilogue -> producers)
  int16_t* s_act = reinterpret_cast<int16_t*>(book + 1024);  // [2][512]: <= 343 entries per parity
  int32_t* s_tbl = reinterpret_cast<int32_t*>(book + C::BOOK);  // [2][TR * K] when K <= kTblK

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = p.K;
  long long* const trc = blockIdx.x == 0 ? p.trace : nullptr;
  // per-CTA record (trace on): [2048 + 4 b] = start, end (globaltimer ns), items, stages
  long long* const ctr = p.trace != nullptr ? p.trace + 2048 + 4 * blockIdx.x : nullptr;
  if (ctr != nullptr && threadIdx.x == 0) ctr[0] = (long long)tc::globaltimer();
  const int n_out = load_count(p.n_out_dev, p.cap_out);
  const int ntiles = (n_out + TR - 1) / TR;
  // split partials are sized for kNumSMs work items
  const int S = split_count(ntiles, min((int)gridDim.x, kSplitItems), p.max_split);
  const int total = ntiles * S;
  // BN partial rows: one per CTA that owns work (the split-K reduction
  // writes them instead when the tiles are split)
  const bool epi = p.epi.mode != 0 && S == 1;
  if (epi && blockIdx.x == 0 && tid == 0) *p.epi.nb = min((int)gridDim.x, total);
  if ((int)blockIdx.x >= total) {
    if (ctr != nullptr && tid == 0) ctr[1] = (long long)tc::globaltimer();
    return;
  }

  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      tc::mbar_init(&full[s], PROD);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < C::ACC; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], kTcEpi);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&ifull[i], 1);
      tc::mbar_init(&iempty[i], 1);
      tc::mbar_init(&tbar[i], 1);
      tc::mbar_init(&sready[i], 1);
    }
    tc::fence_mbar_init();
  }
  if (warp == PW + 4) tc::tmem_alloc(s_tmem, C::TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const uint32_t sbase = tc::smem_u32(smem);

  // BN statistics (epi): lane l of each epilogue warp accumulates channel
  // 32*j + l over the warp's rows of every item, in item order
  float bs1[ND / 32], bs2[ND / 32];
#pragma unroll
  for (int j = 0; j < ND / 32; ++j) bs1[j] = bs2[j] = 0.f;
  if (warp < PW) {
    // ============================ producers ============================
    constexpr bool tbl = TBL;
    // stage work item w's [rows, K] table block into buffer `buf` (thread 0):
    // one bulk copy of the 16 B-aligned prefix, the <= 3 trailing entries by
    // hand before the arrive (its release orders them)
    auto issue_tbl = [&](int w, int buf) {
      const int tile = w / S;
      const int nel = min(TR, n_out - tile * TR) * K;
      const int32_t* src = p.table + (int64_t)tile * TR * K;
      int32_t* dst = s_tbl + buf * TR * K;
      const int pre = nel & ~3;
      for (int e = pre; e < nel; ++e) dst[e] = __ldg(src + e);
      tc::fence_proxy_async_smem();
      tc::mbar_arrive_expect_tx(&tbar[buf], (uint32_t)pre * 4);
      if (pre > 0) tc::bulk_g2s(tc::smem_u32(dst), src, (uint32_t)pre * 4, &tbar[buf]);
    };
    if (tbl && tid == 0) issue_tbl(blockIdx.x, 0);
    uint32_t g = 0;
    int ii = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x, ++ii) {
      trace_ev(1024 + 4 * (ii & 63), tid == 0);
      const int tile = w / S, split = w - (w / S) * S;
      const int rows = min(TR, n_out - tile * TR);
      const int32_t* tt = s_tbl + (ii & 1) * TR * K;  // this item's staged table
      if (tbl) tc::mbar_wait(&tbar[ii & 1], (ii >> 1) & 1);  // landed (the scan waited too): makes it visible here
      asm volatile("bar.sync 1, %0;" ::"n"(PROD) : "memory");
      // the epilogue warps scanned this item's offset activity (scan_item)
      if (warp == 0 && lane == 0) {
        tc::mbar_wait(&sready[ii & 1], (ii >> 1) & 1);
        const int na = s_na[ii & 1];
        const int nu = C::PAIR ? (na + 1) / 2 : na * C::NCH;
        const int u0 = (int)((int64_t)nu * split / S), u1 = (int)((int64_t)nu * (split + 1) / S);
        s_work[0] = u0;
        s_work[1] = u1 - u0;
        s_work[2] = na;
        const int slot = ii & 1;
        if (ii >= 2) tc::mbar_wait(&iempty[slot], ((ii >> 1) - 1) & 1);
        s_info[slot] = max(u1 - u0, 1);
        trace_ev(1024 + 4 * (ii & 63) + 1, true);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&ifull[slot])) : "memory");
        // every producer is past tile ii-1 (barrier below at ii-1's end): its buffer is free
        if (tbl && w + (int)gridDim.x < total) issue_tbl(w + gridDim.x, (ii + 1) & 1);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(PROD) : "memory");
      const int u0 = s_work[0], nun = s_work[1], na = s_work[2];
      const int neff = nun > 0 ? nun : 1;
      // unit -> (offset of A's first half / whole row, second half, 64-col slice)
      const uint32_t s_act_s = tc::smem_u32(s_act + (ii & 1) * 512);
      auto unit_k = [&](int unit, int& ka, int& kb, int& cs) {
        kb = -1;
        cs = 0;
        if (nun == 0) {
          ka = -1;  // zero unit: A = 0, B = any finite weights
        } else if (C::PAIR) {
          ka = tc::lds_s16(s_act_s + 4 * unit);
          kb = (2 * unit + 1 < na) ? tc::lds_s16(s_act_s + 4 * unit + 2) : -1;
        } else {
          ka = tc::lds_s16(s_act_s + 2 * (unit / C::NCH));
          cs = unit % C::NCH;
        }
      };
      // A: 8 lanes per row (16 B chunk q each); this lane's rows are
      // r_i = r0 + 4i, i < 8.  Row r_i's chunk lands at a_s + r_i*128 +
      // ((q ^ (r_i & 7)) << 4) and r_i & 7 = (lane/8) + 4*(i&1).
      const int q = lane & 7;
      const int r0 = warp * (128 / PW) + (lane >> 3);
      const uint32_t a_off0 = r0 * 128 + ((q ^ (lane >> 3)) << 4);
      const uint32_t a_off1 = r0 * 128 + ((q ^ ((lane >> 3) + 4)) << 4);
      const uint32_t tt_s = tc::smem_u32(tt) + r0 * K * 4;  // row r0's staged table entries
      const int32_t* trow0 = p.table + ((int64_t)tile * TR + r0) * K;
      const char* xb = reinterpret_cast<const char*>(p.x);
      const int nst = (neff + RB - 1) / RB;  // stages of this work item
      for (int sj = 0; sj < nst; ++sj, ++g) {
        const int stage = g % C::STAGES;
        if (g >= (uint32_t)C::STAGES) tc::mbar_wait(&empty[stage], ((g / C::STAGES) - 1) & 1);
        trace_ev(4 * (g & 255), tid == 0 && g < 256);
        const uint32_t s_base = sbase + stage * C::STAGE;
        const int na_st = min(RB, neff - sj * RB);  // atoms in use (the MMA skips the rest)
#pragma unroll 1
        for (int at = 0; at < na_st; ++at) {
          const uint32_t a_s0 = s_base + at * TT * C::A_BYTES;
          const uint32_t b_s = s_base + RB * TT * C::A_BYTES + at * C::B_BYTES;
          const int unit = u0 + sj * RB + at;
          int ka, kb, cs;
          unit_k(unit, ka, kb, cs);
#pragma unroll
          for (int t = 0; t < TT; ++t) {
            const uint32_t a_s = a_s0 + t * C::A_BYTES;
            const int kq = C::PAIR ? (q < 4 ? ka : kb) : ka;
            const int col = p.flip ? K - 1 - kq : kq;
            const int ch = C::PAIR ? (q & 3) * 8 : cs * 64 + q * 8;  // first element of this lane's 16 B chunk
            const bool chv = ch < kreal;                               // padded widths: zero chunk
            const char* xq = xb + 2 * (chv ? ch : 0);
            int vr[RPT];
            const bool noa = p.dbg & 4;
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
              if (kq < 0 || noa) vr[i] = -1;
              else if (TBL) vr[i] = tc::lds_s32(tt_s + (uint32_t)((t * 128 * K + i * 4 * K + col) * 4));
              else vr[i] = (t * 128 + r0 + 4 * i < rows) ? __ldg(trow0 + (t * 128 + i * 4) * K + col) : -1;
            }
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
              const int v = vr[i];
              tc::cp_async16(a_s + ((i & 1) ? a_off1 : a_off0) + i * 512,
                             xq + (int64_t)(v > 0 ? v : 0) * (kreal * 2), (v >= 0 && chv) ? 16 : 0);
            }
          }
          // ---- B
          const int kA = ka >= 0 ? ka : 0;
          const int kB = kb >= 0 ? kb : kA;
          if (p.dbg & 2) {
          } else if (!BMN) {  // B[n][kk] = W[k][n][slice] (K-major rows of W); thread: chunk qq = tid & 7, rows n = tid/8 + 16j
            const int qq = tid & 7, n0 = tid >> 3;
            const int k = (C::PAIR && qq >= 4) ? kB : kA;
            const int bc = C::PAIR ? (qq & 3) * 8 : cs * 64 + qq * 8;
            const bool bcv = bc < kreal;
            const bf16* src = p.w + ((int64_t)k * nreal + n0) * kreal + (bcv ? bc : 0);
            const uint32_t dst = b_s + n0 * 128 + ((qq ^ (n0 & 7)) << 4);
            constexpr int NR = PROD / 8;  // B rows per pass
#pragma unroll
            for (int j = 0; j < ND / NR; ++j) {
              const bool ok = bcv && n0 + j * NR < nreal;
              tc::cp_async16(dst + j * NR * 128, ok ? src + (int64_t)j * NR * kreal : p.w, ok ? 16 : 0);
            }
          } else {  // B(n, kk) = W[k][kk][n]: row kk of W_k is N-contiguous (MN-major)
            constexpr int NCHK = ND / 8;        // 16 B chunks per kk row
            constexpr int KKS = PROD / NCHK;  // kk rows per pass
            const int jn = tid % NCHK, kk0 = tid / NCHK;
#pragma unroll
            for (int j = 0; j < 64 / KKS; ++j) {
              const int kk = kk0 + j * KKS;
              const bf16* src;
              int kr;  // row of W_k (the gathered width)
              if (C::PAIR) {
                const int k = kk < 32 ? kA : kB;
                kr = kk & 31;
                src = p.w + ((int64_t)k * kreal + kr) * nreal + jn * 8;
              } else {
                kr = cs * 64 + kk;
                src = p.w + ((int64_t)kA * kreal + kr) * nreal + jn * 8;
              }
              const bool ok = kr < kreal && jn * 8 < nreal;
              const uint32_t off =
                  (uint32_t)((jn >> 3) * 8192 + (kk >> 3) * 1024 + (kk & 7) * 128 + (((jn & 7) ^ (kk & 7)) << 4));
              tc::cp_async16(b_s + off, ok ? src : p.w, ok ? 16 : 0);
            }
          }
        }
        // the stage's full barrier completes when every producer's copies have landed
        tc::cp_async_arrive_noinc(&full[stage]);
        trace_ev(4 * (g & 255) + 1, tid == 0 && g < 256);
      }
    }
    tc::cp_async_wait<0>();
    if (ctr != nullptr && tid == 0) {
      ctr[2] = ii;
      ctr[3] = g;
    }
  } else if (warp < PW + 4) {
    // ============================ epilogue ============================
    const int ep = warp - PW;
    const int etid = tid - PROD;
    // Offset-activity scan of the CTA's iiw-th item (work item wi) into buffer
    // iiw & 1: OR of the rows' neighbour-hit masks -> ascending active-offset
    // list + count, then sready.  Run here, in the epilogue warps' slack, so
    // the producers only publish at a tile boundary.
    auto scan_item = [&](int wi, int iiw) {
      const int b = iiw & 1;
      const int tile_w = wi / S;
      const int rows_w = min(TR, n_out - tile_w * TR);
      uint32_t* msk = s_mask + b * 16;
      if (etid < kTcMaskWords) msk[etid] = 0;
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (TBL) {
        tc::mbar_wait(&tbar[b], (iiw >> 1) & 1);
        int32_t* tw = s_tbl + b * TR * K;
        if (rows_w < TR)  // ragged last tile: rows past the end read as misses
          for (int e = rows_w * K + etid; e < TR * K; e += kTcEpi) tw[e] = -1;
        if (p.dbg & 16) {  // experiment: every offset active, no scan
          if (etid == 0) msk[0] = K >= 32 ? 0xffffffffu : (1u << K) - 1u;
        } else {
          uint32_t bits = 0;
#pragma unroll
          for (int t = 0; t < TT; ++t) {
            const int r = etid + 128 * t;
            if (r < rows_w) {
              if (K == 27) {  // 3^3: all 27 shared-memory loads in flight
                uint32_t m = 0;
#pragma unroll
                for (int k = 0; k < 27; ++k) m |= (tw[r * 27 + k] >= 0 ? 1u : 0u) << k;
                bits |= p.flip ? (__brev(m) >> 5) : m;
              } else {
                for (int k = 0; k < K; ++k)
                  if (tw[r * K + k] >= 0) bits |= 1u << (p.flip ? K - 1 - k : k);
              }
            }
          }
          bits = __reduce_or_sync(0xffffffffu, bits);
          if (lane == 0 && bits) atomicOr(&msk[0], bits);
        }
      } else {
        for (int kb = 0; kb < K; kb += 32) {
          uint32_t bits = 0;
          const int kend = min(32, K - kb);
          for (int t = 0; t < TT; ++t) {
            const int r = etid + 128 * t;
            const int32_t* trow = p.table + ((int64_t)tile_w * TR + r) * K;
            for (int j = 0; j < kend; ++j) {
              const int k = kb + j;
              const int v = r < rows_w ? __ldg(trow + (p.flip ? K - 1 - k : k)) : -1;
              if (v >= 0) bits |= 1u << j;
            }
          }
          bits = __reduce_or_sync(0xffffffffu, bits);
          if (lane == 0 && bits) atomicOr(&msk[kb >> 5], bits);
        }
      }
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (ep == 0) {
        int16_t* act = s_act + b * 512;
        int na = 0;
        for (int kb = 0; kb < K; kb += 32) {
          const uint32_t m = msk[kb >> 5];
          if (m & (1u << lane)) act[na + __popc(m & ((1u << lane) - 1u))] = (int16_t)(kb + lane);
          na += __popc(m);
        }
        __syncwarp();
        if (lane == 0) {
          s_na[b] = na;
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(&sready[b])) : "memory");
        }
      }
    };
    if ((int)blockIdx.x < total) scan_item(blockIdx.x, 0);
    int ii = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x, ++ii) {
      const int tile = w / S, split = w - (w / S) * S;
      // next item's scan: once item ii is published its producers are past
      // item ii-1, whose mask / list / table buffers the scan reuses
      if (w + (int)gridDim.x < total) {
        tc::mbar_wait(&ifull[ii & 1], (ii >> 1) & 1);
        scan_item(w + gridDim.x, ii + 1);
      }
      const int a = ii % C::ACC;
      if (epi && p.epi.mode == 2 && !(p.dbg & 256)) {
        // this item's rows of the BN operands (add / act / pre) head for L2
        // while the accumulator is still being produced: per-line prefetch
        // (C3 51.6k -> 51.9k clouds/s; VP_CONV_DBG bit 5: bulk prefetch
        // instead, bit 8: off)
#pragma unroll 1
        for (int t = 0; t < TT; ++t) {
          const int64_t row = (int64_t)tile * TR + t * 128 + ep * 32 + lane;
          if (row < n_out) {
            const int64_t orow = p.perm != nullptr ? (int64_t)__ldg(p.perm + row) : row;
            const int64_t off = orow * ND * 2;
            const char* srcs[3] = {reinterpret_cast<const char*>(p.epi.add), reinterpret_cast<const char*>(p.epi.act),
                                   reinterpret_cast<const char*>(p.epi.pre)};
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              if (srcs[q] == nullptr) continue;
              if (p.dbg & 32) {
                tc::prefetch_l2(srcs[q] + off, ND * 2);
              } else {
#pragma unroll
                for (int l = 0; l < ND * 2; l += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(srcs[q] + off + l));
              }
            }
          }
        }
      }
      tc::mbar_wait(&tfull[a], (ii / C::ACC) & 1);
      trace_ev(1024 + 4 * (ii & 63) + 2, ep == 0 && lane == 0);
      tc::tc_fence_after();
      const int lrow = ep * 32 + lane;
#pragma unroll 1
      for (int t = 0; t < TT; ++t) {
      const int64_t row = (int64_t)tile * TR + t * 128 + lrow;
      const int64_t orow = (p.perm != nullptr && row < n_out) ? (int64_t)__ldg(p.perm + row) : row;
      if (epi) {  // bf16 output + BN statistics (all lanes: the sums are warp-collective)
#pragma unroll 1
        for (int j = 0; j < ND / 32; ++j) {
          float v[32];
          tc::tmem_ld32(tmem + ((uint32_t)(ep * 32) << 16) + (a * TT + t) * ND + 32 * j, v);
          float s1, s2;
          bn_epi_chunk32<ND>(p.epi, v, row < n_out, orow, 32 * j, reinterpret_cast<bf16*>(p.y), s1, s2);
#pragma unroll
          for (int jj = 0; jj < ND / 32; ++jj)  // register-resident accumulators (no dynamic index)
            if (jj == j) {
              bs1[jj] += s1;
              bs2[jj] += s2;
            }
        }
        continue;
      }
#pragma unroll 1
      for (int c0 = 0; c0 < ND; c0 += 32) {
        float v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(ep * 32) << 16) + (a * TT + t) * ND + c0, v);
        if (row < n_out) {
          if (S > 1) {
            float4* dst = reinterpret_cast<float4*>(p.part + (((int64_t)split * ntiles + tile) * 128 + lrow) * ND + c0);
#pragma unroll
            for (int q = 0; q < 8; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          } else if (p.y_dtype == VP_BF16) {
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(p.y) + orow * nreal + c0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 pk;
              __nv_bfloat162 h0 = __floats2bfloat162_rn(v[8 * q + 0], v[8 * q + 1]);
              __nv_bfloat162 h1 = __floats2bfloat162_rn(v[8 * q + 2], v[8 * q + 3]);
              __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * q + 4], v[8 * q + 5]);
              __nv_bfloat162 h3 = __floats2bfloat162_rn(v[8 * q + 6], v[8 * q + 7]);
              pk.x = *reinterpret_cast<uint32_t*>(&h0);
              pk.y = *reinterpret_cast<uint32_t*>(&h1);
              pk.z = *reinterpret_cast<uint32_t*>(&h2);
              pk.w = *reinterpret_cast<uint32_t*>(&h3);
              if (c0 + 8 * q < nreal) dst[q] = pk;
            }
          } else {
            float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.y) + orow * nreal + c0);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (c0 + 4 * q < nreal) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          }
        }
      }
      }  // t
      tc::tc_fence_before();
      tc::mbar_arrive(&tempty[a]);
      trace_ev(1024 + 4 * (ii & 63) + 3, ep == 0 && lane == 0);
    }
  } else if (lane == 0) {
    // ============================ MMA issuer ============================
    uint32_t g = 0;
    int ii = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x, ++ii) {
      const int slot = ii & 1;
      tc::mbar_wait(&ifull[slot], (ii >> 1) & 1);
      const int neff = s_info[slot];
      tc::mbar_arrive(&iempty[slot]);
      const int a = ii % C::ACC;
      const int use = ii / C::ACC;
      if (use >= 1) tc::mbar_wait(&tempty[a], (use - 1) & 1);
      tc::tc_fence_after();
      const uint32_t d = tmem + a * TT * ND;
      const int nst = (neff + RB - 1) / RB;
      for (int sj = 0; sj < nst; ++sj, ++g) {
        const int stage = g % C::STAGES;
        tc::mbar_wait(&full[stage], (g / C::STAGES) & 1);
        trace_ev(4 * (g & 255) + 2, g < 256);
        tc::tc_fence_after();
        const uint32_t s_base = sbase + stage * C::STAGE;
        const int na_st = (p.dbg & 1) ? 0 : min(RB, neff - sj * RB);
        for (int at = 0; at < na_st; ++at) {
          const uint32_t a_s = s_base + at * TT * C::A_BYTES;
          const uint32_t b_s = s_base + RB * TT * C::A_BYTES + at * C::B_BYTES;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t bd = BMN ? tc::smem_desc(b_s + kk * 2048, 8192, 1024, tc::kSwizzle128)
                                    : tc::smem_desc(b_s + kk * 32, 16, 1024, tc::kSwizzle128);
#pragma unroll
            for (int t = 0; t < TT; ++t) {
              const uint64_t ad = tc::smem_desc(a_s + t * C::A_BYTES + kk * 32, 16, 1024, tc::kSwizzle128);
              if constexpr (TF32) tc::mma_tf32(d + t * ND, ad, bd, C::IDESC, (sj > 0 || at > 0 || kk > 0) ? 1u : 0u);
              else tc::mma_bf16(d + t * ND, ad, bd, C::IDESC, (sj > 0 || at > 0 || kk > 0) ? 1u : 0u);
            }
          }
        }
        if (p.dbg & 8) tc::mbar_arrive(&empty[stage]);
        else tc::mma_commit(&empty[stage]);
        trace_ev(4 * (g & 255) + 3, g < 256);
      }
      tc::mma_commit(&tfull[a]);
    }
  }
  __syncthreads();
  if (ctr != nullptr && tid == 0) ctr[1] = (long long)tc::globaltimer();
  if (warp == PW + 4) tc::tmem_dealloc(tmem, C::TMEM_COLS);
  if (epi && warp >= PW && warp < PW + 4) {
    // the 4 warps' sums in warp order -> this CTA's partial row (the stage
    // ring is free: every copy and MMA has completed)
    float* red = reinterpret_cast<float*>(smem);  // [4][2][ND]
    const int ep = warp - PW, etid = tid - PROD;
#pragma unroll
    for (int j = 0; j < ND / 32; ++j) {
      red[(ep * 2 + 0) * ND + 32 * j + lane] = bs1[j];
      red[(ep * 2 + 1) * ND + 32 * j + lane] = bs2[j];
    }
    asm volatile("bar.sync 2, 128;" ::: "memory");
    float* dst = p.epi.part + (int64_t)blockIdx.x * 2 * ND;
    for (int e = etid; e < 2 * ND; e += kTcEpi) {
      const int h = e / ND, c = e - h * ND;
      float acc = 0.f;
#pragma unroll
      for (int w = 0; w < 4; ++w) acc += red[(w * 2 + h) * ND + c];
      dst[e] = acc;
    }
  }
}

// out[r, n] = sum over splits of the fp32 partials, in split order.
static __global__ void split_reduce_kernel(const float* __restrict__ part, const int32_t* n_out_dev, int64_t cap_out, int ND,
                                    int grid, int max_split, const int32_t* __restrict__ perm, void* __restrict__ y,
                                    int y_dtype, int nreal) {
  ::vp::pdl_begin();
  const int n_out = load_count(n_out_dev, cap_out);
  const int ntiles = (n_out + 127) / 128;
  const int S = split_count(ntiles, grid < kSplitItems ? grid : kSplitItems, max_split);
  if (S <= 1) return;
  const int64_t total = (int64_t)n_out * ND / 4;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t idx = e * 4;
    const int64_t r = idx / ND;
    const int n = (int)(idx - r * ND);
    const int tile = (int)(r >> 7), lr = (int)(r & 127);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int s = 0; s < S; ++s) {  // loads batched, sums stay in split order
      const float4 v = *reinterpret_cast<const float4*>(part + (((int64_t)s * ntiles + tile) * 128 + lr) * ND + n);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    if (n >= nreal) continue;  // padded columns
    const int64_t oidx = (perm ? (int64_t)__ldg(perm + r) : r) * nreal + n;
    if (y_dtype == VP_BF16) {
      __nv_bfloat162* d = reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<bf16*>(y) + oidx);
      d[0] = __floats2bfloat162_rn(acc.x, acc.y);
      d[1] = __floats2bfloat162_rn(acc.z, acc.w);
    } else {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + oidx) = acc;
    }
  }
}

// split_reduce_kernel + the BN epilogue (bn_epi.cuh) for a bf16 output:
// thread t always owns channels [(4t) % ND, +4) (ND divides 4 NT), so its
// statistics accumulate in registers; the block then sums its threads in a
// fixed order into partial row blockIdx.x.
constexpr int kSplitEpiThreads = 1024;  // wide blocks: <= 148 partial rows, as many threads as the plain reduction
template <int ND, int NT = kSplitEpiThreads>
__global__ void __launch_bounds__(NT)
split_reduce_epi_kernel(const float* __restrict__ part, const int32_t* n_out_dev, int64_t cap_out, int grid,
                        int max_split, const int32_t* __restrict__ perm, bf16* __restrict__ y, const BnEpi e) {
  ::vp::pdl_begin();
  __shared__ float s_red[2][NT][4];
  __shared__ double s_fin[32][33];
  __shared__ unsigned int s_last;
  const int n_out = load_count(n_out_dev, cap_out);
  const int ntiles = (n_out + 127) / 128;
  const int S = split_count(ntiles, grid < kSplitItems ? grid : kSplitItems, max_split);
  if (e.out_a && e.early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const bool rows = S <= 1 && e.rows_pass;  // the conv stored raw rows: transform them here
  if (S <= 1 && !rows) {
    // the conv epilogue wrote the partial rows: finalize them here (one
    // 32-channel block per CTA) instead of in a separate launch
    if constexpr (NT == 1024) {  // the finalize needs 1024-thread blocks
      if (e.out_a && (int)blockIdx.x * 32 < ND)
        bn_finalize_block(e.part, *e.nb, ND, n_out, e.mode, e.eps, e.rstd, e.out_a, e.out_b, blockIdx.x, s_fin);
    }
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *e.nb = gridDim.x;
  const int n = (threadIdx.x * 4) % ND;
  float a[4] = {0.f, 0.f, 0.f, 0.f}, b[4] = {0.f, 0.f, 0.f, 0.f};
  const int64_t total = (int64_t)n_out * ND / 4;
  for (int64_t el = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; el < total; el += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = el * 4 / ND;
    const int tile = (int)(r >> 7), lr = (int)(r & 127);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t oidx;
    if (rows) {  // output rows are already in place (perm applied by the conv)
      oidx = r * ND + n;
      const uint2 raw = *reinterpret_cast<const uint2*>(y + oidx);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
      const float2 f0 = __bfloat1622float2(h[0]), f1 = __bfloat1622float2(h[1]);
      acc = make_float4(f0.x, f0.y, f1.x, f1.y);
    } else {
#pragma unroll 4
      for (int s = 0; s < S; ++s) {  // loads batched, sums stay in split order
        const float4 v = *reinterpret_cast<const float4*>(part + (((int64_t)s * ntiles + tile) * 128 + lr) * ND + n);
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
      oidx = (perm ? (int64_t)__ldg(perm + r) : r) * ND + n;
    }
    float v[4] = {acc.x, acc.y, acc.z, acc.w}, o[4], h[4];
    if (e.mode == 2) {
      uint2 ra = e.add ? __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const bf16*>(e.add) + oidx))
                       : make_uint2(0u, 0u);
      uint2 rc = e.act ? __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const bf16*>(e.act) + oidx))
                       : make_uint2(0x3f803f80u, 0x3f803f80u);
      uint2 rp = __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const bf16*>(e.pre) + oidx));
      const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&ra);
      const __nv_bfloat162* hc = reinterpret_cast<const __nv_bfloat162*>(&rc);
      const __nv_bfloat162* hp = reinterpret_cast<const __nv_bfloat162*>(&rp);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float2 fa = __bfloat1622float2(ha[q]), fc = __bfloat1622float2(hc[q]), fp = __bfloat1622float2(hp[q]);
        const float fa2[2] = {fa.x, fa.y}, fc2[2] = {fc.x, fc.y}, fp2[2] = {fp.x, fp.y};
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int c = 2 * q + j;
          const float g = bf16_round(v[c]) + fa2[j];
          o[c] = fc2[j] > 0.f ? bf16_round(g) : 0.f;
          h[c] = o[c] * (fp2[j] - __ldg(e.mean + n + c));
        }
      }
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        o[c] = bf16_round(v[c]);
        h[c] = o[c] * o[c];
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      a[c] += o[c];
      b[c] += h[c];
    }
    __nv_bfloat162* d = reinterpret_cast<__nv_bfloat162*>(y + oidx);
    d[0] = __floats2bfloat162_rn(o[0], o[1]);
    d[1] = __floats2bfloat162_rn(o[2], o[3]);
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    s_red[0][threadIdx.x][c] = a[c];
    s_red[1][threadIdx.x][c] = b[c];
  }
  __syncthreads();
  constexpr int G = ND / 4, M = NT * 4 / ND;  // channel quads, threads per quad
  for (int idx = threadIdx.x; idx < 2 * ND; idx += blockDim.x) {
    const int hh = idx / ND, c = idx - hh * ND;
    float acc = 0.f;
#pragma unroll
    for (int m = 0; m < M; ++m) acc += s_red[hh][c / 4 + m * G][c % 4];
    e.part[((int64_t)blockIdx.x * 2 + hh) * ND + c] = acc;
  }
  if (e.out_a == nullptr) return;
  // the last block to finish (self-re-arming ticket) finalizes every channel
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicInc(e.ticket, gridDim.x - 1) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if constexpr (NT == 1024)
    for (int cb = 0; cb * 32 < ND; ++cb)
      bn_finalize_block(e.part, (int)gridDim.x, ND, n_out, e.mode, e.eps, e.rstd, e.out_a, e.out_b, cb, s_fin);
}

}  // namespace vp
