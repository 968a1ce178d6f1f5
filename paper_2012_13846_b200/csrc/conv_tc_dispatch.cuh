// Tensor-core conv dispatch: (C_in, C_out, operand layout) -> the
// implicit-GEMM instantiation and its (CTAs/SM, atoms/stage) config.  The
// instantiations are compiled in one translation unit per (K width, B
// layout) (conv_tc_*.cu) so the library builds in parallel.
#pragma once
#include <algorithm>
#include <string>

#include "common.cuh"
#include "conv_fwd_tc.cuh"

namespace vp {

constexpr int kMaxSplit = 16;

template <int KD, int ND, bool BMN, int CPS, int RB, int TT = 1, int MODE = 0, int PW = 4>
inline int launch_conv_tc(const FwdParams& p0, void* part, cudaStream_t st) {
  using C = FwdTC<KD, ND, BMN, CPS, RB, TT, MODE>;
  const bool tbl = p0.K <= kTblK && ((uintptr_t)p0.table & 15) == 0;
  auto kern = tbl ? conv_tc_kernel<KD, ND, BMN, CPS, RB, true, TT, MODE, PW>
                  : conv_tc_kernel<KD, ND, BMN, CPS, RB, false, TT, MODE, PW>;
  static_assert(C::SMEM_MAX <= 227 * 1024, "conv_tc: shared memory over the per-CTA limit");
  static bool attr_t = false, attr_f = false;  // immutable per-instantiation attribute cache
  bool& attr = tbl ? attr_t : attr_f;
  if (!attr) {
    VP_REQUIRE(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_MAX) == cudaSuccess,
               VP_EINTERNAL, "conv_tc: cannot reserve shared memory");
    attr = true;
  }
  const int64_t tiles = ceil_div(p0.cap_out, 128 * TT);
  if (TT > 1) part = nullptr;  // multi-tile items are only used where no split-K is needed
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles * kMaxSplit, (int64_t)kNumSMs * CPS));
  FwdParams p = p0;
  p.part = (float*)part;
  // backward-BN transform of wide outputs as a row pass in the split-K
  // reduction kernel instead of the epilogue (VP_EPI_ROWS_MIN_ND, default 64)
  static const int rows_min_nd = getenv("VP_EPI_ROWS_MIN_ND") ? atoi(getenv("VP_EPI_ROWS_MIN_ND")) : 64;
  BnEpi rows_epi{};
  bool rows_pass = false;
  if (p.epi.mode == 2 && ND >= rows_min_nd && rows_min_nd > 0 && part != nullptr) {
    rows_pass = true;
    rows_epi = p.epi;
    rows_epi.rows_pass = 1;
    p.epi = BnEpi{};  // plain epilogue
  }
  static const int max_split = getenv("VP_CONV_MAX_SPLIT") ? std::max(1, std::min(kMaxSplit, atoi(getenv("VP_CONV_MAX_SPLIT"))))
                                                          : kMaxSplit;  // tuning
  p.max_split = part ? max_split : 1;
  p.stage_tbl = tbl;
  static const int dbg = getenv("VP_CONV_DBG") ? atoi(getenv("VP_CONV_DBG")) : 0;
  p.dbg = dbg;
  p.trace = g_conv_trace_host;
  ::vp::launch(kern, grid, tc_threads<PW>(), C::smem_bytes(p0.K, p.stage_tbl), st, p);
  VP_CHECK_LAUNCH("conv_tc");
  if (rows_pass) {
    // 256-thread blocks: schedulable next to the side-stream kernels (1024-thread
    // blocks waited for half an SM); up to kBnPartRows partial rows
    constexpr int NT = 256;
    const int64_t work = p.cap_out * ND / 4;
    // partial rows = blocks: the finalize below reads them all (VP_ROWS_PASS_BLOCKS caps them, tuning)
    static const int64_t rp_cap = getenv("VP_ROWS_PASS_BLOCKS") ? std::max(1, atoi(getenv("VP_ROWS_PASS_BLOCKS"))) : kBnPartRows;
    const int64_t blocks = std::max<int64_t>(std::min<int64_t>(ceil_div(work, NT * 4), std::min<int64_t>(rp_cap, kBnPartRows)), 1);
    BnEpi e = rows_epi;
    e.out_a = e.out_b = nullptr;  // finalized by the 32-channel-per-block kernel below
    ::vp::launch(split_reduce_epi_kernel<ND, NT>, (int)blocks, NT, 0, st, (const float*)part, p.n_out_dev,
                 p.cap_out, grid, p.max_split, p.perm, (bf16*)p.y, e);
    VP_CHECK_LAUNCH("split_reduce_epi");
    if (rows_epi.out_a) {
      ::vp::launch(bn_finalize_kernel, (int)ceil_div(ND, 32), 1024, 0, st, rows_epi, ND, p.n_out_dev, p.cap_out);
      VP_CHECK_LAUNCH("bn_finalize");
    }
  } else if (part && p.epi.mode != 0) {  // bf16 output + BN statistics: at most one partial row per SM
    const int64_t work = p.cap_out * ND / 4;
    // >= one block per 32 channels: without a split they finalize the conv's partial rows.
    // When even the capacity's tile count is split for sure (few rows), the
    // ~148 reduction rows are finalized by a separate 32-channel-per-block
    // kernel instead of the split kernel's last block (a serial tail).
    const int64_t tiles_cap = ceil_div(p.cap_out, 128);
    const bool split_sure = tiles_cap * 2 <= std::min<int64_t>(grid, kSplitItems) && p.max_split > 1;
    BnEpi e = p.epi;
    if (split_sure) e.out_a = e.out_b = nullptr;
    const int64_t blocks = std::max<int64_t>(std::min<int64_t>(ceil_div(work, kSplitEpiThreads), kNumSMs), ND / 32);
    ::vp::launch(split_reduce_epi_kernel<ND>, (int)blocks, kSplitEpiThreads, 0, st, (const float*)part, p.n_out_dev,
                 p.cap_out, grid, p.max_split, p.perm, (bf16*)p.y, e);
    VP_CHECK_LAUNCH("split_reduce_epi");
    if (split_sure && p.epi.out_a) {
      ::vp::launch(bn_finalize_kernel, (int)ceil_div(ND, 32), 1024, 0, st, p.epi, ND, p.n_out_dev, p.cap_out);
      VP_CHECK_LAUNCH("bn_finalize");
    }
  } else if (p.epi.mode != 0 && p.epi.out_a) {  // statistics rows from the epilogue only: finalize them
    ::vp::launch(bn_finalize_kernel, (int)ceil_div(ND, 32), 1024, 0, st, p.epi, ND, p.n_out_dev, p.cap_out);
    VP_CHECK_LAUNCH("bn_finalize");
  } else if (part) {
    const int64_t work = p.cap_out * ND / 4;
    ::vp::launch(split_reduce_kernel, (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, 256), grid_cap(8))), 256, 0, st, 
        (const float*)part, p.n_out_dev, p.cap_out, ND, grid, p.max_split, p.perm, p.y, p.y_dtype, p.nreal);
    VP_CHECK_LAUNCH("split_reduce");
  }
  return VP_OK;
}

// (CTAs per SM, atoms per stage) candidates for the gather-bound implicit
// GEMM; conv_cfg picks one per output width (VP_CONV_CFG=i overrides, for
// tuning).  Infeasible ones (ring < 2 stages, TMEM) fall through.
constexpr int kCfgCps[] = {1, 1, 2, 2, 3};
constexpr int kCfgRb[] = {2, 1, 2, 1, 1};

inline int conv_cfg(int64_t nd, int64_t cap_out) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("VP_CONV_CFG");
    env = e ? atoi(e) : -1;
  }
  if (env >= 0 && env < 5) return env;
  // per output width (VP_CONV_CFG_<ND>, tuning)
  static int per[4] = {-2, -2, -2, -2};
  const int slot = nd == 32 ? 0 : nd == 64 ? 1 : nd == 128 ? 2 : 3;
  if (per[slot] == -2) {
    const std::string name = "VP_CONV_CFG_" + std::to_string(nd);
    const char* e = getenv(name.c_str());
    per[slot] = e ? atoi(e) : -1;
  }
  if (per[slot] >= 0 && per[slot] < 5) return per[slot];
  // C_out = 128 at <= 64k rows (C3's level 3: ~80 tiles, split-K): one CTA
  // per SM with single-atom stages measured 45.9k -> 47.2k clouds/s
  if (nd == 128 && cap_out <= 65536) return 1;
  return 3;
}

template <int KD, int ND, bool BMN, int I>
inline int try_cfg(const FwdParams& p, void* part, cudaStream_t st) {
  using C = FwdTC<KD, ND, BMN, kCfgCps[I], kCfgRb[I]>;
  if constexpr (C::FITS) return launch_conv_tc<KD, ND, BMN, kCfgCps[I], kCfgRb[I]>(p, part, st);
  return -1;
}

// rows at which a 256-row work item (two tiles sharing each weight stage)
// replaces the 128-row one for C_out >= 128: enough 256-row items to fill
// the machine without split-K (VP_CONV_TT2_ROWS overrides; 0 disables)
inline int64_t tt2_rows() {
  static const int64_t v = getenv("VP_CONV_TT2_ROWS") ? atoll(getenv("VP_CONV_TT2_ROWS")) : 0;  // off by default: at 1M rows it helps strided dgrad (-9%) but slows C=256 fwd (+14%)
  return v;
}

template <int KD, int ND, bool BMN>
inline int launch_conv_tc_cfg(const FwdParams& p, void* part, cudaStream_t st) {
  if constexpr (ND >= 128 && FwdTC<KD, ND, BMN, 1, 1, 2>::FITS) {
    if (tt2_rows() > 0 && p.cap_out >= tt2_rows()) return launch_conv_tc<KD, ND, BMN, 1, 1, 2>(p, part, st);
  }
  int r = -1;
  switch (conv_cfg(ND, p.cap_out)) {
    case 0: r = try_cfg<KD, ND, BMN, 0>(p, part, st); break;
    case 1: r = try_cfg<KD, ND, BMN, 1>(p, part, st); break;
    case 2: r = try_cfg<KD, ND, BMN, 2>(p, part, st); break;
    case 3: r = try_cfg<KD, ND, BMN, 3>(p, part, st); break;
    case 4: r = try_cfg<KD, ND, BMN, 4>(p, part, st); break;
  }
  if (r >= 0) return r;
  r = try_cfg<KD, ND, BMN, 0>(p, part, st);  // (1, 2): fits every width but 256
  if (r >= 0) return r;
  return launch_conv_tc<KD, ND, BMN, 1, 1>(p, part, st);
}

template <int KD, bool BMN>
inline int conv_tc_nd(int64_t nd, const FwdParams& p, void* part, cudaStream_t st) {
  switch (nd) {
    case 32: return launch_conv_tc_cfg<KD, 32, BMN>(p, part, st);
    case 64: return launch_conv_tc_cfg<KD, 64, BMN>(p, part, st);
    case 128: return launch_conv_tc_cfg<KD, 128, BMN>(p, part, st);
    case 256: return launch_conv_tc_cfg<KD, 256, BMN>(p, part, st);
  }
  return VP_EINTERNAL;
}


// padded bf16 (MODE 1) and tf32 (MODE 2, K-major weights only): the default
// config and its fallbacks
template <int KD, int ND, bool BMN, int MODE>
inline int launch_conv_mode(const FwdParams& p, void* part, cudaStream_t st) {
  if constexpr (FwdTC<KD, ND, BMN, kCfgCps[3], kCfgRb[3], 1, MODE>::FITS)
    return launch_conv_tc<KD, ND, BMN, kCfgCps[3], kCfgRb[3], 1, MODE>(p, part, st);
  else if constexpr (FwdTC<KD, ND, BMN, kCfgCps[0], kCfgRb[0], 1, MODE>::FITS)
    return launch_conv_tc<KD, ND, BMN, kCfgCps[0], kCfgRb[0], 1, MODE>(p, part, st);
  else
    return launch_conv_tc<KD, ND, BMN, 1, 1, 1, MODE>(p, part, st);
}

template <int KD, bool BMN, int MODE>
inline int conv_mode_nd(int64_t nd, const FwdParams& p, void* part, cudaStream_t st) {
  switch (nd) {
    case 32: return launch_conv_mode<KD, 32, BMN, MODE>(p, part, st);
    case 64: return launch_conv_mode<KD, 64, BMN, MODE>(p, part, st);
    case 128: return launch_conv_mode<KD, 128, BMN, MODE>(p, part, st);
    case 256: return launch_conv_mode<KD, 256, BMN, MODE>(p, part, st);
  }
  return VP_EINTERNAL;
}

template <bool BMN, int MODE>
inline int conv_mode(int64_t kd, int64_t nd, const FwdParams& p, void* part, cudaStream_t st) {
  switch (kd) {
    case 32: return conv_mode_nd<32, BMN, MODE>(nd, p, part, st);
    case 64: return conv_mode_nd<64, BMN, MODE>(nd, p, part, st);
    case 128: return conv_mode_nd<128, BMN, MODE>(nd, p, part, st);
    case 256: return conv_mode_nd<256, BMN, MODE>(nd, p, part, st);
  }
  return VP_EINTERNAL;
}

int conv_tc_tf32(int64_t kd, int64_t nd, const FwdParams& p, void* part, cudaStream_t st);      // conv_tc_tf32.cu
int conv_tc_pad_fwd(int64_t kd, int64_t nd, const FwdParams& p, void* part, cudaStream_t st);   // conv_tc_pad.cu
int conv_tc_pad_dgrad(int64_t kd, int64_t nd, const FwdParams& p, void* part, cudaStream_t st); // conv_tc_pad.cu

// one translation unit each (conv_tc_k<KD>_<f|d>.cu)
#define VP_CONV_TC_DECL(KD, T) int conv_tc_k##KD##_##T(int64_t nd, const FwdParams& p, void* part, cudaStream_t st);
VP_CONV_TC_DECL(32, f)
VP_CONV_TC_DECL(64, f)
VP_CONV_TC_DECL(128, f)
VP_CONV_TC_DECL(256, f)
VP_CONV_TC_DECL(32, d)
VP_CONV_TC_DECL(64, d)
VP_CONV_TC_DECL(128, d)
VP_CONV_TC_DECL(256, d)
#undef VP_CONV_TC_DECL

}  // namespace vp
