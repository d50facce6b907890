// iono_launch.cuh -- launch helpers shared by the ionospheric-stage translation units (iono_small.cu,
// iono_fourstep.cu, iono_rows.cu; split so the kernel instantiations compile in parallel).
#pragma once
#include "dc_kernels.h"
#include "tile_fft.cuh"
#include "wfft.cuh"
#include "tcol.cuh"
#include "wsmall.cuh"
#include "wtiny.cuh"
#include "wcorrect.cuh"
#include "tma_host.h"

#include <algorithm>

#ifndef DC_FS_LOGE
#define DC_FS_LOGE 5  // samples per thread (log2) in the four-step tile kernels
#endif

namespace dc {

template <int P>
static constexpr int small_loge() {
  // pick E in {16, 32} minimising the pass count (tie -> 16)
  return ((P + 4) / 5 < (P + 3) / 4) ? 5 : 4;
}
static constexpr int small_nb(int P) { return (8192 >> P) < 1 ? 1 : (8192 >> P); }
// column-tile width for N1 = 2^P1 (8192-sample tiles, >= 4 columns = 32-byte row segments)
static constexpr int col_c(int P1) { return (8192 >> P1) < 4 ? 4 : (8192 >> P1); }
static constexpr int row_nb(int P2) { return (8192 >> P2) < 1 ? 1 : (8192 >> P2); }

template <int P, int LOGE, int NB, bool ROW, int MODE, int VAR>
static cudaError_t launch_tile_cfg(const TileArgs &a, int64_t total, cudaStream_t st, int cap) {
  using CFG = TileCfg<P, LOGE, NB, ROW, MODE>;
  auto kern = tile_fft_kernel<P, LOGE, NB, ROW, MODE, VAR>;
  const size_t smem = CFG::smem_bytes(a.H, a.log2n);
  LaunchShape ls;
  cudaError_t e = launch_shape(kern, CFG::T, smem, &ls);
  if (e != cudaSuccess) return e;
  const int sms = ls.sms, per_sm = ls.per_sm;
  int64_t grid = std::min<int64_t>(total, (int64_t)sms * std::max(per_sm, 1));
  if (cap > 0) grid = std::min<int64_t>(grid, cap);
  return launch_pdl(kern, dim3((unsigned)grid), dim3(CFG::T), smem, st, a);
}

// ---- warp-level 1024-point kernels (wfft.cuh)
constexpr bool kRowStage = (DC_ROW_NW <= 12);
static size_t warp_row_smem(int log2n, int H, bool outer) {
  return RowCfg<DC_ROW_NW, kRowStage>::elems(outer, log2n, H) * sizeof(float2);
}
template <class K>
static cudaError_t launch_persistent(K kern, size_t smem, int64_t total, const WarpArgs &a, cudaStream_t st, int cap,
                                     int nw = kWW) {
  LaunchShape ls;
  cudaError_t e = launch_shape(kern, nw * 32, smem, &ls);
  if (e != cudaSuccess) return e;
  const int sms = ls.sms, per_sm = ls.per_sm;
  int64_t grid = std::min<int64_t>(total, (int64_t)sms * std::max(per_sm, 1));
  if (cap > 0) grid = std::min<int64_t>(grid, cap);
  return launch_pdl(kern, dim3((unsigned)grid), dim3(nw * 32), smem, st, a);
}
template <int MODE>
static cudaError_t launch_warp_row_mode(const WarpArgs &a, int var, size_t smem, int64_t items, cudaStream_t st, int cap) {
  constexpr int NW = DC_ROW_NW;
  switch (var) {
    case VAR_CORRECT: return launch_persistent(warp_row_kernel<MODE, VAR_CORRECT, NW, kRowStage>, smem, items, a, st, cap, NW);
    case VAR_DISTORT: return launch_persistent(warp_row_kernel<MODE, VAR_DISTORT, NW, kRowStage>, smem, items, a, st, cap, NW);
    case VAR_COMPRESS: return launch_persistent(warp_row_kernel<MODE, VAR_COMPRESS, NW, kRowStage>, smem, items, a, st, cap, NW);
    case VAR_REFERENCE: return launch_persistent(warp_row_kernel<MODE, VAR_REFERENCE, NW, kRowStage>, smem, items, a, st, cap, NW);
    default: return cudaErrorInvalidValue;
  }
}
// whole 1024-sample pulses (MODE_SMALL) or the rows of four-step pass B (MODE_ROWB)
template <int MODE>
static cudaError_t launch_warp_row(const WarpArgs &a, int var, cudaStream_t st, int cap) {
  constexpr int NW = DC_ROW_NW;
  if constexpr (MODE == MODE_SMALL) {
    return launch_warp_row_mode<MODE_SMALL>(a, var, warp_row_smem(a.log2n, a.H, false), (a.pulses + NW - 1) / NW, st, cap);
  } else {
    const int64_t total_w = a.pulses << (a.log2n - 10);
    return launch_warp_row_mode<MODE_ROWB>(a, var, warp_row_smem(a.log2n, a.H, true), (total_w + NW - 1) / NW, st, cap);
  }
}
static cudaError_t launch_warp_col(const WarpArgs &a, bool inv, cudaStream_t st, int cap) {
  const int64_t total = a.pulses * ((1ll << (a.log2n - 10)) / kWW);
  // source tensor {t2, t1, pulse} of 8-byte samples, box {8 columns, 256 rows, 1}, 64-byte swizzle
  CUtensorMap smap;
  const int n2 = 1 << (a.log2n - 10);
  const uint64_t dims[3] = {(uint64_t)n2, 1024, (uint64_t)a.pulses};
  const uint64_t strides[2] = {(uint64_t)n2 * sizeof(float2), (uint64_t)a.pulse_stride * sizeof(float2)};
  const uint32_t box[3] = {(uint32_t)kWW, 256, 1};
  if (!encode_tile_map(&smap, a.src, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B)) return cudaErrorInvalidValue;
  const size_t launch_smem = warp_col3_smem_bytes();
  auto kern = inv ? warp_col3_kernel<true> : warp_col3_kernel<false>;
  constexpr int threads = 2 * kWW * 32;
  LaunchShape ls;
  cudaError_t e = launch_shape(kern, threads, launch_smem, &ls);
  if (e != cudaSuccess) return e;
  const int sms = ls.sms, per_sm = ls.per_sm;
  int64_t grid = std::min<int64_t>(total, (int64_t)sms * std::max(per_sm, 1));
  if (cap > 0) grid = std::min<int64_t>(grid, cap);
  return launch_pdl(kern, dim3((unsigned)grid), dim3(threads), launch_smem, st, a, smap);
}
template <int N1>
static cudaError_t launch_tcol_n(const WarpArgs &a, bool inv, cudaStream_t st, int cap) {
  auto kern = inv ? thread_col_kernel<N1, true> : thread_col_kernel<N1, false>;
  LaunchShape ls;
  cudaError_t e = launch_shape(kern, kTcolT, 0, &ls);
  if (e != cudaSuccess) return e;
  const int sms = ls.sms, per_sm = ls.per_sm;
  const int64_t items = a.pulses * (1024 / 32);  // warp items
  int64_t grid = std::min<int64_t>((items + kTcolT / 32 - 1) / (kTcolT / 32), (int64_t)sms * std::max(per_sm, 1));
  if (cap > 0) grid = std::min<int64_t>(grid, cap);
  return launch_pdl(kern, dim3((unsigned)grid), dim3(kTcolT), 0, st, a);
}
static cudaError_t launch_tcol(const WarpArgs &a, int P1, bool inv, cudaStream_t st, int cap) {
  switch (P1) {
    case 4: return launch_tcol_n<16>(a, inv, st, cap);
    case 5: return launch_tcol_n<32>(a, inv, st, cap);
    case 6: return launch_tcol_n<64>(a, inv, st, cap);
    default: return cudaErrorInvalidValue;
  }
}

static WarpArgs warp_args(const TileArgs &t, const float2 *tw1024, const float2 *gtab = nullptr) {
  WarpArgs w{};
  w.src = t.src;
  w.dst = t.dst;
  w.pulses = t.pulses;
  w.pulse_stride = t.pulse_stride;
  w.pulse_base = t.pulse_base;
  w.log2n = t.log2n;
  w.pp = t.pp;
  w.tw = tw1024;
  w.twh = t.twh;
  w.twl = t.twl;
  w.H = t.H;
  w.fs_over_n = t.fs_over_n;
  w.fc = t.fc;
  w.scale = 1.0f / (float)(1 << t.log2n);
  w.gtab = gtab;
  w.ref = t.ref;
  w.ref_idx = t.ref_idx;
  w.ref_out = t.ref_out;
  return w;
}
// pass-2 section (NS = 32, R = 32) of the P = 10, E = 32 forward table: float4 [r/2][k] layout
static constexpr int kTw1024Off = PassPlan<10, 5>::tw_off_fwd(1);

// four-step pass B on the tile kernel (N2 != 1024), iono_rows.cu
cudaError_t launch_fourstep_row_tile(int P2, const TileArgs &a, int var, cudaStream_t st, int cap);

}  // namespace dc
