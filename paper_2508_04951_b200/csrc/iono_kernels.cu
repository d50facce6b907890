// iono_kernels.cu -- fused FFT -> ionospheric phase -> IFFT kernels (Eq. 15).
//
// Regime 0 (n <= 8192): one CTA holds whole pulses; forward FFT, phase and inverse FFT
//   run back to back on registers + shared memory: one HBM read and one HBM write per
//   sample (16 B / sample).
// Regime 1 (n > 8192): four-step split n = N1 N2, t = N2 t1 + t2, k = k1 + N1 k2:
//   pass A  column DFTs over t1 (N1 points) for each t2, times w_n^(k1 t2)        -> Z[k1][t2]
//   pass B  row DFT over t2 (N2 points) -> bin k = k1 + N1 k2 -> phase (Eq. 15) ->
//           inverse row DFT over k2, times w_n^(-k1 t2)                             -> Z'[k1][t2]
//   pass C  inverse column DFTs over k1 -> y[N2 t1 + t2]
//   Z and Z' live in the output buffer itself (in place); for dc_correct the output is a
//   plan-owned chunk buffer sized to stay L2-resident, so HBM sees ~16 B / sample.
#include "dc_kernels.h"
#include "tile_fft.cuh"
#include "wfft.cuh"
#include "tcol.cuh"
#include "wsmall.cuh"
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
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, CFG::T, smem);
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
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, smem);
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
static cudaError_t launch_warp_row(const WarpArgs &a, bool small, int var, cudaStream_t st, int cap) {
  constexpr int NW = DC_ROW_NW;
  if (small) return launch_warp_row_mode<MODE_SMALL>(a, var, warp_row_smem(a.log2n, a.H, false), (a.pulses + NW - 1) / NW, st, cap);
  const int64_t total_w = a.pulses << (a.log2n - 10);
  return launch_warp_row_mode<MODE_ROWB>(a, var, warp_row_smem(a.log2n, a.H, true), (total_w + NW - 1) / NW, st, cap);
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
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)launch_smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, launch_smem);
  int64_t grid = std::min<int64_t>(total, (int64_t)sms * std::max(per_sm, 1));
  if (cap > 0) grid = std::min<int64_t>(grid, cap);
  return launch_pdl(kern, dim3((unsigned)grid), dim3(threads), launch_smem, st, a, smap);
}
template <int N1>
static cudaError_t launch_tcol_n(const WarpArgs &a, bool inv, cudaStream_t st, int cap) {
  auto kern = inv ? thread_col_kernel<N1, true> : thread_col_kernel<N1, false>;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTcolT, 0);
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

template <int P, int VAR>
static cudaError_t launch_small_pv(const TileArgs &a, cudaStream_t st, int cap) {
  constexpr int NB = small_nb(P);
  const int64_t total = (a.pulses + NB - 1) / NB;
  return launch_tile_cfg<P, small_loge<P>(), NB, true, MODE_SMALL, VAR>(a, total, st, cap);
}
template <int P>
static cudaError_t launch_small_p(const TileArgs &a, int var, cudaStream_t st, int cap) {
  switch (var) {
    case VAR_CORRECT: return launch_small_pv<P, VAR_CORRECT>(a, st, cap);
    case VAR_DISTORT: return launch_small_pv<P, VAR_DISTORT>(a, st, cap);
    case VAR_COMPRESS: return launch_small_pv<P, VAR_COMPRESS>(a, st, cap);
    case VAR_REFERENCE: return launch_small_pv<P, VAR_REFERENCE>(a, st, cap);
    default: return cudaErrorInvalidValue;
  }
}

template <int N1>
static cudaError_t launch_wsmall(const WarpArgs &a, int var, cudaStream_t st, int cap) {
  auto kern = (var == VAR_DISTORT) ? warp_small_kernel<N1, VAR_DISTORT> : warp_small_kernel<N1, VAR_CORRECT>;
  const size_t smem = wsmall_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (a.pulses + (8 / N1) - 1) / (8 / N1);
  int64_t grid = std::min<int64_t>(tiles, sms);
  if (cap > 0) grid = std::min<int64_t>(grid, cap);
  return launch_pdl(kern, dim3((unsigned)grid), dim3(kWsT), smem, st, a);
}

cudaError_t launch_iono_small(const IonoSmallArgs &s, int var) {
  TileArgs a{};
  a.src = s.xin;
  a.dst = s.xout;
  a.pulses = s.batch;
  a.pulse_stride = (int64_t)1 << s.log2n;
  a.pulse_base = 0;
  a.log2n = s.log2n;
  a.pp = s.pp;
  a.twf = s.twf;
  a.twi = s.twi;
  a.H = 0;
  a.fs_over_n = s.fs_over_n;
  a.fc = s.fc;
  a.ref = s.ref;
  a.ref_idx = s.ref_idx;
  a.ref_out = s.ref_out;
  if (s.log2n == 10 && s.tw1024 && s.gtab)
    return launch_warp_row(warp_args(a, s.tw1024, s.gtab), true, var, s.stream, s.grid_cap);
  // in-CTA four-step on the warp FFT (wsmall.cuh) for 4096 / 8192: +5 % / +18 % over the tile
  // kernel; for 2048 the tile kernel is faster (128 vs 148 GS/s measured) and stays.  Pulse
  // compression and spectrum output (var 2, 3) run on the tile kernel (natural bin order).
  if (s.log2n >= 12 && s.log2n <= 13 && s.tw1024 && s.gtab && (var == VAR_CORRECT || var == VAR_DISTORT)) {
    const WarpArgs w = warp_args(a, s.tw1024, s.gtab);
    return (s.log2n == 12) ? launch_wsmall<4>(w, var, s.stream, s.grid_cap) : launch_wsmall<8>(w, var, s.stream, s.grid_cap);
  }
  switch (s.log2n) {
    case 1: return launch_small_p<1>(a, var, s.stream, s.grid_cap);
    case 2: return launch_small_p<2>(a, var, s.stream, s.grid_cap);
    case 3: return launch_small_p<3>(a, var, s.stream, s.grid_cap);
    case 4: return launch_small_p<4>(a, var, s.stream, s.grid_cap);
    case 5: return launch_small_p<5>(a, var, s.stream, s.grid_cap);
    case 6: return launch_small_p<6>(a, var, s.stream, s.grid_cap);
    case 7: return launch_small_p<7>(a, var, s.stream, s.grid_cap);
    case 8: return launch_small_p<8>(a, var, s.stream, s.grid_cap);
    case 9: return launch_small_p<9>(a, var, s.stream, s.grid_cap);
    case 10: return launch_small_p<10>(a, var, s.stream, s.grid_cap);
    case 11: return launch_small_p<11>(a, var, s.stream, s.grid_cap);
    case 12: return launch_small_p<12>(a, var, s.stream, s.grid_cap);
    case 13: return launch_small_p<13>(a, var, s.stream, s.grid_cap);
    default: return cudaErrorInvalidValue;
  }
}

// Pass plans (radix sequences) exported to the host so it can build the twiddle tables.
template <int P, int LOGR>
static void fill_plan(PlanDesc &d) {
  using PP = PassPlan<P, LOGR>;
  d.npass = PP::npass;
  for (int i = 0; i < PP::npass; ++i) {
    d.log_radix_fwd[i] = PP::log_radix_fwd(i);
    d.log_radix_inv[i] = PP::log_radix_inv(i);
    d.log_ns_fwd[i] = PP::log_ns_fwd(i);
    d.log_ns_inv[i] = PP::log_ns_inv(i);
    d.tw_off_fwd[i] = PP::tw_off_fwd(i);
    d.tw_off_inv[i] = PP::tw_off_inv(i);
  }
  d.tw_size = PP::tw_size();
}

template <int P>
static void fill_small(PlanDesc &d) { fill_plan<P, small_loge<P>()>(d); }

bool describe_small_plan(int P, PlanDesc &d) {
  switch (P) {
    case 1: fill_small<1>(d); return true;
    case 2: fill_small<2>(d); return true;
    case 3: fill_small<3>(d); return true;
    case 4: fill_small<4>(d); return true;
    case 5: fill_small<5>(d); return true;
    case 6: fill_small<6>(d); return true;
    case 7: fill_small<7>(d); return true;
    case 8: fill_small<8>(d); return true;
    case 9: fill_small<9>(d); return true;
    case 10: fill_small<10>(d); return true;
    case 11: fill_small<11>(d); return true;
    case 12: fill_small<12>(d); return true;
    case 13: fill_small<13>(d); return true;
    default: return false;
  }
}

bool describe_fourstep_plan(int P, PlanDesc &d) {
  switch (P) {
    case 7: fill_plan<7, DC_FS_LOGE>(d); return true;
    case 8: fill_plan<8, DC_FS_LOGE>(d); return true;
    case 9: fill_plan<9, DC_FS_LOGE>(d); return true;
    case 10: fill_plan<10, DC_FS_LOGE>(d); return true;
    case 11: fill_plan<11, DC_FS_LOGE>(d); return true;
    case 12: fill_plan<12, DC_FS_LOGE>(d); return true;
    case 13: fill_plan<13, DC_FS_LOGE>(d); return true;
    default: return false;
  }
}

void fourstep_split(int log2n, int &P1, int &P2) {
  if (log2n == 22 || log2n == 23) {  // warp column passes (N1 = 1024) + tile row pass (N2 = 2^12, 2^13):
    P1 = 10;                         // 63 vs 47 GS/s at 2^22 over the tile-only split
    P2 = log2n - 10;
    return;
  }
  // row pass on the warp-level 1024-point FFT; 2^14 .. 2^16: columns of N1 = 16 .. 64 on the
  // thread-per-column kernel (tcol.cuh)
  if (log2n >= 14 && log2n <= 21) {
    P2 = 10;
    P1 = log2n - 10;
    return;
  }
  P2 = (log2n + 1) / 2;
  if (log2n - P2 > 11) P2 = log2n - 11;
  if (P2 > 13) P2 = 13;
  P1 = log2n - P2;
}



template <int P1, int MODE>
static cudaError_t launch_col_p(const TileArgs &a, cudaStream_t st, int cap) {
  constexpr int C = col_c(P1);
  const int64_t total = a.pulses * ((1ll << (a.log2n - P1)) / C);
  return launch_tile_cfg<P1, DC_FS_LOGE, C, false, MODE, VAR_CORRECT>(a, total, st, cap);
}

template <int P2, int VAR>
static cudaError_t launch_row_pv(const TileArgs &a, cudaStream_t st, int cap) {
  constexpr int NB = row_nb(P2);
  const int64_t total = a.pulses * ((1ll << (a.log2n - P2)) / NB);
  return launch_tile_cfg<P2, DC_FS_LOGE, NB, true, MODE_ROWB, VAR>(a, total, st, cap);
}
template <int P2>
static cudaError_t launch_row_p(const TileArgs &a, int var, cudaStream_t st, int cap) {
  switch (var) {
    case VAR_CORRECT: return launch_row_pv<P2, VAR_CORRECT>(a, st, cap);
    case VAR_DISTORT: return launch_row_pv<P2, VAR_DISTORT>(a, st, cap);
    case VAR_COMPRESS: return launch_row_pv<P2, VAR_COMPRESS>(a, st, cap);
    case VAR_REFERENCE: return launch_row_pv<P2, VAR_REFERENCE>(a, st, cap);
    default: return cudaErrorInvalidValue;
  }
}

template <int MODE>
static cudaError_t launch_col(int P1, const TileArgs &a, cudaStream_t st, int cap) {
  switch (P1) {
    case 7: return launch_col_p<7, MODE>(a, st, cap);
    case 8: return launch_col_p<8, MODE>(a, st, cap);
    case 9: return launch_col_p<9, MODE>(a, st, cap);
    case 10: return launch_col_p<10, MODE>(a, st, cap);
    case 11: return launch_col_p<11, MODE>(a, st, cap);
    default: return cudaErrorInvalidValue;
  }
}

static cudaError_t launch_row(int P2, const TileArgs &a, int var, cudaStream_t st, int cap) {
  switch (P2) {
    case 7: return launch_row_p<7>(a, var, st, cap);
    case 8: return launch_row_p<8>(a, var, st, cap);
    case 9: return launch_row_p<9>(a, var, st, cap);
    case 10: return launch_row_p<10>(a, var, st, cap);
    case 11: return launch_row_p<11>(a, var, st, cap);
    case 12: return launch_row_p<12>(a, var, st, cap);
    case 13: return launch_row_p<13>(a, var, st, cap);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_iono_fourstep_pass(const FourStepArgs &f, int pass, int var) {
  int P1, P2;
  fourstep_split(f.log2n, P1, P2);
  TileArgs a{};
  a.pulses = f.pulses;
  a.pulse_stride = f.pulse_stride;
  a.pulse_base = f.pulse_base;
  a.log2n = f.log2n;
  a.pp = f.pp;
  a.twh = f.twh;
  a.twl = f.twl;
  a.H = f.H;
  a.fs_over_n = f.fs_over_n;
  a.fc = f.fc;
  a.ref = f.ref;
  a.ref_idx = f.ref_idx;
  a.ref_out = f.ref_out;
  switch (pass) {
    case 0:
      a.src = f.src;
      a.dst = f.dst;
      a.twf = f.tw1f;
      if (P1 == 10 && f.tw1024) return launch_warp_col(warp_args(a, f.tw1024), false, f.stream, f.grid_cap);
      if (P1 <= 6) return launch_tcol(warp_args(a, f.tw1024), P1, false, f.stream, f.grid_cap);
      return launch_col<MODE_COLA>(P1, a, f.stream, f.grid_cap);
    case 1:
      a.src = f.dst;
      a.dst = f.dst;
      a.twf = f.tw2f;
      a.twi = f.tw2i;
      if (P2 == 10 && f.tw1024 && f.gtab)
        return launch_warp_row(warp_args(a, f.tw1024, f.gtab), false, var, f.stream, f.grid_cap);
      return launch_row(P2, a, var, f.stream, f.grid_cap);
    case 2:
      a.src = f.dst;
      a.dst = f.dst;
      a.twi = f.tw1i;
      if (P1 == 10 && f.tw1024) return launch_warp_col(warp_args(a, f.tw1024), true, f.stream, f.grid_cap);
      if (P1 <= 6) return launch_tcol(warp_args(a, f.tw1024), P1, true, f.stream, f.grid_cap);
      return launch_col<MODE_COLC>(P1, a, f.stream, f.grid_cap);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace dc

namespace dc {
int tw1024_offset() { return kTw1024Off; }
}  // namespace dc
