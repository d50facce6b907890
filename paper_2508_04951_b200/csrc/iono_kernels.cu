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

template <int P, int LOGE, int NB, bool ROW, int MODE, bool DISTORT>
static cudaError_t launch_tile_cfg(const TileArgs &a, int64_t total, cudaStream_t st) {
  using CFG = TileCfg<P, LOGE, NB, ROW, MODE>;
  auto kern = tile_fft_kernel<P, LOGE, NB, ROW, MODE, DISTORT>;
  const size_t smem = CFG::smem_bytes(a.H, a.log2n);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, CFG::T, smem);
  const int64_t grid = std::min<int64_t>(total, (int64_t)sms * std::max(per_sm, 1));
  kern<<<(unsigned)grid, CFG::T, smem, st>>>(a);
  return cudaGetLastError();
}

template <int P>
static cudaError_t launch_small_p(const TileArgs &a, bool distort, cudaStream_t st) {
  constexpr int NB = small_nb(P);
  const int64_t total = (a.pulses + NB - 1) / NB;
  return distort ? launch_tile_cfg<P, small_loge<P>(), NB, true, MODE_SMALL, true>(a, total, st)
                 : launch_tile_cfg<P, small_loge<P>(), NB, true, MODE_SMALL, false>(a, total, st);
}

cudaError_t launch_iono_small(const IonoSmallArgs &s, bool distort) {
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
  switch (s.log2n) {
    case 1: return launch_small_p<1>(a, distort, s.stream);
    case 2: return launch_small_p<2>(a, distort, s.stream);
    case 3: return launch_small_p<3>(a, distort, s.stream);
    case 4: return launch_small_p<4>(a, distort, s.stream);
    case 5: return launch_small_p<5>(a, distort, s.stream);
    case 6: return launch_small_p<6>(a, distort, s.stream);
    case 7: return launch_small_p<7>(a, distort, s.stream);
    case 8: return launch_small_p<8>(a, distort, s.stream);
    case 9: return launch_small_p<9>(a, distort, s.stream);
    case 10: return launch_small_p<10>(a, distort, s.stream);
    case 11: return launch_small_p<11>(a, distort, s.stream);
    case 12: return launch_small_p<12>(a, distort, s.stream);
    case 13: return launch_small_p<13>(a, distort, s.stream);
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
  P2 = (log2n + 1) / 2;
  if (log2n - P2 > 11) P2 = log2n - 11;
  if (P2 > 13) P2 = 13;
  P1 = log2n - P2;
}

template <int P1, int MODE>
static cudaError_t launch_col_p(const TileArgs &a, cudaStream_t st) {
  constexpr int C = col_c(P1);
  const int64_t total = a.pulses * ((1ll << (a.log2n - P1)) / C);
  return launch_tile_cfg<P1, DC_FS_LOGE, C, false, MODE, false>(a, total, st);
}

template <int P2, bool DISTORT>
static cudaError_t launch_row_p(const TileArgs &a, cudaStream_t st) {
  constexpr int NB = row_nb(P2);
  const int64_t total = a.pulses * ((1ll << (a.log2n - P2)) / NB);
  return launch_tile_cfg<P2, DC_FS_LOGE, NB, true, MODE_ROWB, DISTORT>(a, total, st);
}

template <int MODE>
static cudaError_t launch_col(int P1, const TileArgs &a, cudaStream_t st) {
  switch (P1) {
    case 7: return launch_col_p<7, MODE>(a, st);
    case 8: return launch_col_p<8, MODE>(a, st);
    case 9: return launch_col_p<9, MODE>(a, st);
    case 10: return launch_col_p<10, MODE>(a, st);
    case 11: return launch_col_p<11, MODE>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

template <bool DISTORT>
static cudaError_t launch_row(int P2, const TileArgs &a, cudaStream_t st) {
  switch (P2) {
    case 7: return launch_row_p<7, DISTORT>(a, st);
    case 8: return launch_row_p<8, DISTORT>(a, st);
    case 9: return launch_row_p<9, DISTORT>(a, st);
    case 10: return launch_row_p<10, DISTORT>(a, st);
    case 11: return launch_row_p<11, DISTORT>(a, st);
    case 12: return launch_row_p<12, DISTORT>(a, st);
    case 13: return launch_row_p<13, DISTORT>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_iono_fourstep_pass(const FourStepArgs &f, int pass, bool distort) {
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
  switch (pass) {
    case 0:
      a.src = f.src;
      a.dst = f.dst;
      a.twf = f.tw1f;
      return launch_col<MODE_COLA>(P1, a, f.stream);
    case 1:
      a.src = f.dst;
      a.dst = f.dst;
      a.twf = f.tw2f;
      a.twi = f.tw2i;
      return distort ? launch_row<true>(P2, a, f.stream) : launch_row<false>(P2, a, f.stream);
    case 2:
      a.src = f.dst;
      a.dst = f.dst;
      a.twi = f.tw1i;
      return launch_col<MODE_COLC>(P1, a, f.stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace dc
