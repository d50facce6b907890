// iono_fourstep.cu -- fused FFT -> ionospheric phase -> IFFT kernels (Eq. 15).
//
// Regime 0 (n <= 8192): one CTA holds whole pulses; forward FFT, phase and inverse FFT
//   run back to back on registers + shared memory: one HBM read and one HBM write per
//   sample (16 B / sample).
// Regime 1 (n > 8192): four-step split n = N1 N2, t = N2 t1 + t2, k = k1 + N1 k2:
//   pass A  column DFTs over t1 (N1 points) for each t2, times w_n^(k1 t2)        -> Z[k1][t2]
//   pass B  row DFT over t2 (N2 points) -> bin k = k1 + N1 k2 -> phase (Eq. 15) ->
//           inverse row DFT over k2, times w_n^(-k1 t2)                             -> Z'[k1][t2]
//   pass C  inverse column DFTs over k1 -> y[N2 t1 + t2]
//   (n = 2^20: the conj outer twiddle of pass B is applied by pass C on load instead.)
//   Z and Z' live in the output buffer itself (in place); for dc_correct the output is the
//   plan-owned launch-group buffer (2 GiB groups), so each pass streams ~16 B / sample through HBM
//   (48 B / sample for the stage; ncu: profiles/r1b_ncu_full_summary.md).
// (this unit: the four-step passes of n >= 2^14: column passes, warp row pass, pass dispatch)
#include "iono_launch.cuh"

namespace dc {

template <int P1, int MODE>
static cudaError_t launch_col_p(const TileArgs &a, cudaStream_t st, int cap) {
  constexpr int C = col_c(P1);
  const int64_t total = a.pulses * ((1ll << (a.log2n - P1)) / C);
  return launch_tile_cfg<P1, DC_FS_LOGE, C, false, MODE, VAR_CORRECT>(a, total, st, cap);
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
  // warp row pass with a warp-level (n = 2^20) or thread-per-column (2^14 .. 2^16) pass C: the conj outer
  // twiddle moves from the compute-bound row pass to the memory-bound column pass (applied on load):
  // row pass 246 -> 267 GS/s at 2^20, 252 -> 272 at 2^16 (stage +1.2 % / +3 %)
  const bool outer_c = (P1 == 10 || P1 <= 6) && P2 == 10 && f.tw1024 && f.gtab;
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
      if (P2 == 10 && f.tw1024 && f.gtab) {
        WarpArgs w = warp_args(a, f.tw1024, f.gtab);
        w.outer_c = outer_c;
        return launch_warp_row<MODE_ROWB>(w, var, f.stream, f.grid_cap);
      }
      return launch_fourstep_row_tile(P2, a, var, f.stream, f.grid_cap);
    case 2:
      a.src = f.dst;
      a.dst = f.dst;
      a.twi = f.tw1i;
      if (P1 == 10 && f.tw1024) {
        WarpArgs w = warp_args(a, f.tw1024);
        w.outer_c = outer_c;
        return launch_warp_col(w, true, f.stream, f.grid_cap);
      }
      if (P1 <= 6) {
        WarpArgs w = warp_args(a, f.tw1024);
        w.outer_c = outer_c;
        return launch_tcol(w, P1, true, f.stream, f.grid_cap);
      }
      return launch_col<MODE_COLC>(P1, a, f.stream, f.grid_cap);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace dc
