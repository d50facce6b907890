// iono_small.cu -- fused FFT -> ionospheric phase -> IFFT kernels (Eq. 15).
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
// (this unit: single-CTA pulses n <= 8192, the pass plans and the four-step split)
#include "iono_launch.cuh"

namespace dc {

#ifndef DC_WSMALL3
#define DC_WSMALL3 1  // n = 2^11 .. 2^13 on the in-CTA four-step kernels (0: the tile kernels, for A/B tuning builds)
#endif

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
static cudaError_t launch_wsmall3(const WarpArgs &a, int var, cudaStream_t st, int cap) {
  auto kern = (var == VAR_DISTORT) ? warp_small3_kernel<N1, VAR_DISTORT> : warp_small3_kernel<N1, VAR_CORRECT>;
  const size_t smem = wsmall3_smem_bytes(N1, 0);
  LaunchShape ls;
  cudaError_t e = launch_shape(kern, kWs3T, smem, &ls);
  if (e != cudaSuccess) return e;
  const int64_t tiles = (a.pulses + wsmall3_ppt(N1) - 1) / wsmall3_ppt(N1);
  int64_t grid = std::min<int64_t>(tiles, ls.sms);
  if (cap > 0) grid = std::min<int64_t>(grid, cap);
  return launch_pdl(kern, dim3((unsigned)grid), dim3(kWs3T), smem, st, a, (float2 *)nullptr, 0.0);
}

template <int Q>
static cudaError_t launch_wtiny(const WarpArgs &a, int var, cudaStream_t st, int cap) {
  auto kern = (var == VAR_DISTORT) ? warp_tiny_kernel<Q, VAR_DISTORT> : warp_tiny_kernel<Q, VAR_CORRECT>;
  const size_t smem = wtiny_smem_bytes(32 * Q);
  LaunchShape ls;
  cudaError_t e = launch_shape(kern, kTinyNW * 32, smem, &ls);
  if (e != cudaSuccess) return e;
  const int64_t items = (a.pulses + (32 / Q) - 1) / (32 / Q);
  int64_t grid = std::min<int64_t>((items + kTinyNW - 1) / kTinyNW, (int64_t)ls.sms * ls.per_sm);
  if (cap > 0) grid = std::min<int64_t>(grid, cap);
  return launch_pdl(kern, dim3((unsigned)grid), dim3(kTinyNW * 32), smem, st, a);
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
    return launch_warp_row<MODE_SMALL>(warp_args(a, s.tw1024, s.gtab), var, s.stream, s.grid_cap);
  // n = 128 .. 512: warp-level kernel (wtiny.cuh) for the correction / forward model
  if (s.log2n >= 7 && s.log2n <= 9 && s.gtab && (var == VAR_CORRECT || var == VAR_DISTORT)) {
    const WarpArgs w = warp_args(a, nullptr, s.gtab);
    if (s.log2n == 7) return launch_wtiny<4>(w, var, s.stream, s.grid_cap);
    if (s.log2n == 8) return launch_wtiny<8>(w, var, s.stream, s.grid_cap);
    return launch_wtiny<16>(w, var, s.stream, s.grid_cap);
  }
  // in-CTA four-step on the warp FFT (wsmall.cuh) for 2048 .. 8192 (two warp groups, three slots):
  // 158 / 156 / 169 GS/s vs 154 (tile kernel) / 135 / 137 (one 8-warp group, two buffers) measured.
  // Pulse compression and spectrum output (var 2, 3) run on the tile kernel (natural bin order).
  if (DC_WSMALL3 && s.log2n >= 11 && s.log2n <= 14 && s.tw1024 && s.gtab && (var == VAR_CORRECT || var == VAR_DISTORT)) {
    const WarpArgs w = warp_args(a, s.tw1024, s.gtab);
    if (s.log2n == 14) return launch_wsmall3<16>(w, var, s.stream, s.grid_cap);
    if (s.log2n == 11) return launch_wsmall3<2>(w, var, s.stream, s.grid_cap);
    return (s.log2n == 12) ? launch_wsmall3<4>(w, var, s.stream, s.grid_cap) : launch_wsmall3<8>(w, var, s.stream, s.grid_cap);
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

// ---- fused single-round-trip dc_correct for single-CTA pulses (NEXT-1): n = 2^11 .. 2^13, W in {16, 32}
template <int P, int W, bool SECOND>
static cudaError_t launch_correct_small_pw(const TileArgs &a, cudaStream_t st, int cap) {
  constexpr int NB = small_nb(P);
  constexpr int LOGE = small_loge<P>();
  using CFG = TileCfg<P, LOGE, NB, true, MODE_SMALL>;
  auto kern = tile_fft_kernel<P, LOGE, NB, true, MODE_SMALL, VAR_CORRECT, W, SECOND>;
  const size_t smem = CFG::smem_bytes(0, P, true);
  LaunchShape ls;
  cudaError_t e = launch_shape(kern, CFG::T, smem, &ls);
  if (e != cudaSuccess) return e;
  const int sms = ls.sms, per_sm = ls.per_sm;
  const int64_t total = (a.pulses + NB - 1) / NB;
  int64_t grid = std::min<int64_t>(total, (int64_t)sms * std::max(per_sm, 1));
  if (cap > 0) grid = std::min<int64_t>(grid, cap);
  return launch_pdl(kern, dim3((unsigned)grid), dim3(CFG::T), smem, st, a);
}
template <int P>
static cudaError_t launch_correct_small_p(const TileArgs &a, int W, bool second, cudaStream_t st, int cap) {
  if (W == 16) return second ? launch_correct_small_pw<P, 16, true>(a, st, cap) : launch_correct_small_pw<P, 16, false>(a, st, cap);
  if (W == 32) return second ? launch_correct_small_pw<P, 32, true>(a, st, cap) : launch_correct_small_pw<P, 32, false>(a, st, cap);
  return cudaErrorInvalidValue;
}

template <int W, bool SECOND>
static cudaError_t launch_correct1024_w(const WarpArgs &a, float2 *y, double carrier, cudaStream_t st, int cap) {
  auto kern = warp_correct1024_kernel<W, SECOND>;
  const size_t smem = wcorrect_smem_bytes<W>();
  LaunchShape ls;
  cudaError_t e = launch_shape(kern, kWcNW * 32, smem, &ls);
  if (e != cudaSuccess) return e;
  int64_t grid = std::min<int64_t>((a.pulses + kWcNW - 1) / kWcNW, (int64_t)ls.sms * ls.per_sm);
  if (cap > 0) grid = std::min<int64_t>(grid, cap);
  return launch_pdl(kern, dim3((unsigned)grid), dim3(kWcNW * 32), smem, st, a, y, carrier);
}

template <int N1, int W, bool SECOND>
static cudaError_t launch_wscorrect(const WarpArgs &a, float2 *y, double carrier, cudaStream_t st, int cap) {
  auto kern = warp_small3_kernel<N1, VAR_CORRECT, W, SECOND>;
  const size_t smem = wsmall3_smem_bytes(N1, W);
  LaunchShape ls;
  cudaError_t e = launch_shape(kern, kWs3T, smem, &ls);
  if (e != cudaSuccess) return e;
  const int64_t tiles = (a.pulses + wsmall3_ppt(N1) - 1) / wsmall3_ppt(N1);
  int64_t grid = std::min<int64_t>(tiles, ls.sms);
  if (cap > 0) grid = std::min<int64_t>(grid, cap);
  return launch_pdl(kern, dim3((unsigned)grid), dim3(kWs3T), smem, st, a, y, carrier);
}
template <int N1>
static cudaError_t launch_wscorrect_n(const WarpArgs &a, float2 *y, double carrier, int W, bool second, cudaStream_t st,
                                      int cap) {
  if (W == 16) return second ? launch_wscorrect<N1, 16, true>(a, y, carrier, st, cap) : launch_wscorrect<N1, 16, false>(a, y, carrier, st, cap);
  return second ? launch_wscorrect<N1, 32, true>(a, y, carrier, st, cap) : launch_wscorrect<N1, 32, false>(a, y, carrier, st, cap);
}

bool correct_small_supported(int log2n, int W) {
  return log2n >= 10 && log2n <= (DC_WSMALL3 ? 14 : 13) && (W == 16 || W == 32);
}

cudaError_t launch_correct_small(const IonoSmallArgs &s, float2 *y, double carrier, int W, bool second) {
  TileArgs a{};
  a.src = s.xin;
  a.dst = nullptr;
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
  a.dop_y = y;
  a.dop_carrier = carrier;
  if (s.log2n == 10) {  // warp-level FFT, one warp per pulse (wcorrect.cuh)
    if (!s.tw1024 || !s.gtab) return cudaErrorInvalidValue;
    const WarpArgs w = warp_args(a, s.tw1024, s.gtab);
    if (W == 16) return second ? launch_correct1024_w<16, true>(w, y, carrier, s.stream, s.grid_cap)
                               : launch_correct1024_w<16, false>(w, y, carrier, s.stream, s.grid_cap);
    return second ? launch_correct1024_w<32, true>(w, y, carrier, s.stream, s.grid_cap)
                  : launch_correct1024_w<32, false>(w, y, carrier, s.stream, s.grid_cap);
  }
  // n = 2^11 .. 2^13: the in-CTA four-step kernel with the Doppler stage on its slots (wsmall.cuh)
  if (DC_WSMALL3 && s.log2n >= 11 && s.log2n <= 14 && s.tw1024 && s.gtab) {
    const WarpArgs w = warp_args(a, s.tw1024, s.gtab);
    if (s.log2n == 14) return launch_wscorrect_n<16>(w, y, carrier, W, second, s.stream, s.grid_cap);
    if (s.log2n == 11) return launch_wscorrect_n<2>(w, y, carrier, W, second, s.stream, s.grid_cap);
    if (s.log2n == 12) return launch_wscorrect_n<4>(w, y, carrier, W, second, s.stream, s.grid_cap);
    return launch_wscorrect_n<8>(w, y, carrier, W, second, s.stream, s.grid_cap);
  }
  switch (s.log2n) {
    case 11: return launch_correct_small_p<11>(a, W, second, s.stream, s.grid_cap);
    case 12: return launch_correct_small_p<12>(a, W, second, s.stream, s.grid_cap);
    case 13: return launch_correct_small_p<13>(a, W, second, s.stream, s.grid_cap);
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

int tw1024_offset() { return kTw1024Off; }

}  // namespace dc
