// dc_kernels.h -- internal launch interface between the C-ABI layer and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dc_common.cuh"

namespace dc {

// cached launch preparation (launch_cache.cu): sets the kernel's dynamic shared-memory limit once and
// returns the SM count and resident CTAs per SM for (kernel, current device, block size, smem)
struct LaunchShape {
  int sms, per_sm;
};
cudaError_t launch_shape(const void *fn, int threads, size_t smem, LaunchShape *out);
template <class K>
inline cudaError_t launch_shape(K *fn, int threads, size_t smem, LaunchShape *out) {
  return launch_shape(reinterpret_cast<const void *>(fn), threads, smem, out);
}

constexpr int kMaxPasses = 8;

// radix sequence of one FFT size, as compiled into the kernels (for twiddle-table building)
struct PlanDesc {
  int npass = 0;
  int log_radix_fwd[kMaxPasses] = {};
  int log_radix_inv[kMaxPasses] = {};
  int log_ns_fwd[kMaxPasses] = {};
  int log_ns_inv[kMaxPasses] = {};
  int tw_off_fwd[kMaxPasses] = {};
  int tw_off_inv[kMaxPasses] = {};
  int tw_size = 0;
};

bool describe_small_plan(int P, PlanDesc &d);
bool describe_fourstep_plan(int P, PlanDesc &d);
void fourstep_split(int log2n, int &P1, int &P2);

struct IonoSmallArgs {
  const float2 *xin;
  float2 *xout;
  int64_t batch;
  int log2n;
  const PulseParams *pp;
  const float2 *twf, *twi;
  double fs_over_n, fc;
  cudaStream_t stream;
  const float2 *tw1024;  // 1024-point pass-2 table for the warp-level kernels (n = 1024), or null
  int grid_cap;          // max CTAs of the persistent grid (0: one wave of the whole GPU)
  const float2 *gtab;    // per-bin 1/f_k FP32 pairs for the warp-level kernel, or null
  const float2 *ref;     // var 2: T = conj(R) tables (natural bin order, n entries each), else null
  const int *ref_idx;    // var 2: per-pulse table index (pre-offset like pp), or null = table 0
  float2 *ref_out;       // var 3: conj spectrum output per pulse (natural order), else null
};
// var: 0 Eq. 15 correction, 1 Eq. 14 distortion, 2 correction + matched filter (T table `ref`),
// 3 forward spectra stored conjugated to `ref_out` (no inverse transform)
cudaError_t launch_iono_small(const IonoSmallArgs &a, int var);
// fused single-round-trip dc_correct (iono + first/second-order Doppler in one kernel, NEXT-1) for
// short pulses: n = 2^10 (warp-level FFT) and 2^11 .. 2^13 (tile FFT), W in {16, 32} (correct_small_supported)
bool correct_small_supported(int log2n, int W);
cudaError_t launch_correct_small(const IonoSmallArgs &a, float2 *y, double carrier, int W, bool second);

struct FourStepArgs {
  const float2 *src;  // pass A input (pulse-major, pulse_stride apart)
  float2 *dst;        // passes A/B/C output (may equal src)
  int64_t pulses;     // pulses in this launch group
  int64_t pulse_stride;
  int64_t pulse_base; // index of the first pulse in pp[]
  int log2n;
  const PulseParams *pp;
  const float2 *tw1f, *tw1i;  // N1-point pass tables
  const float2 *tw2f, *tw2i;  // N2-point pass tables
  const float2 *twh, *twl;    // outer twiddle two-level table
  int H;
  double fs_over_n, fc;
  cudaStream_t stream;
  const float2 *tw1024;       // 1024-point pass-2 table for the warp-level kernels, or null
  int grid_cap;               // max CTAs of the persistent grid (0: one wave of the whole GPU)
  const float2 *gtab;         // per-bin 1/f_k FP32 pairs (row layout) for the warp-level row kernel
  const float2 *ref;          // var 2: T = conj(R) tables in the row layout (k1 N2 + k2), n entries each
  const int *ref_idx;         // var 2: per-pulse table index (indexed like pp), or null = table 0
  float2 *ref_out;            // var 3: conj spectra per pulse (row layout), else null
};
// offset (float2 entries) of the NS = 32 section inside the P = 10, radix-32 forward pass table
int tw1024_offset();
// pass 0 = A (columns, forward), 1 = B (rows, phase), 2 = C (columns, inverse); var as launch_iono_small
// (var 3 runs passes A and B only)
cudaError_t launch_iono_fourstep_pass(const FourStepArgs &a, int pass, int var);

// Kaiser taper of the sinc window (reading R17): K(d) = P(q), q = kb^2/4 (1 - (d/L)^2), L = W/2,
// P(q) = sum_j q^j / ((j!)^2 I0(kb)) -- the I0 power series, normalised, truncated at kTaperTerms
constexpr int kTaperTerms = 25;
// Hann taper (reading R17): K(d) = (1 + cos(pi d / L)) / 2; selected by the taper code kTaperHann in place
// of a Kaiser series length
constexpr int kTaperHann = 1;
struct TaperCoef {
  float c[kTaperTerms];  // c[j] = 1 / ((j!)^2 I0(kb)), FP32 (from binary64)
  float qa;              // kb^2 / 4
  float inv_L2;          // 1 / L^2
  float pi_over_L;       // Hann: pi / L
};

struct DopplerArgs {
  const float2 *x;
  float2 *y;
  int64_t pulses;
  int64_t n;
  int taps;
  const PulseParams *pp;
  int64_t pulse_base;
  double carrier_cycles_per_sample;  // fc / fs; carrier phase psi_m = fc (1 - beta) m / fs
  cudaStream_t stream;
  int grid_cap;  // max CTAs of the persistent grid (0: one wave of the whole GPU)
  bool taper;       // taper on (coefficients in tc)
  TaperCoef tc;
  int taper_terms;  // Kaiser: series terms needed (17 or kTaperTerms); kTaperHann: the Hann window
  void *desc;       // plan-owned per-CTA tile-geometry slots (kDopDescBytes)
};
constexpr int kDopMaxCtas = 1024;                       // persistent Doppler grid cap
constexpr size_t kDopDescBytes = (size_t)kDopMaxCtas * 4 * 48;
cudaError_t launch_doppler(const DopplerArgs &a, double max_abs_beta_m1);
int doppler_path(double max_abs_beta_m1, bool taper = false, int W = 32);

// FFT P/Q resampling (pq_kernels.cu, reading R18).  Mv: per-pulse length M (device int[pulses]).
cudaError_t launch_pq_gather(const float2 *Xc, float2 *a, int64_t pulses, int log2n, int P1, const int *Mv,
                             cudaStream_t st);
cudaError_t launch_pq_chirp(float2 *r, int64_t n, int64_t M, cudaStream_t st);
cudaError_t launch_pq_post(const float2 *c, const float2 *x, float2 *y, int64_t pulses, int log2n, const int *Mv,
                           double fc, double fs, cudaStream_t st);

}  // namespace dc
