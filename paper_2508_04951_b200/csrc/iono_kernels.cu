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
#include "fft_engine.cuh"

namespace dc {

// Eq. 15 multiplier of bin k (signed index kk = k - n [k >= n/2]), scaled by 1/n (reading R6):
//   f = fc + fs kk / n (R2); nu = nu_coef / f if f > 0 else 0 (R3); exp(-+ i 2 pi (nu - rint(nu))).
// nu is formed and range-reduced in binary64 (nu reaches ~1e3..1e11
// cycles, far beyond FP32), the rotation itself is FP32.
template <bool DISTORT>
__device__ __forceinline__ float2 iono_multiplier(int kk, double fs_over_n, double fc, double nu_coef, float scale) {
  double f = fc + fs_over_n * (double)kk;
  if (!(f > 0.0) || nu_coef == 0.0) return make_float2(scale, 0.f);
  double nu = nu_coef * drcp(f);
  double r = nu - rint(nu);
  float rf = __double2float_rn(r);
  float2 w = expm2pi(DISTORT ? -rf : rf);
  return make_float2(w.x * scale, w.y * scale);
}

// ============================================================================= regime 0
template <int P, int LOGE, bool DISTORT>
__global__ void __launch_bounds__(Tile<P, (1 << LOGE), (8192 >> P) < 1 ? 1 : (8192 >> P), true>::T)
    iono_small_kernel(const float2 *__restrict__ xin, float2 *__restrict__ xout, int64_t batch,
                      const PulseParams *__restrict__ pp, const float2 *__restrict__ twf,
                      const float2 *__restrict__ twi, double fs_over_n, double fc) {
  constexpr int L = 1 << P;
  constexpr int E = 1 << LOGE;
  constexpr int NB = (8192 >> P) < 1 ? 1 : (8192 >> P);
  using TL = Tile<P, E, NB, true>;
  using PP = PassPlan<P, LOGE>;
  constexpr int NP = PP::npass;
  constexpr int R0 = 1 << PP::log_radix_fwd(0);
  constexpr int RL = 1 << PP::log_radix_fwd(NP - 1);
  constexpr int RI = 1 << PP::log_radix_inv(NP - 1);
  extern __shared__ float4 smem4[];
  float2 *s = reinterpret_cast<float2 *>(smem4);
  const int tid = threadIdx.x;
  const int64_t pulse0 = (int64_t)blockIdx.x * NB;

  float2 v[E];
  // first forward pass inputs straight from HBM: butterfly j reads j + r L/R0 (coalesced)
#pragma unroll
  for (int q = 0; q < E / R0; ++q) {
    int b, j;
    TL::template bmap<R0>(tid + q * TL::T, b, j);
    const int64_t p = pulse0 + b;
    const float2 *src = xin + p * L;
#pragma unroll
    for (int r = 0; r < R0; ++r) v[q * R0 + r] = (p < batch) ? __ldcs(src + j + r * (L / R0)) : make_float2(0.f, 0.f);
  }
  run_passes<TL, PP, 0, NP - 1, false>(v, s, tid, twf);

  // frequency domain: registers hold bins k = j + r L/RL of pulse b
  const float inv_n = 1.0f / (float)L;
#pragma unroll
  for (int q = 0; q < E / RL; ++q) {
    int b, j;
    TL::template bmap<RL>(tid + q * TL::T, b, j);
    const int64_t p = pulse0 + b;
    const double nu_coef = (p < batch) ? pp[p].nu_coef : 0.0;
#pragma unroll
    for (int r = 0; r < RL; ++r) {
      int k = j + r * (L / RL);
      int kk = (k >= L / 2) ? k - L : k;
      v[q * RL + r] = cmul(v[q * RL + r], iono_multiplier<DISTORT>(kk, fs_over_n, fc, nu_coef, inv_n));
    }
  }

  run_passes<TL, PP, 0, NP - 1, true>(v, s, tid, twi);
  // last inverse pass outputs t = j + r L/RI of pulse b, straight to HBM
#pragma unroll
  for (int q = 0; q < E / RI; ++q) {
    int b, j;
    TL::template bmap<RI>(tid + q * TL::T, b, j);
    const int64_t p = pulse0 + b;
    if (p < batch) {
      float2 *dst = xout + p * L;
#pragma unroll
      for (int r = 0; r < RI; ++r) __stcs(dst + j + r * (L / RI), v[q * RI + r]);
    }
  }
}

// ============================================================================= regime 1
// outer twiddle w_n^(m) = exp(-2 pi i m / n) from a two-level table: m = mh 2^H + ml
__device__ __forceinline__ float2 outer_tw(uint32_t m, int H, const float2 *__restrict__ twh,
                                           const float2 *__restrict__ twl) {
  float2 a = __ldg(twh + (m >> H));
  float2 b = __ldg(twl + (m & ((1u << H) - 1u)));
  return cmul(a, b);
}

// pass A (INV = false): columns t2 of x, forward DFT over t1, times w_n^(k1 t2) -> Z[k1][t2]
// pass C (INV = true):  columns t2 of Z', inverse DFT over k1 -> y[N2 t1 + t2]
template <int P1, int C, bool INV>
__global__ void __launch_bounds__(Tile<P1, 32, C, false>::T)
    fourstep_col_kernel(const float2 *__restrict__ src, float2 *__restrict__ dst, int64_t pulse_stride,
                        int log2n, const float2 *__restrict__ tw, const float2 *__restrict__ twh,
                        const float2 *__restrict__ twl, int H) {
  constexpr int N1 = 1 << P1;
  constexpr int E = 32;
  using TL = Tile<P1, E, C, false>;
  using PP = PassPlan<P1, 5>;
  constexpr int NP = PP::npass;
  constexpr int R0 = 1 << (INV ? PP::log_radix_inv(0) : PP::log_radix_fwd(0));
  constexpr int RL = 1 << (INV ? PP::log_radix_inv(NP - 1) : PP::log_radix_fwd(NP - 1));
  extern __shared__ float4 smem4[];
  float2 *s = reinterpret_cast<float2 *>(smem4);
  const int tid = threadIdx.x;
  const int n2 = 1 << (log2n - P1);
  const int c0 = blockIdx.x * C;
  const int64_t pulse = blockIdx.y;
  const float2 *in = src + pulse * pulse_stride;
  float2 *out = dst + pulse * pulse_stride;

  float2 v[E];
#pragma unroll
  for (int q = 0; q < E / R0; ++q) {
    int b, j;
    TL::template bmap<R0>(tid + q * TL::T, b, j);
#pragma unroll
    for (int r = 0; r < R0; ++r) {
      const int row = j + r * (N1 / R0);
      const float2 *a = in + (int64_t)row * n2 + c0 + b;
      v[q * R0 + r] = INV ? __ldcg(a) : __ldcs(a);
    }
  }
  run_passes<TL, PP, 0, NP - 1, INV>(v, s, tid, tw);
  const uint32_t nmask = (1u << log2n) - 1u;
#pragma unroll
  for (int q = 0; q < E / RL; ++q) {
    int b, j;
    TL::template bmap<RL>(tid + q * TL::T, b, j);
    const uint32_t t2 = c0 + b;
#pragma unroll
    for (int r = 0; r < RL; ++r) {
      const uint32_t row = j + r * (N1 / RL);  // k1 (pass A) or t1 (pass C)
      float2 val = v[q * RL + r];
      float2 *a = out + (int64_t)row * n2 + t2;
      if constexpr (!INV) {
        val = cmul(val, outer_tw((row * t2) & nmask, H, twh, twl));
        __stcg(a, val);
      } else {
        __stcg(a, val);  // dc_correct reads it back from L2 (Doppler stage)
      }
    }
  }
}

// pass B: rows k1 of Z, forward DFT over t2 -> bins k1 + N1 k2 -> Eq. 15 phase / n ->
// inverse DFT over k2 -> times w_n^(-k1 t2) -> Z'
template <int P2, int NBR, bool DISTORT>
__global__ void __launch_bounds__(Tile<P2, 32, NBR, true>::T)
    fourstep_row_kernel(float2 *__restrict__ z, int64_t pulse_stride, int log2n,
                        const PulseParams *__restrict__ pp, int64_t pulse_base,
                        const float2 *__restrict__ twf, const float2 *__restrict__ twi,
                        const float2 *__restrict__ twh, const float2 *__restrict__ twl, int H,
                        double fs_over_n, double fc) {
  constexpr int N2 = 1 << P2;
  constexpr int E = 32;
  using TL = Tile<P2, E, NBR, true>;
  using PP = PassPlan<P2, 5>;
  constexpr int NP = PP::npass;
  constexpr int R0 = 1 << PP::log_radix_fwd(0);
  constexpr int RL = 1 << PP::log_radix_fwd(NP - 1);
  constexpr int RI = 1 << PP::log_radix_inv(NP - 1);
  extern __shared__ float4 smem4[];
  float2 *s = reinterpret_cast<float2 *>(smem4);
  const int tid = threadIdx.x;
  const int r0 = blockIdx.x * NBR;
  const int64_t pulse = blockIdx.y;
  float2 *zp = z + pulse * pulse_stride;
  const int P1 = log2n - P2;
  const int n = 1 << log2n;

  float2 v[E];
#pragma unroll
  for (int q = 0; q < E / R0; ++q) {
    int b, j;
    TL::template bmap<R0>(tid + q * TL::T, b, j);
    const float2 *a = zp + (int64_t)(r0 + b) * N2 + j;
#pragma unroll
    for (int r = 0; r < R0; ++r) v[q * R0 + r] = __ldcg(a + r * (N2 / R0));
  }
  run_passes<TL, PP, 0, NP - 1, false>(v, s, tid, twf);

  const double nu_coef = pp[pulse_base + pulse].nu_coef;
  const float inv_n = 1.0f / (float)n;
#pragma unroll
  for (int q = 0; q < E / RL; ++q) {
    int b, j;
    TL::template bmap<RL>(tid + q * TL::T, b, j);
    const int k1 = r0 + b;
#pragma unroll
    for (int r = 0; r < RL; ++r) {
      const int k2 = j + r * (N2 / RL);
      const int k = k1 + (k2 << P1);
      const int kk = (k >= n / 2) ? k - n : k;
      v[q * RL + r] = cmul(v[q * RL + r], iono_multiplier<DISTORT>(kk, fs_over_n, fc, nu_coef, inv_n));
    }
  }
  run_passes<TL, PP, 0, NP - 1, true>(v, s, tid, twi);
  const uint32_t nmask = (uint32_t)n - 1u;
#pragma unroll
  for (int q = 0; q < E / RI; ++q) {
    int b, j;
    TL::template bmap<RI>(tid + q * TL::T, b, j);
    const uint32_t k1 = r0 + b;
    float2 *a = zp + (int64_t)k1 * N2 + j;
#pragma unroll
    for (int r = 0; r < RI; ++r) {
      const uint32_t t2 = j + r * (N2 / RI);
      float2 val = cmulc(v[q * RI + r], outer_tw((k1 * t2) & nmask, H, twh, twl));
      __stcg(a + r * (N2 / RI), val);
    }
  }
}

// ============================================================================= launch helpers
template <int P>
static constexpr int small_loge() {
  // pick E in {16, 32} minimising the pass count (tie -> 16)
  return ((P + 4) / 5 < (P + 3) / 4) ? 5 : 4;
}

template <int P>
static cudaError_t launch_small_p(const IonoSmallArgs &a, bool distort) {
  constexpr int LOGE = small_loge<P>();
  constexpr int NB = (8192 >> P) < 1 ? 1 : (8192 >> P);
  using TL = Tile<P, (1 << LOGE), NB, true>;
  const size_t smem = sizeof(float2) * TL::SMEM_ELEMS;
  auto kern = distort ? iono_small_kernel<P, LOGE, true> : iono_small_kernel<P, LOGE, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t grid = (a.batch + NB - 1) / NB;
  kern<<<(unsigned)grid, TL::T, smem, a.stream>>>(a.xin, a.xout, a.batch, a.pp, a.twf, a.twi, a.fs_over_n, a.fc);
  return cudaGetLastError();
}

template <int P>
static int small_tw_entries() {
  return PassPlan<P, small_loge<P>()>::tw_size();
}

cudaError_t launch_iono_small(const IonoSmallArgs &a, bool distort) {
  switch (a.log2n) {
    case 1: return launch_small_p<1>(a, distort);
    case 2: return launch_small_p<2>(a, distort);
    case 3: return launch_small_p<3>(a, distort);
    case 4: return launch_small_p<4>(a, distort);
    case 5: return launch_small_p<5>(a, distort);
    case 6: return launch_small_p<6>(a, distort);
    case 7: return launch_small_p<7>(a, distort);
    case 8: return launch_small_p<8>(a, distort);
    case 9: return launch_small_p<9>(a, distort);
    case 10: return launch_small_p<10>(a, distort);
    case 11: return launch_small_p<11>(a, distort);
    case 12: return launch_small_p<12>(a, distort);
    case 13: return launch_small_p<13>(a, distort);
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
    case 7: fill_plan<7, 5>(d); return true;
    case 8: fill_plan<8, 5>(d); return true;
    case 9: fill_plan<9, 5>(d); return true;
    case 10: fill_plan<10, 5>(d); return true;
    case 11: fill_plan<11, 5>(d); return true;
    case 12: fill_plan<12, 5>(d); return true;
    case 13: fill_plan<13, 5>(d); return true;
    default: return false;
  }
}

// column-tile width C for N1 = 2^P1: tile of 8192 samples (64 KiB), at least 4 columns
static constexpr int col_c(int P1) { return (8192 >> P1) < 4 ? 4 : (8192 >> P1); }
static constexpr int row_nb(int P2) { return (8192 >> P2) < 1 ? 1 : (8192 >> P2); }

template <int P1, bool INV>
static cudaError_t launch_col_p(const FourStepArgs &a, const float2 *src, float2 *dst) {
  constexpr int C = col_c(P1);
  using TL = Tile<P1, 32, C, false>;
  const size_t smem = sizeof(float2) * TL::SMEM_ELEMS;
  auto kern = fourstep_col_kernel<P1, C, INV>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int n2 = 1 << (a.log2n - P1);
  dim3 grid(n2 / C, (unsigned)a.pulses);
  kern<<<grid, TL::T, smem, a.stream>>>(src, dst, a.pulse_stride, a.log2n, INV ? a.tw1i : a.tw1f, a.twh, a.twl, a.H);
  return cudaGetLastError();
}

template <int P2, bool DISTORT>
static cudaError_t launch_row_p(const FourStepArgs &a) {
  constexpr int NBR = row_nb(P2);
  using TL = Tile<P2, 32, NBR, true>;
  const size_t smem = sizeof(float2) * TL::SMEM_ELEMS;
  auto kern = fourstep_row_kernel<P2, NBR, DISTORT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int n1 = 1 << (a.log2n - P2);
  dim3 grid(n1 / NBR, (unsigned)a.pulses);
  kern<<<grid, TL::T, smem, a.stream>>>(a.dst, a.pulse_stride, a.log2n, a.pp, a.pulse_base, a.tw2f, a.tw2i, a.twh,
                                        a.twl, a.H, a.fs_over_n, a.fc);
  return cudaGetLastError();
}

template <bool INV>
static cudaError_t launch_col(int P1, const FourStepArgs &a, const float2 *src, float2 *dst) {
  switch (P1) {
    case 7: return launch_col_p<7, INV>(a, src, dst);
    case 8: return launch_col_p<8, INV>(a, src, dst);
    case 9: return launch_col_p<9, INV>(a, src, dst);
    case 10: return launch_col_p<10, INV>(a, src, dst);
    case 11: return launch_col_p<11, INV>(a, src, dst);
    default: return cudaErrorInvalidValue;
  }
}

template <bool DISTORT>
static cudaError_t launch_row(int P2, const FourStepArgs &a) {
  switch (P2) {
    case 7: return launch_row_p<7, DISTORT>(a);
    case 8: return launch_row_p<8, DISTORT>(a);
    case 9: return launch_row_p<9, DISTORT>(a);
    case 10: return launch_row_p<10, DISTORT>(a);
    case 11: return launch_row_p<11, DISTORT>(a);
    case 12: return launch_row_p<12, DISTORT>(a);
    case 13: return launch_row_p<13, DISTORT>(a);
    default: return cudaErrorInvalidValue;
  }
}

void fourstep_split(int log2n, int &P1, int &P2) {
  P2 = (log2n + 1) / 2;
  if (log2n - P2 > 11) P2 = log2n - 11;
  if (P2 > 13) P2 = 13;
  P1 = log2n - P2;
}

cudaError_t launch_iono_fourstep_pass(const FourStepArgs &a, int pass, bool distort) {
  int P1, P2;
  fourstep_split(a.log2n, P1, P2);
  switch (pass) {
    case 0: return launch_col<false>(P1, a, a.src, a.dst);
    case 1: return distort ? launch_row<true>(P2, a) : launch_row<false>(P2, a);
    case 2: return launch_col<true>(P1, a, a.dst, a.dst);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace dc
