// doppler_kernel.cu -- windowed Whittaker-Shannon (sinc) resampling onto t/alpha.
//
// Method (Eq. 16, restricted to W samples: Alg. 1 P:L510-528,
// window P:L533; correction direction per Eq. 13):
//   t_m = m beta (beta = 1/alpha, binary64)
//   y_m = exp(-i 2 pi fc (1 - beta) m / fs) * sum_{k = K_m}^{K_m + W - 1} [0 <= k < n] x_k sinc(t_m - k),
//   K_m = floor(t_m - W/2) + 1   (window {k : -W/2 < k - t_m <= W/2}, R9)
//
// B200 design:
//   * A CTA owns M = T*R consecutive outputs of one pulse; the input span they need
//     (~M*beta + W + 2 samples) is staged once into shared memory (zero-filled outside
//     [0, n)), with one pad slot per 8 samples so that lanes whose windows start ~8 samples
//     apart hit distinct banks.
//   * A thread owns R consecutive outputs.  Their windows slide by one sample per output
//     except where the fractional position wraps; all R windows lie inside a union of W+1
//     taps [B, B + W] relative to a per-output base B + r, so the thread streams the union
//     once through a register window (one LDS per tap, reused by all R outputs) and masks
//     the single edge tap each output does not own.
//   * Taps are evaluated on the fly in FP32 (no LUT; LUT quantisation breaks 1e-5 parity):
//     per thread, per tap, w = sinc(v - jj) and w' = sinc'(v - jj) at the thread's reference
//     position v (exact binary64 position, reduced to [-1/2, 1/2] before the FP32 cast so
//     the centre tap keeps full relative precision); each output then uses
//     h = w + w' delta_r (+ w''/2 delta_r^2), delta_r = (r - r_ref)(beta - 1) exactly.
//     With |delta| <= 2e-3 the truncation error is < 2e-9 (second order), far inside 1e-5.
//   * The slow path (|beta - 1| too large for the union/Taylor scheme) evaluates every
//     output directly (Alg. 1 structure).
#include "dc_kernels.h"

namespace dc {

constexpr int kDopT = 256;  // threads per CTA
constexpr int kDopR = 8;    // outputs per thread
constexpr int kDopM = kDopT * kDopR;
constexpr double kDopMaxDrift = 2.0e-3;  // max |beta - 1| * (R - 1) / 2 for the fast path

__device__ __forceinline__ int dpad(int i) { return i + (i >> 3); }

__device__ __forceinline__ float frcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// sinc weight and first/second derivative at d = u - m (u in [-1/2, 1/2] FP32, m integer):
// sin(pi d) = (-1)^m sin(pi u), cos(pi d) = (-1)^m cos(pi u).
struct TapW {
  float w, w1, w2;
};

__device__ __forceinline__ TapW tap_weight(float u, int m, float S, float Cc, bool second) {
  // S = sin(pi u) / pi, Cc = cos(pi u)
  TapW t;
  const float d = u - (float)m;
  const float sg = (m & 1) ? -1.f : 1.f;
  if (m == 0 && fabsf(u) < 0.25f) {
    // centre tap near d = 0: series (sinc is even; avoid C/d - S/(pi d^2) cancellation)
    const float pd2 = 9.8696044010893586f * u * u;  // (pi u)^2
    if (u == 0.f) {
      t.w = 1.f;
    } else {
      t.w = S * frcp(u);
    }
    // sinc'(d) = -(pi^2 d / 3) (1 - (pi d)^2 / 10 + (pi d)^4 / 280)
    t.w1 = -3.2898681336964529f * u * (1.f - pd2 * (0.1f - pd2 * (1.f / 280.f)));
    // sinc''(d) = -(pi^2 / 3)(1 - 3 (pi d)^2 / 10 + (pi d)^4 / 56)
    t.w2 = -3.2898681336964529f * (1.f - pd2 * (0.3f - pd2 * (1.f / 56.f)));
    return t;
  }
  const float inv = frcp(d);
  const float s = sg * S;   // sin(pi d) / pi
  const float c = sg * Cc;  // cos(pi d)
  t.w = s * inv;                          // sin(pi d)/(pi d)
  t.w1 = inv * fmaf(-s, inv, c);          // cos(pi d)/d - sin(pi d)/(pi d^2)
  if (second) {
    // sinc''(d) = -pi^2 sinc(d) - 2 sinc'(d) / d
    t.w2 = fmaf(-9.8696044010893586f, t.w, -2.f * t.w1 * inv);
  } else {
    t.w2 = 0.f;
  }
  return t;
}

template <bool SECOND>
__global__ void __launch_bounds__(kDopT) doppler_fast_kernel(const float2 *__restrict__ x, float2 *__restrict__ y,
                                                            int64_t n, int W, const PulseParams *__restrict__ pp,
                                                            int64_t pulse_base, double carrier) {
  extern __shared__ float2 xs[];
  const int tid = threadIdx.x;
  const int64_t pulse = blockIdx.y;
  const float2 *xp = x + pulse * n;
  float2 *yp = y + pulse * n;
  const double beta = pp[pulse_base + pulse].beta;
  const double halfW = 0.5 * (double)W;
  const int64_t m0 = (int64_t)blockIdx.x * kDopM;
  if (m0 >= n) return;
  // union base of output r of a thread whose first output is mt: B + r with
  // B = K(mt) - 1 if beta < 1 (a window may start one sample early), else K(mt).
  const int lo_shift = (beta < 1.0) ? 1 : 0;
  const double tc0 = (double)m0 * beta;
  const int64_t Bcta = (int64_t)floor(tc0 - halfW) + 1 - lo_shift;
  const int64_t mlast = min(m0 + kDopM, n) - 1;
  const int64_t Kend = (int64_t)floor((double)mlast * beta - halfW) + 1 + W + 1;  // exclusive, with slack
  const int span = (int)(Kend - Bcta);

  // ---- stage the input span (zero outside [0, n)) into padded shared memory
  for (int i = tid; i < span; i += kDopT) {
    const int64_t k = Bcta + i;
    xs[dpad(i)] = (k >= 0 && k < n) ? __ldcs(xp + k) : make_float2(0.f, 0.f);
  }
  __syncthreads();

  const int64_t mt = m0 + (int64_t)tid * kDopR;
  if (mt >= n) return;
  const int nout = (int)min((int64_t)kDopR, n - mt);

  // ---- exact binary64 window bookkeeping per output
  const double t0 = (double)mt * beta;
  const int64_t B = (int64_t)floor(t0 - halfW) + 1 - lo_shift;
  float mask0[kDopR], maskW[kDopR], delta[kDopR];
  constexpr int rref = kDopR / 2;
  const double tref = (double)(mt + rref) * beta;
  const double vref = tref - (double)(B + rref);  // continuous position inside the union (~W/2)
#pragma unroll
  for (int r = 0; r < kDopR; ++r) {
    const double tr = (double)(mt + r) * beta;
    const int64_t Kr = (int64_t)floor(tr - halfW) + 1;
    const int a = (int)(Kr - r - B);  // 0 or 1: offset of this output's window inside the union
    mask0[r] = (a == 0) ? 1.f : 0.f;
    maskW[r] = (a == 1) ? 1.f : 0.f;
    delta[r] = __double2float_rn((tr - (double)(B + r)) - vref);
  }
  // reference position split into nearest integer + fraction in [-1/2, 1/2]
  const double ic_d = rint(vref);
  const int ic = (int)ic_d;
  const float u = __double2float_rn(vref - ic_d);
  float S, Cc;
  sincospif(u, &S, &Cc);
  S *= 0.31830988618379067f;  // sin(pi u) / pi

  float2 acc[kDopR];
#pragma unroll
  for (int r = 0; r < kDopR; ++r) acc[r] = make_float2(0.f, 0.f);

  const int lb = (int)(B - Bcta);  // thread base inside the staged span
  // register window: win[i] = x[B + jj0 + i]
  float2 win[2 * kDopR];
#pragma unroll
  for (int i = 0; i < kDopR; ++i) win[i] = xs[dpad(lb + i)];

  // taps jj = 0 .. W (W + 1 union taps), streamed in chunks of R
  int jj0 = 0;
  const int ntaps = W + 1;
  for (; jj0 < ntaps; jj0 += kDopR) {
#pragma unroll
    for (int i = 0; i < kDopR; ++i) win[kDopR + i] = xs[dpad(lb + jj0 + kDopR + i)];
#pragma unroll
    for (int q = 0; q < kDopR; ++q) {
      const int jj = jj0 + q;
      if (jj < ntaps) {
        TapW tw = tap_weight(u, jj - ic, S, Cc, SECOND);
        const bool e0 = (jj == 0), eW = (jj == W);
#pragma unroll
        for (int r = 0; r < kDopR; ++r) {
          float h = SECOND ? fmaf(fmaf(0.5f * tw.w2, delta[r], tw.w1), delta[r], tw.w) : fmaf(tw.w1, delta[r], tw.w);
          if (e0) h *= mask0[r];
          if (eW) h *= maskW[r];
          const float2 xv = win[q + r];
          acc[r].x = fmaf(xv.x, h, acc[r].x);
          acc[r].y = fmaf(xv.y, h, acc[r].y);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kDopR; ++i) win[i] = win[kDopR + i];
  }

  // ---- carrier rotation exp(-i 2 pi fc (1 - beta) m / fs) (reading R10), phase reduced in binary64
  const double g = carrier * (1.0 - beta);
  float2 out[kDopR];
#pragma unroll
  for (int r = 0; r < kDopR; ++r) {
    float2 v = acc[r];
    if (g != 0.0) {
      const double psi = g * (double)(mt + r);
      const float rr = __double2float_rn(psi - rint(psi));
      v = cmul(v, expm2pi(rr));
    }
    out[r] = v;
  }
  if (nout == kDopR) {
    float4 *y4 = reinterpret_cast<float4 *>(yp + mt);
#pragma unroll
    for (int h = 0; h < kDopR / 2; ++h) __stcs(y4 + h, make_float4(out[2 * h].x, out[2 * h].y, out[2 * h + 1].x, out[2 * h + 1].y));
  } else {
    for (int r = 0; r < nout; ++r) yp[mt + r] = out[r];
  }
}

// Exact-tap, one-output-per-thread path (Alg. 1 structure) for any alpha.
// Used when |beta - 1| is too large for the union-window / Taylor scheme, and for alpha == 1
// pulses handled by the generic path it returns x exactly (u == 0 case).
__global__ void __launch_bounds__(256) doppler_exact_kernel(const float2 *__restrict__ x, float2 *__restrict__ y,
                                                           int64_t n, int W, const PulseParams *__restrict__ pp,
                                                           int64_t pulse_base, double carrier) {
  const int64_t pulse = blockIdx.y;
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  const float2 *xp = x + pulse * n;
  const double beta = pp[pulse_base + pulse].beta;
  const double t = (double)m * beta;
  const int64_t K = (int64_t)floor(t - 0.5 * (double)W) + 1;
  float2 acc = make_float2(0.f, 0.f);
  const double tc = rint(t);
  if (t == tc) {
    // sinc is a Kronecker delta at integer positions
    const int64_t k = (int64_t)tc;
    if (k >= 0 && k < n && k >= K && k < K + W) acc = xp[k];
  } else {
    const float u = __double2float_rn(t - tc);  // in [-1/2, 1/2]
    float S, Cc;
    sincospif(u, &S, &Cc);
    S *= 0.31830988618379067f;
    for (int64_t k = K; k < K + W; ++k) {
      if (k < 0 || k >= n) continue;
      const int mm = (int)(k - (int64_t)tc);  // d = t - k = u - mm
      const float d = u - (float)mm;
      const float s = (mm & 1) ? -S : S;
      const float h = s / d;
      const float2 xv = __ldg(xp + k);
      acc.x = fmaf(xv.x, h, acc.x);
      acc.y = fmaf(xv.y, h, acc.y);
    }
  }
  const double g = carrier * (1.0 - beta);
  if (g != 0.0) {
    const double psi = g * (double)m;
    acc = cmul(acc, expm2pi(__double2float_rn(psi - rint(psi))));
  }
  y[pulse * n + m] = acc;
}

static cudaError_t launch_doppler_fast(const DopplerArgs &a, bool second) {
  const int64_t tiles = (a.n + kDopM - 1) / kDopM;
  // staged span <= M * max(beta) + W + 3, plus the register window's read-ahead (2R)
  const int span = (int)(kDopM * (1.0 + 2.0 * kDopMaxDrift)) + a.taps + 3 * kDopR + 8;
  const size_t smem = sizeof(float2) * (size_t)(span + (span >> 3) + 8);
  auto kern = second ? doppler_fast_kernel<true> : doppler_fast_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)tiles, (unsigned)a.pulses);
  kern<<<grid, kDopT, smem, a.stream>>>(a.x, a.y, a.n, a.taps, a.pp, a.pulse_base, a.carrier_cycles_per_sample);
  return cudaGetLastError();
}

static cudaError_t launch_doppler_exact(const DopplerArgs &a) {
  dim3 grid((unsigned)((a.n + 255) / 256), (unsigned)a.pulses);
  doppler_exact_kernel<<<grid, 256, 0, a.stream>>>(a.x, a.y, a.n, a.taps, a.pp, a.pulse_base, a.carrier_cycles_per_sample);
  return cudaGetLastError();
}

// Path choice from the largest |beta - 1| among the launched pulses (host-known):
//   drift = |beta - 1| * R / 2 is the largest Taylor step delta of the fast kernel.
//   first order  if drift <= 2e-4 (truncation <= 1.64 delta^2 <= 7e-8 per tap weight)
//   second order if drift <= 2e-3 (truncation <= 1.3 delta^3 <= 1.1e-8)
//   exact taps otherwise.
int doppler_path(double max_abs_beta_m1) {
  const double drift = max_abs_beta_m1 * (kDopR / 2);
  if (drift <= 2.0e-4) return 1;
  if (drift <= kDopMaxDrift) return 2;
  return 0;
}

cudaError_t launch_doppler(const DopplerArgs &a, double max_abs_beta_m1) {
  const int path = doppler_path(max_abs_beta_m1);
  if (path == 0) return launch_doppler_exact(a);
  return launch_doppler_fast(a, path == 2);
}

}  // namespace dc
