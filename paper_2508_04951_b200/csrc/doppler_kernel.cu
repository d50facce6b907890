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
#include <algorithm>

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

// async 8-byte global -> shared copy with zero fill when `valid` is false (cp.async, LDGSTS)
__device__ __forceinline__ void cp_async8(float2 *smem_dst, const float2 *gsrc, bool valid) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int src_size = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gsrc), "r"(src_size) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

struct DopTile {
  int64_t pulse, m0, Bcta;
  double beta;
  int span;
};

__device__ __forceinline__ DopTile dop_tile(int64_t item, int64_t tiles_per_pulse, int64_t n, int W,
                                            const PulseParams *__restrict__ pp, int64_t pulse_base) {
  DopTile t;
  t.pulse = item / tiles_per_pulse;
  t.m0 = (item - t.pulse * tiles_per_pulse) * kDopM;
  t.beta = pp[pulse_base + t.pulse].beta;
  const double halfW = 0.5 * (double)W;
  const int lo_shift = (t.beta < 1.0) ? 1 : 0;
  t.Bcta = (int64_t)floor((double)t.m0 * t.beta - halfW) + 1 - lo_shift;
  const int64_t mlast = t.m0 + kDopM - 1;
  const int64_t Kend = (int64_t)floor((double)mlast * t.beta - halfW) + 1 + W + 2 * kDopR + 8;
  t.span = (int)(Kend - t.Bcta);
  return t;
}

// stage x[Bcta, Bcta + span) of the tile's pulse into padded shared memory (zeros outside [0, n))
__device__ __forceinline__ void dop_stage(float2 *buf, const DopTile &t, const float2 *__restrict__ x, int64_t n) {
  const float2 *xp = x + t.pulse * n;
  for (int i = threadIdx.x; i < t.span; i += kDopT) {
    const int64_t k = t.Bcta + i;
    const bool ok = (k >= 0 && k < n);
    cp_async8(buf + dpad(i), xp + (ok ? k : 0), ok);
  }
}

// Persistent, double-buffered pipeline: while the CTA computes tile i from one shared buffer,
// the input span of tile i + gridDim.x streams into the other with cp.async (zero-filled).
template <bool SECOND>
__global__ void __launch_bounds__(kDopT, 2)
    doppler_pipe_kernel(const float2 *__restrict__ x, float2 *__restrict__ y, int64_t n, int W,
                        const PulseParams *__restrict__ pp, int64_t pulse_base, double carrier, int64_t pulses,
                        int buf_elems) {
  extern __shared__ float2 xs[];
  const int tid = threadIdx.x;
  const int64_t tiles_per_pulse = (n + kDopM - 1) / kDopM;
  const int64_t total = pulses * tiles_per_pulse;
  const double halfW = 0.5 * (double)W;
  int64_t item = blockIdx.x;
  if (item >= total) return;
  DopTile cur = dop_tile(item, tiles_per_pulse, n, W, pp, pulse_base);
  dop_stage(xs, cur, x, n);
  cp_async_commit();
  int bsel = 0;
  for (; item < total; item += gridDim.x) {
    // ---- prefetch the next tile into the other buffer
    const int64_t nitem = item + gridDim.x;
    DopTile nxt;
    if (nitem < total) {
      nxt = dop_tile(nitem, tiles_per_pulse, n, W, pp, pulse_base);
      dop_stage(xs + (bsel ^ 1) * buf_elems, nxt, x, n);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const float2 *sb = xs + bsel * buf_elems;

    // ---- this thread's R consecutive outputs
    const int64_t mt = cur.m0 + (int64_t)tid * kDopR;
    const double beta = cur.beta;
    const int lo_shift = (beta < 1.0) ? 1 : 0;
    const int64_t B = (int64_t)floor((double)mt * beta - halfW) + 1 - lo_shift;
    float mask0[kDopR], maskW[kDopR];
#pragma unroll
    for (int r = 0; r < kDopR; ++r) {
      const int64_t Kr = (int64_t)floor((double)(mt + r) * beta - halfW) + 1;
      const int a = (int)(Kr - r - B);  // 0 or 1: this output's window offset inside the union
      mask0[r] = (a == 0) ? 1.f : 0.f;
      maskW[r] = (a == 1) ? 1.f : 0.f;
    }
    // Taylor steps delta_r = (r - R/2)(beta - 1), paired for FFMA2
    const float db = (float)(beta - 1.0);
    float2 dl[kDopR / 2];
#pragma unroll
    for (int h = 0; h < kDopR / 2; ++h) dl[h] = make_float2((2 * h - kDopR / 2) * db, (2 * h + 1 - kDopR / 2) * db);
    // reference position inside the union, split into nearest integer + fraction in [-1/2, 1/2]
    const double vref = (double)(mt + kDopR / 2) * beta - (double)(B + kDopR / 2);
    const double ic_d = rint(vref);
    const int ic = (int)ic_d;
    const float u = __double2float_rn(vref - ic_d);
    float S, Cc;
    sincospif(u, &S, &Cc);
    S *= 0.31830988618379067f;  // sin(pi u) / pi
    // centre-tap weights (d = u): series near 0 (sinc even; avoids C/d - S/(pi d^2) cancellation)
    float wc, w1c, w2c;
    {
      const float pd2 = 9.8696044010893586f * u * u;
      if (fabsf(u) < 0.25f) {
        wc = (u == 0.f) ? 1.f : S * frcp(u);
        w1c = -3.2898681336964529f * u * (1.f - pd2 * (0.1f - pd2 * (1.f / 280.f)));
        w2c = -3.2898681336964529f * (1.f - pd2 * (0.3f - pd2 * (1.f / 56.f)));
      } else {
        const float inv = frcp(u);
        wc = S * inv;
        w1c = inv * fmaf(-S, inv, Cc);
        w2c = fmaf(-9.8696044010893586f, wc, -2.f * w1c * inv);
      }
    }
    const int lb = (int)(B - cur.Bcta);
    float2 acc[kDopR];
#pragma unroll
    for (int r = 0; r < kDopR; ++r) acc[r] = make_float2(0.f, 0.f);

    // weights of union tap jj (d = u - (jj - ic)); returns (w, w1, w2)
    auto weight = [&](int jj, float &w, float &w1, float &w2) {
      const int m = jj - ic;
      const float d = u - (float)m;
      const float inv = frcp(d);
      const float sg = (m & 1) ? -1.f : 1.f;
      const float s = sg * S, c = sg * Cc;
      w = s * inv;
      w1 = inv * fmaf(-s, inv, c);
      w2 = SECOND ? fmaf(-9.8696044010893586f, w, -2.f * w1 * inv) : 0.f;
      if (m == 0) {
        w = wc;
        w1 = w1c;
        w2 = w2c;
      }
    };
    auto mac_tap = [&](const float2 *xv, float w, float w1, float w2, const float *mask) {
#pragma unroll
      for (int h = 0; h < kDopR / 2; ++h) {
        float2 hh;
        if (SECOND) {
          float2 t = __ffma2_rn(make_float2(0.5f * w2, 0.5f * w2), dl[h], make_float2(w1, w1));
          hh = __ffma2_rn(t, dl[h], make_float2(w, w));
        } else {
          hh = __ffma2_rn(make_float2(w1, w1), dl[h], make_float2(w, w));
        }
        if (mask) {
          hh.x *= mask[2 * h];
          hh.y *= mask[2 * h + 1];
        }
        acc[2 * h] = __ffma2_rn(xv[2 * h], make_float2(hh.x, hh.x), acc[2 * h]);
        acc[2 * h + 1] = __ffma2_rn(xv[2 * h + 1], make_float2(hh.y, hh.y), acc[2 * h + 1]);
      }
    };

    {  // edge tap jj = 0 (owned by outputs with a_r == 0)
      float2 xv[kDopR];
#pragma unroll
      for (int r = 0; r < kDopR; ++r) xv[r] = sb[dpad(lb + r)];
      float w, w1, w2;
      weight(0, w, w1, w2);
      mac_tap(xv, w, w1, w2, mask0);
    }
    // interior taps jj = 1 .. W-1, streamed in chunks of R through a register window
    float2 win[2 * kDopR];
#pragma unroll
    for (int i = 0; i < kDopR; ++i) win[i] = sb[dpad(lb + 1 + i)];
    for (int jj0 = 1; jj0 < W; jj0 += kDopR) {
#pragma unroll
      for (int i = 0; i < kDopR; ++i) win[kDopR + i] = sb[dpad(lb + jj0 + kDopR + i)];
#pragma unroll
      for (int q = 0; q < kDopR; ++q) {
        float w, w1, w2;
        weight(jj0 + q, w, w1, w2);
        if (jj0 + q >= W) w = w1 = w2 = 0.f;  // padding taps of the last chunk
        mac_tap(&win[q], w, w1, w2, nullptr);
      }
#pragma unroll
      for (int i = 0; i < kDopR; ++i) win[i] = win[kDopR + i];
    }
    {  // edge tap jj = W (owned by outputs with a_r == 1)
      float2 xv[kDopR];
#pragma unroll
      for (int r = 0; r < kDopR; ++r) xv[r] = sb[dpad(lb + r + W)];
      float w, w1, w2;
      weight(W, w, w1, w2);
      mac_tap(xv, w, w1, w2, maskW);
    }

    // ---- carrier rotation (reading R10) and store
    const double g = carrier * (1.0 - beta);
    float2 *yp = y + cur.pulse * n;
    if (g != 0.0) {
#pragma unroll
      for (int r = 0; r < kDopR; ++r) {
        const double psi = g * (double)(mt + r);
        acc[r] = cmul(acc[r], expm2pi(__double2float_rn(psi - rint(psi))));
      }
    }
    if (mt + kDopR <= n) {
      float4 *y4 = reinterpret_cast<float4 *>(yp + mt);
#pragma unroll
      for (int h = 0; h < kDopR / 2; ++h)
        __stcs(y4 + h, make_float4(acc[2 * h].x, acc[2 * h].y, acc[2 * h + 1].x, acc[2 * h + 1].y));
    } else {
#pragma unroll
      for (int r = 0; r < kDopR; ++r)
        if (mt + r < n) yp[mt + r] = acc[r];
    }
    __syncthreads();  // everyone is done with buffer bsel before it is refilled
    cur = nxt;
    bsel ^= 1;
  }
  cp_async_wait<0>();
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
  const int64_t tiles = (a.n + kDopM - 1) / kDopM * a.pulses;
  // staged span <= M * max(beta) + W + 2R + 10 samples (fast path: |beta - 1| <= 5e-4), padded 9/8
  const int span = (int)(kDopM * (1.0 + 2.0 * kDopMaxDrift)) + a.taps + 2 * kDopR + 16;
  const int buf = span + (span >> 3) + 8;
  const size_t smem = 2 * sizeof(float2) * (size_t)buf;
  auto kern = second ? doppler_pipe_kernel<true> : doppler_pipe_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per_sm = 2;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDopT, smem);
  const int64_t grid = std::min<int64_t>(tiles, (int64_t)sms * std::max(per_sm, 1));
  kern<<<(unsigned)grid, kDopT, smem, a.stream>>>(a.x, a.y, a.n, a.taps, a.pp, a.pulse_base, a.carrier_cycles_per_sample,
                                                  a.pulses, buf);
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
