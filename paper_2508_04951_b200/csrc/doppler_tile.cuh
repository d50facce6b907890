// doppler_tile.cuh -- Doppler (windowed sinc) tile machinery shared by the doppler kernels
// and the fused persistent correction kernel.  See doppler_kernel.cu for the method notes.
#pragma once
#include <algorithm>
#include <type_traits>

#include "dc_kernels.h"
#include "tma.cuh"

namespace dc {

constexpr int kDopT = 256;  // threads per CTA
#ifndef DC_DOP_R
#define DC_DOP_R 11
#endif
constexpr int kDopR = DC_DOP_R;  // outputs per thread: odd, so lanes' windows (R samples apart) hit distinct banks
constexpr int kDopM = kDopT * kDopR;     // outputs per tile
constexpr double kDopMaxDrift = 2.0e-3;  // max |beta - 1| * R / 2 for the fast path

__device__ __forceinline__ float frcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
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

__device__ __forceinline__ DopTile dop_tile(int64_t item, int64_t tiles_per_pulse, int W,
                                            const PulseParams *__restrict__ pp, int64_t pulse_base) {
  DopTile t;
  t.pulse = item / tiles_per_pulse;
  t.m0 = (item - t.pulse * tiles_per_pulse) * kDopM;
  t.beta = pp[pulse_base + t.pulse].beta;
  const double halfW = 0.5 * (double)W;
  const int lo_shift = (t.beta < 1.0) ? 1 : 0;
  t.Bcta = (int64_t)floor((double)t.m0 * t.beta - halfW) + 1 - lo_shift;
  t.Bcta -= (t.Bcta & 1);  // TMA boxes must start 16-byte aligned: even sample index
  const int64_t mlast = t.m0 + kDopM - 1;
  const int64_t Kend = (int64_t)floor((double)mlast * t.beta - halfW) + 1 + W + kDopR + 4;
  t.span = (int)(Kend - t.Bcta);
  return t;
}

// stage x[Bcta, Bcta + span) of the tile's pulse into shared memory with the TMA engine:
// ceil(span / 256) boxes of 256 samples; coordinates outside [0, n) are zero-filled by hardware
// (R12).  Issued by one thread; completion is the buffer's transaction-count mbarrier.
constexpr int kDopBox = 256;
__device__ __forceinline__ int dop_nbox(const DopTile &t) { return (t.span + kDopBox - 1) / kDopBox; }
__device__ __forceinline__ void dop_stage_tma(float2 *buf, const DopTile &t, const CUtensorMap *xmap, uint64_t *bar) {
  const int nb = dop_nbox(t);
  fence_proxy_async();
  mbar_arrive_expect_tx(bar, (unsigned)(nb * kDopBox * sizeof(float2)));
  for (int i = 0; i < nb; ++i) tma_load_2d(buf + i * kDopBox, xmap, (int)(t.Bcta + i * kDopBox), (int)t.pulse, bar);
}

// sinc weight w = sinc(d), w1 = sinc'(d), w2 = sinc''(d) at d = u - m (u in [-1/2, 1/2]):
// sin(pi d) = (-1)^m sin(pi u), cos(pi d) = (-1)^m cos(pi u); S = sin(pi u)/pi, Cc = cos(pi u).
template <bool SECOND>
__device__ __forceinline__ void tap_w(float u, int m, float S, float Cc, float &w, float &w1, float &w2) {
  const float d = u - (float)m;
  const float inv = frcp(d);
  const float s = (m & 1) ? -S : S, c = (m & 1) ? -Cc : Cc;
  w = s * inv;
  w1 = inv * (c - w);
  w2 = SECOND ? fmaf(-9.8696044010893586f, w, -2.f * w1 * inv) : 0.f;
}

// Kaiser taper K(d) and K'(d) (reading R17) by Horner on the normalised I0 series in
// q = qa (1 - d^2 / L^2); the coefficients sit in the kernel-parameter (constant) bank.
// NT = number of series terms evaluated (17 when the plan's kb <= 8, else kTaperTerms)
template <int NT = kTaperTerms>
__device__ __forceinline__ void kaiser_taper(const TaperCoef &tc, float d, float &K, float &dK) {
  const float q = tc.qa * fmaf(-d * d, tc.inv_L2, 1.0f);
  float b = tc.c[NT - 1], db = 0.f;
#pragma unroll
  for (int j = NT - 2; j >= 0; --j) {
    db = fmaf(db, q, b);
    b = fmaf(b, q, tc.c[j]);
  }
  K = b;
  dK = db * (-2.0f * tc.qa * tc.inv_L2 * d);  // dP/dq * dq/dd
}

// One doppler tile: R = 9 outputs per thread from the staged span sb (x[Bcta + i] = sb[i]),
// carrier rotation, then a coalesced store of the tile's M outputs through `ob` (one barrier
// inside; callers add the trailing barrier before ob / sb are reused).
// BAR = 0: the whole CTA (kDopT threads) computes the tile; BAR > 0: named barrier BAR over the
// kDopT threads 0 .. kDopT-1 (the consumer warps of a warp-specialised kernel).
// TAPER > 0: Kaiser-tapered weights h = sinc K, h' = sinc' K + sinc K' (first-order path only), with
// TAPER series terms.
template <bool SECOND, int WT, int BAR = 0, int TAPER = 0>
__device__ __forceinline__ void dop_tile_compute(const float2 *__restrict__ sb, const DopTile &cur, int W_rt,
                                                 float2 *__restrict__ ob, float2 *__restrict__ y, int64_t n,
                                                 double carrier, const TaperCoef *tcp = nullptr) {
  static_assert(!(TAPER > 0 && SECOND), "the tapered path is first order");
  const int W = (WT > 0) ? WT : W_rt;
  const double halfW = 0.5 * (double)W;
  const int tid = threadIdx.x;
    // ---- this thread's R consecutive outputs: exact binary64 window bookkeeping
  const int64_t mt = cur.m0 + (int64_t)tid * kDopR;
  const double beta = cur.beta;
  const int lo_shift = (beta < 1.0) ? 1 : 0;
  // window decisions use the oracle's two separately rounded binary64 operations, fl(fl(m beta) - W/2)
  // (__dmul_rn / __dsub_rn: never contracted into an FMA), so membership matches R9 exactly
  const int64_t B = (int64_t)floor(__dsub_rn(__dmul_rn((double)mt, beta), halfW)) + 1 - lo_shift;
  float mask0[kDopR], maskW[kDopR];
#pragma unroll
  for (int r = 0; r < kDopR; ++r) {
    const int64_t Kr = (int64_t)floor(__dsub_rn(__dmul_rn((double)(mt + r), beta), halfW)) + 1;
    const int a = (int)(Kr - r - B);  // 0 or 1: this output's window offset inside the union
    mask0[r] = (a == 0) ? 1.f : 0.f;
    maskW[r] = (a == 1) ? 1.f : 0.f;
  }
  // Taylor steps delta_r = (r - R/2)(beta - 1): pairs for FFMA2 + one single
  constexpr int RC = kDopR / 2;  // reference output
  const float db = (float)(beta - 1.0);
  float2 dl[kDopR / 2];
#pragma unroll
  for (int h = 0; h < kDopR / 2; ++h) dl[h] = make_float2((2 * h - RC) * db, (2 * h + 1 - RC) * db);
  const float dlast = (kDopR - 1 - RC) * db;
  // reference position inside the union, split into nearest integer + fraction in [-1/2, 1/2]
  const double vref = (double)(mt + RC) * beta - (double)(B + RC);
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
      w1c = inv * (Cc - wc);
      w2c = fmaf(-9.8696044010893586f, wc, -2.f * w1c * inv);
    }
  }
  // the generic formula is exact enough except at the centre tap when |u| is tiny; decide per warp
  const bool tiny = __any_sync(0xffffffffu, fabsf(u) < 1.0e-3f);
  const float2 *xb = sb + (B - cur.Bcta);  // x[B + i] = xb[i]
  // sign of tap jj: (-1)^(jj - ic); fold (-1)^ic into the per-thread constants
  const float Sp = (ic & 1) ? -S : S, Cp = (ic & 1) ? -Cc : Cc;
  const float icf = (float)ic;
  float2 acc[kDopR];
#pragma unroll
  for (int r = 0; r < kDopR; ++r) acc[r] = make_float2(0.f, 0.f);

  auto mac = [&](const float2 *xv, float w, float w1, float w2, const float *mask) {
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
    float hl = SECOND ? fmaf(fmaf(0.5f * w2, dlast, w1), dlast, w) : fmaf(w1, dlast, w);
    if (mask) hl *= mask[kDopR - 1];
    acc[kDopR - 1] = __ffma2_rn(xv[kDopR - 1], make_float2(hl, hl), acc[kDopR - 1]);
  };
  // weights of union tap jj: d = u - (jj - ic) (exact integer subtraction, then one rounding);
  // sinc = (-1)^(jj-ic) S / d, sinc' = ((-1)^(jj-ic) C - sinc) / d, sinc'' = -pi^2 sinc - 2 sinc'/d.
  // TINY: override the centre tap (jj == ic) with its series values.
  auto weights = [&](int jj, auto TINYc, float &w, float &w1, float &w2) {
    constexpr bool TINY = decltype(TINYc)::value;
    const float d = u - ((float)jj - icf);
    const float inv = frcp(d);
    const float s = (jj & 1) ? -Sp : Sp, c = (jj & 1) ? -Cp : Cp;
    w = s * inv;
    w1 = inv * (c - w);
    w2 = SECOND ? fmaf(-9.8696044010893586f, w, -2.f * w1 * inv) : 0.f;
    if (TINY && jj == ic) {
      w = wc;
      w1 = w1c;
      w2 = w2c;
    }
    if constexpr (TAPER > 0) {
      float K, dK;
      kaiser_taper<TAPER>(*tcp, d, K, dK);
      // the taper's centre weight is 1 exactly (R17): the FP32 Horner sum need not round to 1
      if (TINY && d == 0.f) K = 1.f;
      w1 = fmaf(w1, K, w * dK);
      w *= K;
    }
  };
  auto taps = [&](auto TINYc) {
    // register window xw[r] = x[B + jj + r]; union taps jj = 0 .. W
    float2 xw[kDopR];
#pragma unroll
    for (int r = 0; r < kDopR; ++r) xw[r] = xb[r];
    {
      float w, w1, w2;
      weights(0, TINYc, w, w1, w2);
      mac(xw, w, w1, w2, mask0);
    }
    auto step = [&](int jj) {  // slide the window to tap jj and apply it (interior taps)
#pragma unroll
      for (int r = 0; r < kDopR - 1; ++r) xw[r] = xw[r + 1];
      xw[kDopR - 1] = xb[jj + kDopR - 1];
      float w, w1, w2;
      weights(jj, TINYc, w, w1, w2);
      mac(xw, w, w1, w2, nullptr);
    };
    if constexpr (WT > 0) {
#pragma unroll
      for (int jj = 1; jj < WT; ++jj) step(jj);
    } else {
#pragma unroll 1
      for (int jj = 1; jj < W; ++jj) step(jj);
    }
    {
#pragma unroll
      for (int r = 0; r < kDopR - 1; ++r) xw[r] = xw[r + 1];
      xw[kDopR - 1] = xb[W + kDopR - 1];
      float w, w1, w2;
      weights(W, TINYc, w, w1, w2);
      mac(xw, w, w1, w2, maskW);
    }
  };
  if (tiny) {
    taps(std::true_type());
  } else {
    taps(std::false_type());
  }

  // ---- carrier rotation (reading R10), then coalesced store through shared memory
  const double g = carrier * (1.0 - beta);
  if (g != 0.0) {
#pragma unroll
    for (int r = 0; r < kDopR; ++r) {
      const double psi = g * (double)(mt + r);
      acc[r] = cmul(acc[r], expm2pi(__double2float_rn(psi - rint(psi))));
    }
  }
  // a warp's 32 x R outputs are contiguous (thread t owns outputs [t R, t R + R)): each warp stages
  // its own segment and stores it with coalesced 16-byte stores -- no CTA barrier (BAR unused)
#pragma unroll
  for (int r = 0; r < kDopR; ++r) ob[tid * kDopR + r] = acc[r];
  __syncwarp();
  {
    constexpr int kSeg = 32 * kDopR;  // outputs per warp (even: 16-byte aligned segments)
    const int w = tid >> 5, lane = tid & 31;
    const int64_t mw = cur.m0 + (int64_t)w * kSeg;
    float2 *yp = y + cur.pulse * n + mw;
    const float2 *os = ob + w * kSeg;
    const int64_t valid = min((int64_t)kSeg, n - mw);
    if (valid == kSeg) {
      const float4 *o4 = reinterpret_cast<const float4 *>(os);
      float4 *y4 = reinterpret_cast<float4 *>(yp);
      for (int i = lane; i < kSeg / 2; i += 32) __stcs(y4 + i, o4[i]);
    } else {
      for (int i = lane; i < valid; i += 32) yp[i] = os[i];
    }
  }
}

}  // namespace dc
