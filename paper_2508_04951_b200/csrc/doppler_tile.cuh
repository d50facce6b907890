// doppler_tile.cuh -- Doppler (windowed sinc) tile machinery of doppler_pipe_kernel.
// See doppler_kernel.cu for the method notes (Eq. 16; window P:L533; readings R8-R12).
#pragma once
#include <algorithm>
#include <type_traits>

#include "dc_kernels.h"
#include "tma.cuh"

namespace dc {

// threads per CTA of the Doppler pipeline kernel: a template parameter chosen per launch (doppler_kernel.cu);
// kDopT is the default (tapered windows, W = 16) and the unit of the tile-geometry constants below
constexpr int kDopT = 256;
#ifndef DC_DOP_R
#define DC_DOP_R 11
#endif
constexpr int kDopR = DC_DOP_R;  // outputs per thread: odd, so lanes' windows (R samples apart) hit distinct banks
// R per compile-time W: R = 9 at W = 128 (the 129-tap loop of R = 11 is register-bound: 58 vs 45 GS/s
// measured), 11 otherwise (W = 32: 201 vs 190 GS/s for R = 9, 146 for R = 13)
__host__ __device__ constexpr int dop_r(int WT) { return WT >= 128 ? 9 : kDopR; }
// R of doppler_pipe_kernel<.., T>: 13 for the compile-time W <= 32 at T >= 256 (round 2, on the first-order
// path: W = 32 204.7 vs 199.5 GS/s, W = 16 320 vs 304, Kaiser-8 103 vs 96); T = 128 (n < 2^16) keeps 11
// (4096-sample pulses: 169 vs 146 -- tile quantisation), W = 64 keeps 11 (111.6 vs 109.5), W = 128 keeps 9
__host__ __device__ constexpr int dop_r_pipe(int WT, int T) {
  return WT >= 128 ? 9 : (T >= 256 && WT > 0 && WT <= 32) ? 13 : kDopR;
}
constexpr int kDopM = kDopT * kDopR;     // outputs per tile (R = kDopR)
constexpr int kDopSeg = 32 * kDopR;      // outputs per warp (even: 16-byte aligned bulk stores)
constexpr double kDopMaxDrift = 2.0e-3;  // max |beta - 1| * R / 2 for the fast path
#ifndef DC_DOP_NBUF
#define DC_DOP_NBUF 3
#endif
constexpr int kDopBufs = DC_DOP_NBUF;    // input staging buffers (tile i + kDopBufs is staged once tile i is read)
static_assert(kDopSeg % 2 == 0 && (32 * dop_r(128)) % 2 == 0, "warp segments must be 16-byte multiples");

__device__ __forceinline__ float frcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Geometry of one tile (pulse, first output m0, staged span [Bcta, Bcta + span), beta): computed
// by the producer thread when it stages the tile and kept in shared memory next to the buffer.
struct __align__(16) DopTile {
  int64_t pulse, m0, Bcta;
  double beta;
  int span, pad0;
  int64_t pad1;
};
static_assert(sizeof(DopTile) == 48, "bulk copies move multiples of 16 bytes");

// tile `item` = (pulse, tile of kDopM outputs) -- 32-bit index arithmetic (items < 2^32: pulses per
// launch <= 65535, tiles per pulse <= 2^24 / kDopM); beta = that pulse's 1/alpha
__device__ __forceinline__ uint32_t dop_pulse(uint32_t item, uint32_t tiles_per_pulse) { return item / tiles_per_pulse; }
template <int R = kDopR, int T = kDopT>
__device__ __forceinline__ DopTile dop_tile(uint32_t item, uint32_t tiles_per_pulse, int W, double beta) {
  constexpr int M = T * R;
  DopTile t;
  const uint32_t pulse = item / tiles_per_pulse;
  t.pulse = pulse;
  t.m0 = (int64_t)(item - pulse * tiles_per_pulse) * M;
  t.beta = beta;
  const double halfW = 0.5 * (double)W;
  const int lo_shift = (t.beta < 1.0) ? 1 : 0;
  t.Bcta = (int64_t)floor((double)t.m0 * t.beta - halfW) + 1 - lo_shift;
  t.Bcta -= (t.Bcta & 1);  // TMA boxes must start 16-byte aligned: even sample index
  const int64_t mlast = t.m0 + M - 1;
  const int64_t Kend = (int64_t)floor((double)mlast * t.beta - halfW) + 1 + W + R + 4;
  t.span = (int)(Kend - t.Bcta);
  t.pad0 = 0;
  t.pad1 = 0;
  return t;
}

// stage x[Bcta, Bcta + span) of the tile's pulse into shared memory with the TMA engine:
// ceil(span / 256) boxes of 256 samples; coordinates outside [0, n) are zero-filled by hardware
// (R12).  Issued by one thread; completion is the buffer's transaction-count mbarrier.
constexpr int kDopBox = 256;
__device__ __forceinline__ int dop_nbox(const DopTile &t) { return (t.span + kDopBox - 1) / kDopBox; }
// The tile's geometry travels with it: the producer writes it to its CTA's global slot and the TMA
// engine lands it in `desc` (a 48-byte box of the tensor map dmap over the slots), counted by the same
// mbarrier as the data -- consumers read it after their wait; no generic shared-memory write passes
// between producer and consumers.
__device__ __forceinline__ void dop_stage_tma(float2 *buf, const DopTile &t, const CUtensorMap *xmap, uint64_t *bar,
                                              DopTile *desc, DopTile *gslot, const CUtensorMap *dmap, int slot) {
  const int nb = dop_nbox(t);
  *gslot = t;
  fence_proxy_async_global();  // the generic write above -> visible to the TMA read below
  fence_proxy_async();
  mbar_arrive_expect_tx(bar, (unsigned)(nb * kDopBox * sizeof(float2) + sizeof(DopTile)));
  tma_load_2d(desc, dmap, 0, slot, bar);
  for (int i = 0; i < nb; ++i) tma_load_2d(buf + i * kDopBox, xmap, (int)(t.Bcta + i * kDopBox), (int)t.pulse, bar);
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

// Hann taper K(d) = (1 + cos(pi d / L)) / 2 and K'(d) = -(pi / 2L) sin(pi d / L), |d| <= L (reading R17):
// SFU sin/cos of an argument in [-pi, pi] (absolute error ~4e-7, i.e. ~2e-7 in K)
__device__ __forceinline__ void hann_taper(const TaperCoef &tc, float d, float &K, float &dK) {
  float sn, cs;
  __sincosf(d * tc.pi_over_L, &sn, &cs);
  K = fmaf(0.5f, cs, 0.5f);
  dK = -0.5f * tc.pi_over_L * sn;
}

// taper code TAPER: 0 none, kTaperHann, else a Kaiser series of TAPER terms
template <int TAPER>
__device__ __forceinline__ void taper_eval(const TaperCoef &tc, float d, float &K, float &dK) {
  if constexpr (TAPER == kTaperHann) {
    hann_taper(tc, d, K, dK);
  } else {
    kaiser_taper<TAPER>(tc, d, K, dK);
  }
}

// Window membership of the thread's R outputs (reading R9, the oracle's roundings): output r owns the
// union taps [a_r, a_r + W - 1], a_r in {0, 1}, a_r = 1 iff its window start K_r = floor(x_r) + 1
// equals B + r + 1, i.e. iff x_r = fl(fl((mt + r) beta) - W/2) >= B + r (exact binary64 comparison:
// integers below 2^53).  X_r = x_r - (B + r) moves linearly in r by beta - 1 up to ~1 ulp(t) of
// rounding, so when the first and last outputs are on the same side by a clear margin all R decisions
// agree; only a thread whose outputs straddle a window step (~R |beta - 1| of all threads) evaluates
// each output.  Returns the bit set {r : a_r = 1}.
template <int R = kDopR>
__device__ __forceinline__ uint32_t dop_membership(double md, double beta, double halfW, double Bd, double x0) {
  constexpr uint32_t kAll = (1u << R) - 1u;
  constexpr double kMargin = 1.0e-7;  // >> rounding of t (ulp(2^25) = 7.5e-9)
  const double X0 = x0 - Bd;          // exact (Sterbenz: |x0 - Bd| <= 1)
  const double XL = __dsub_rn(__dmul_rn(md + (double)(R - 1), beta), halfW) - (Bd + (double)(R - 1));
  if (X0 >= kMargin && XL >= kMargin) return kAll;
  if (X0 <= -kMargin && XL <= -kMargin) return 0u;
  uint32_t own1 = 0;
#pragma unroll 1
  for (int r = 0; r < R; ++r)
    own1 |= (__dsub_rn(__dmul_rn(md + (double)r, beta), halfW) >= Bd + (double)r) ? (1u << r) : 0u;
  return own1;
}

// One doppler tile: R outputs per thread from the staged span sb (x[Bcta + i] = sb[i]), carrier
// rotation, then the warp's R x 32 contiguous outputs leave through its shared-memory segment `ob`
// (kDopSeg samples) as ONE bulk async copy issued by lane 0 (no LDS/STG per output, no CTA barrier).
// TAPER > 0: tapered weights h = sinc K, h' = sinc' K + sinc K' (first-order path only): the Hann window
// (TAPER == kTaperHann) or a Kaiser window of TAPER series terms.
// DIRECT: each thread stores its own R outputs (m < n) straight to y -- no staging segment (`ob` unused),
// for the fused kernels whose shared memory is taken by their FFT tiles.
template <bool SECOND, int WT, int TAPER = 0, int R = dop_r(WT), bool DIRECT = false>
__device__ __forceinline__ void dop_tile_compute(const float2 *__restrict__ sb, const DopTile &cur, int W_rt,
                                                 float2 *__restrict__ ob, float2 *__restrict__ y, int64_t n,
                                                 double carrier, const TaperCoef *tcp = nullptr) {
  static_assert(!(TAPER > 0 && SECOND), "the tapered path is first order");
  constexpr int SEG = 32 * R;  // outputs per warp
  const int W = (WT > 0) ? WT : W_rt;
  const double halfW = 0.5 * (double)W;
  const int tid = threadIdx.x, lane = tid & 31;
  // ---- this thread's R consecutive outputs: exact binary64 window bookkeeping.  Window decisions
  // use the oracle's two separately rounded binary64 operations fl(fl(m beta) - W/2) (__dmul_rn /
  // __dsub_rn: never contracted into an FMA), so membership matches R9 exactly.
  const int64_t mt = cur.m0 + (int64_t)tid * R;
  const double beta = cur.beta;
  const int lo_shift = (beta < 1.0) ? 1 : 0;
  const double md = (double)mt;
  const double x0 = __dsub_rn(__dmul_rn(md, beta), halfW);
  const int64_t B = (int64_t)floor(x0) + 1 - lo_shift;  // union base: x[B + i], i = 0 .. W + R - 1
#ifdef DC_DEBUG_CHECKS
  // debug builds (tests/test_gpu_debug_checks.py): the union window lies inside the staged / resident span
  if (mt < n && (B - cur.Bcta < 0 || B - cur.Bcta + W + R > cur.span)) __trap();
#endif
  const double Bd = (double)B;
  const uint32_t own1 = dop_membership<R>(md, beta, halfW, Bd, x0);
  // Taylor steps delta_r = (r - R/2)(beta - 1): pairs for FFMA2 (+ one single for odd R)
  constexpr int RC = R / 2;  // reference output
  const float db = (float)(beta - 1.0);
  float2 dl[R / 2];
#pragma unroll
  for (int h = 0; h < R / 2; ++h) dl[h] = make_float2((2 * h - RC) * db, (2 * h + 1 - RC) * db);
  const float dlast = (R - 1 - RC) * db;  // the unpaired last output (odd R)
  // Reference position (output RC) relative to the union's middle tap Mi = floor(W/2): vrel lies in
  // (-1.0002, 1.5002), so the sample nearest to it is union tap Mi + k0, k0 = rint(vrel) in {-1, .., 2}.
  // Union tap jj = Mi + k sits at distance d_k = vrel - k.  Taps k != k0 (|d| >= 1/2) take d = uf - k, one
  // FADD with a compile-time k from the FP32 vrel (absolute error <= 2^-24: relative <= 2^-23); the nearest
  // tap takes its weights from u = vrel - k0 rounded from binary64 (full relative precision next to the
  // sample) by the series below -- so the tap loop has a single code path (no per-warp "tiny u" branch).
  const int Mi = W >> 1;
  const double vrel = (md + (double)RC) * beta - (Bd + (double)(RC + Mi));
  const double k0d = rint(vrel);
  const int k0 = (int)k0d;
  const float u = __double2float_rn(vrel - k0d);
  const float uf = __double2float_rn(vrel);
  float S, Cc;
  sincospif(u, &S, &Cc);  // (the SFU __sincosf measured 1.2e-5 rel-L2 at W = 32: too coarse)
  S *= 0.31830988618379067f;  // sin(pi u) / pi
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
  const float2 *xb = sb + (B - cur.Bcta);  // x[B + i] = xb[i]
  const float Sp = (k0 & 1) ? -S : S, Cp = (k0 & 1) ? -Cc : Cc;
  float2 acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = make_float2(0.f, 0.f);
  auto mac = [&](const float2 *xv, float w, float w1, float w2, auto EDGEc) {
    constexpr int EDGE = decltype(EDGEc)::value;
    auto keep = [&](int r) { return EDGE == 0 || (((own1 >> r) & 1u) == (EDGE == 2 ? 1u : 0u)); };
#pragma unroll
    for (int h = 0; h < R / 2; ++h) {
      float2 hh;
      if (SECOND) {
        float2 t = __ffma2_rn(make_float2(0.5f * w2, 0.5f * w2), dl[h], make_float2(w1, w1));
        hh = __ffma2_rn(t, dl[h], make_float2(w, w));
      } else {
        hh = __ffma2_rn(make_float2(w1, w1), dl[h], make_float2(w, w));
      }
      if (EDGE) {
        hh.x = keep(2 * h) ? hh.x : 0.f;
        hh.y = keep(2 * h + 1) ? hh.y : 0.f;
      }
      acc[2 * h] = __ffma2_rn(xv[2 * h], make_float2(hh.x, hh.x), acc[2 * h]);
      acc[2 * h + 1] = __ffma2_rn(xv[2 * h + 1], make_float2(hh.y, hh.y), acc[2 * h + 1]);
    }
    if constexpr (R & 1) {
      float hl = SECOND ? fmaf(fmaf(0.5f * w2, dlast, w1), dlast, w) : fmaf(w1, dlast, w);
      if (EDGE) hl = keep(R - 1) ? hl : 0.f;
      acc[R - 1] = __ffma2_rn(xv[R - 1], make_float2(hl, hl), acc[R - 1]);
    }
  };
  // weights of union tap jj = Mi + k at distance d: sinc = (-1)^k Sp / d, sinc' = ((-1)^k Cp - sinc) / d,
  // sinc'' = -pi^2 sinc - 2 sinc'/d; the nearest tap (k == k0, possible only for k in [-1, 2]) takes wc, w1c, w2c
  auto weights = [&](int k, float d, float &w, float &w1, float &w2) {
    const float inv = frcp(d);
    const float s = (k & 1) ? -Sp : Sp, c = (k & 1) ? -Cp : Cp;
    w = s * inv;
    w1 = inv * (c - w);
    w2 = SECOND ? fmaf(-9.8696044010893586f, w, -2.f * w1 * inv) : 0.f;
    const bool near = (WT == 0 || (k >= -1 && k <= 2)) && k == k0;
    if (near) {
      w = wc;
      w1 = w1c;
      w2 = w2c;
    }
    if constexpr (TAPER > 0) {
      float K, dK;
      taper_eval<TAPER>(*tcp, near ? u : d, K, dK);
      if (near && u == 0.f) K = 1.f;
      w1 = fmaf(w1, K, w * dK);
      w *= K;
    }
  };
  // distance of union tap Mi + k
  auto dist = [&](int k) { return ((WT == 0 || (k >= -1 && k <= 2)) && k == k0) ? u : uf - (float)k; };
  {
    float2 xw[R];
#pragma unroll
    for (int r = 0; r < R; ++r) xw[r] = xb[r];
    {
      float w, w1, w2;
      weights(-Mi, dist(-Mi), w, w1, w2);
      mac(xw, w, w1, w2, std::integral_constant<int, 1>());
    }
    auto step = [&](int jj) {
#pragma unroll
      for (int r = 0; r < R - 1; ++r) xw[r] = xw[r + 1];
      xw[R - 1] = xb[jj + R - 1];
      float w, w1, w2;
      weights(jj - Mi, dist(jj - Mi), w, w1, w2);
      mac(xw, w, w1, w2, std::integral_constant<int, 0>());
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
      for (int r = 0; r < R - 1; ++r) xw[r] = xw[r + 1];
      xw[R - 1] = xb[W + R - 1];
      float w, w1, w2;
      weights(W - Mi, dist(W - Mi), w, w1, w2);
      mac(xw, w, w1, w2, std::integral_constant<int, 2>());
    }
  }

  // ---- carrier rotation (reading R10)
  const double g = carrier * (1.0 - beta);
  if (g != 0.0) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double psi = g * (double)(mt + r);
      acc[r] = cmul(acc[r], expm2pi(__double2float_rn(psi - rint(psi))));
    }
  }
  if constexpr (DIRECT) {
    float2 *yp = y + cur.pulse * n;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (mt + r < n) __stcs(yp + mt + r, acc[r]);
    return;
  }
  // ---- store: the warp's 32 x R outputs are contiguous (thread t owns [t R, t R + R)).  Lane 0's
  // previous bulk store must have finished reading the segment before it is overwritten.
  if (lane == 0) bulk_store_wait_read();
  __syncwarp();
#pragma unroll
  for (int r = 0; r < R; ++r) ob[lane * R + r] = acc[r];
  fence_proxy_async();  // generic-proxy writes -> visible to the bulk copy (async proxy)
  __syncwarp();
  if (lane == 0) {
    const int64_t mw = cur.m0 + (int64_t)(tid >> 5) * SEG;
    const int64_t valid = min((int64_t)SEG, n - mw);  // even: n and mw are even
    if (valid > 0) {
      bulk_store(y + cur.pulse * n + mw, ob, (unsigned)(valid * sizeof(float2)));
      bulk_commit();
    }
  }
}

}  // namespace dc
