// doppler_kernel.cu -- windowed Whittaker-Shannon (sinc) resampling onto t/alpha.
//
// Method (Eq. 16, restricted to W samples: Alg. 1 P:L510-528,
// window P:L533; correction direction per Eq. 13):
//   t_m = m beta (beta = 1/alpha, binary64)
//   y_m = exp(-i 2 pi fc (1 - beta) m / fs) * sum_{k = K_m}^{K_m + W - 1} [0 <= k < n] x_k sinc(t_m - k),
//   K_m = floor(t_m - W/2) + 1   (window {k : -W/2 < k - t_m <= W/2}, R9)
//
// B200 design:
//   * A persistent CTA (8 warps, 2 per SM) owns tiles of M = 256 R consecutive outputs of one
//     pulse.  The input span a tile needs (~M beta + W + R samples) is staged into shared memory by
//     the TMA engine (2-D tensor map {n, pulses}, hardware zero fill outside [0, n): R12) one tile
//     ahead into one of three buffers with full/empty mbarriers, so HBM latency hides behind the
//     taps and warps drift up to a tile apart without a CTA barrier.
//   * A thread owns R = 11 consecutive outputs (odd: lanes' windows start R samples apart and land
//     on distinct banks).  Their windows slide by one sample per output except where the position
//     wraps; all R windows lie inside a union of W + 1 taps, streamed once through a register window
//     (one LDS per tap, reused by all R outputs); each output masks the one edge tap it does not own.
//     The complex x real MACs are FFMA2 (packed f32x2).  Each warp's 32 R contiguous outputs leave
//     as one bulk async copy (shared -> global) issued by lane 0.
//   * Taps are evaluated on the fly in FP32 (no LUT; LUT quantisation breaks 1e-5 parity):
//     per thread, per tap, w = sinc(v - jj) and w' = sinc'(v - jj) at the thread's reference
//     position v (exact binary64 position, reduced to [-1/2, 1/2] before the FP32 cast so
//     the centre tap keeps full relative precision); each output then uses
//     h = w + w' delta_r (+ w''/2 delta_r^2), delta_r = (r - r_ref)(beta - 1) exactly.
//   * The slow path (|beta - 1| too large for the union/Taylor scheme) evaluates every
//     output directly (Alg. 1 structure).
#include "doppler_tile.cuh"
#include "tma_host.h"

namespace dc {

// Persistent pipeline over kDopBufs input buffers: buffer b holds local tiles b, b + kDopBufs, ...; each
// has a `full` transaction mbarrier (TMA bytes) and a release counter.  A warp that has finished reading
// buffer b counts itself out; the LAST warp to do so restages the buffer with tile i + kDopBufs right
// away, so the load is issued as early as possible (kDopBufs - 1 tiles of compute ahead of its first
// consumer) and no warp ever blocks on a slower one -- warps run up to kDopBufs - 1 tiles apart with no
// CTA-wide barrier.  (The previous design had thread 0 wait on an `empty` barrier before staging tile
// i + 1, which stalled warp 0 -- and with it the prefetch -- behind the slowest warp.)  The tile geometry
// reaches the consumers through the TMA engine too (from a per-CTA global slot), counted by the same
// `full` barrier as the data.
// WT > 0: the tap count W is a compile-time constant (fully unrolled tap loop); WT = 0: runtime W.
// T threads per CTA at 128 registers: 2 CTAs per SM for T = 256, 1 for T = 512, 4 for T = 128
template <bool SECOND, int WT, int TAPER, int T>
__global__ void __launch_bounds__(T, 65536 / (T * 128))
    doppler_pipe_kernel(const __grid_constant__ CUtensorMap xmap, float2 *__restrict__ y, int64_t n, int W_rt,
                        const PulseParams *__restrict__ pp, int64_t pulse_base, double carrier, int64_t pulses,
                        int buf_elems, const __grid_constant__ TaperCoef tc, DopTile *__restrict__ gdesc,
                        const __grid_constant__ CUtensorMap dmap) {
  pdl_wait();  // programmatic dependent launch (dc_common.cuh); the trigger is implicit at exit
  constexpr int R = dop_r_pipe(WT, T), M = T * R, SEG = 32 * R;
  extern __shared__ __align__(1024) float4 xs4[];
  float2 *xs = reinterpret_cast<float2 *>(xs4);                     // kDopBufs x buf_elems input spans
  float2 *ob = xs + kDopBufs * buf_elems;                            // M output staging (per warp)
  // geometry of the tile in each buffer: 128-byte slots (TMA destinations are 128-byte aligned)
  DopTile *tiles = reinterpret_cast<DopTile *>(ob + M);
  auto dslot = [&](int b) { return reinterpret_cast<DopTile *>(reinterpret_cast<char *>(tiles) + 128 * b); };
  uint64_t *full = reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(tiles) + 128 * kDopBufs);  // TMA completion
  uint32_t *released = reinterpret_cast<uint32_t *>(full + kDopBufs);  // warps done with each buffer
  const int W = (WT > 0) ? WT : W_rt;
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t tiles_per_pulse = (uint32_t)((n + M - 1) / M);
  const uint32_t total = (uint32_t)pulses * tiles_per_pulse;
  if (blockIdx.x >= total) return;
  const uint32_t my_tiles = (total - blockIdx.x + gridDim.x - 1) / gridDim.x;
  auto produce = [&](uint32_t i) {  // one thread: stage local tile i into buffer i % kDopBufs (free)
    const int b = (int)(i % kDopBufs);
    const uint32_t it = blockIdx.x + i * gridDim.x;
    const DopTile t = dop_tile<R, T>(it, tiles_per_pulse, W, pp[pulse_base + dop_pulse(it, tiles_per_pulse)].beta);
#ifdef DC_DEBUG_CHECKS
    if (dop_nbox(t) * kDopBox > buf_elems) __trap();  // the staged span fits its buffer
#endif
    const int slot = (int)blockIdx.x * kDopBufs + b;
    dop_stage_tma(xs + b * buf_elems, t, &xmap, &full[b], dslot(b), gdesc + slot, &dmap, slot);
  };
  if (tid == 0) {
    for (int b = 0; b < kDopBufs; ++b) {
      mbar_init(&full[b], 1);
      released[b] = 0u;
    }
    mbar_fence_init();
    for (uint32_t i = 0; i < (uint32_t)kDopBufs && i < my_tiles; ++i) produce(i);
  }
  __syncthreads();
  float2 *obw = ob + (tid >> 5) * SEG;
  for (uint32_t i = 0; i < my_tiles; ++i) {
    const int b = (int)(i % kDopBufs);
    mbar_wait(&full[b], (i / kDopBufs) & 1u);
    const DopTile cur = *dslot(b);
    // a pulse's last tile is ragged: warps whose outputs all lie past n skip it (their issue slots go to
    // the other CTA of the SM), so short pulses waste at most one warp segment instead of a tile
    if (cur.m0 + (int64_t)(tid >> 5) * SEG < n)
      dop_tile_compute<SECOND, WT, TAPER, R>(xs + b * buf_elems, cur, W, obw, y, n, carrier, &tc);
    __syncwarp();
    if (lane == 0) {
      // this warp's reads of buffer b are done (release); the last warp out acquires and restages it.
      // Nobody else touches released[b] until tile i + kDopBufs -- the one staged here -- is consumed.
      __threadfence_block();
      if (atomicAdd(&released[b], 1u) == (uint32_t)(T / 32 - 1)) {
        released[b] = 0u;
        __threadfence_block();
        if (i + kDopBufs < my_tiles) produce(i + kDopBufs);
      }
    }
  }
  if (lane == 0) bulk_store_wait_all();  // the warp's last output segment has left shared memory
}

// Exact-tap, one-output-per-thread path (Alg. 1 structure) for any alpha.
// Used when |beta - 1| is too large for the union-window / Taylor scheme, and for alpha == 1
// pulses handled by the generic path it returns x exactly (u == 0 case).
template <int TAPER>
__global__ void __launch_bounds__(256) doppler_exact_kernel(const float2 *__restrict__ x, float2 *__restrict__ y,
                                                           int64_t n, int W, const PulseParams *__restrict__ pp,
                                                           int64_t pulse_base, double carrier,
                                                           const __grid_constant__ TaperCoef tcoef) {
  pdl_wait();  // programmatic dependent launch; the trigger is implicit at exit
  const int64_t pulse = blockIdx.y;
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  const float2 *xp = x + pulse * n;
  const double beta = pp[pulse_base + pulse].beta;
  const double t = __dmul_rn((double)m, beta);  // fl(m beta), fl(t - W/2): the oracle's roundings (R9, R14)
  const int64_t K = (int64_t)floor(__dsub_rn(t, 0.5 * (double)W)) + 1;
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
      float h = s / d;
      if constexpr (TAPER > 0) {
        float Kt, dKt;
        taper_eval<TAPER>(tcoef, d, Kt, dKt);
        h *= Kt;
      }
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

template <bool SECOND, int WT, int TAPER, int T>
static cudaError_t launch_pipe(const DopplerArgs &a) {
  constexpr int R = dop_r_pipe(WT, T), M = T * R;
  const int64_t tiles = (a.n + M - 1) / M * a.pulses;
  // staged span <= M * max(beta) + W + R + 6 samples (fast path: |beta - 1| <= 4.4e-4)
  const int span = (int)(M * (1.0 + kDopMaxDrift)) + a.taps + R + 16;
  const int buf = (span + kDopBox - 1) / kDopBox * kDopBox;  // whole TMA boxes
  const size_t smem = sizeof(float2) * (kDopBufs * (size_t)buf + M) + kDopBufs * (128 + sizeof(uint64_t) + 4) + 1024;
  CUtensorMap xmap;
  {
    const uint64_t dims[2] = {(uint64_t)a.n, (uint64_t)a.pulses};
    const uint64_t strides[1] = {(uint64_t)a.n * sizeof(float2)};
    const uint32_t box[2] = {(uint32_t)kDopBox, 1u};
    if (!encode_tile_map(&xmap, a.x, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
  }
  auto kern = doppler_pipe_kernel<SECOND, WT, TAPER, T>;
  LaunchShape ls;
  cudaError_t e = launch_shape(kern, T, smem, &ls);
  if (e != cudaSuccess) return e;
  const int sms = ls.sms, per_sm = ls.per_sm;
  int64_t grid = std::min<int64_t>(tiles, (int64_t)sms * std::max(per_sm, 1));
  if (a.grid_cap > 0) grid = std::min<int64_t>(grid, a.grid_cap);
#ifdef DC_DOP_GRID_CAP
  grid = std::min<int64_t>(grid, DC_DOP_GRID_CAP);  // tuning builds only
#endif
  grid = std::min<int64_t>(grid, kDopMaxCtas);
  static_assert(kDopBufs <= 4 && sizeof(DopTile) == 48, "kDopDescBytes sizing");
  CUtensorMap dmap;  // the per-CTA geometry slots: {6 x 8 bytes, slot}, one 48-byte box per tile
  {
    const uint64_t dims[2] = {6, (uint64_t)kDopMaxCtas * 4};
    const uint64_t strides[1] = {sizeof(DopTile)};
    const uint32_t box[2] = {6u, 1u};
    if (!encode_tile_map(&dmap, a.desc, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
  }
  return launch_pdl(kern, dim3((unsigned)grid), dim3(T), smem, a.stream, xmap, a.y, a.n, a.taps, a.pp, a.pulse_base,
                    a.carrier_cycles_per_sample, a.pulses, buf, a.tc, reinterpret_cast<DopTile *>(a.desc), dmap);
}

// CTA size per configuration (measured, W = 32 at 2^20 / 4096: T = 256 191.8 / 127.8, T = 512 201.0 / 132.8,
// T = 128 187.5 / 169.2 GS/s): short pulses (n < 2^16, a few tiles per pulse) take 128-thread CTAs (4 per
// SM: finer tiles, less quantisation); long pulses 512 (one 16-warp CTA per SM: one set of staging buffers
// and fewer, longer tiles), except W <= 16 (256: 303 vs 286 GS/s) and the tapered windows (256).
#ifndef DC_DOP_FORCE_T
#define DC_DOP_FORCE_T 0  // tuning builds only: force the CTA size (128 / 256 / 512)
#endif
template <bool SECOND, int WT, int TAPER>
static cudaError_t launch_pipe_t(const DopplerArgs &a) {
  if constexpr (DC_DOP_FORCE_T > 0) return launch_pipe<SECOND, WT, TAPER, DC_DOP_FORCE_T>(a);
  if constexpr (TAPER == 0) {
    if (a.n < (1 << 16)) return launch_pipe<SECOND, WT, TAPER, 128>(a);
    if constexpr (WT == 0 || WT > 16) {
      return launch_pipe<SECOND, WT, TAPER, 512>(a);
    } else {
      return launch_pipe<SECOND, WT, TAPER, 256>(a);
    }
  } else {
    return launch_pipe<SECOND, WT, TAPER, 256>(a);
  }
}

template <bool SECOND, int TAPER = 0>
static cudaError_t launch_pipe_w(const DopplerArgs &a) {
  switch (a.taps) {  // compile-time tap counts of the benchmark / sweep configurations
    case 8: return launch_pipe_t<SECOND, 8, TAPER>(a);
    case 16: return launch_pipe_t<SECOND, 16, TAPER>(a);
    case 25: return launch_pipe_t<SECOND, 25, TAPER>(a);
    case 32: return launch_pipe_t<SECOND, 32, TAPER>(a);
    case 64: return launch_pipe_t<SECOND, 64, TAPER>(a);
    case 128: return launch_pipe_t<SECOND, 128, TAPER>(a);
    default: return launch_pipe_t<SECOND, 0, TAPER>(a);
  }
}

static cudaError_t launch_doppler_fast(const DopplerArgs &a, bool second) {
  if (a.taper) {
    if (second) return cudaErrorInvalidValue;
    if (a.taper_terms == kTaperHann) return launch_pipe_w<false, kTaperHann>(a);
    return a.taper_terms <= 17 ? launch_pipe_w<false, 17>(a) : launch_pipe_w<false, kTaperTerms>(a);
  }
  return second ? launch_pipe_w<true>(a) : launch_pipe_w<false>(a);
}

static cudaError_t launch_doppler_exact(const DopplerArgs &a) {
  dim3 grid((unsigned)((a.n + 255) / 256), (unsigned)a.pulses);
  auto kern = !a.taper                         ? doppler_exact_kernel<0>
              : a.taper_terms == kTaperHann ? doppler_exact_kernel<kTaperHann>
              : a.taper_terms <= 17         ? doppler_exact_kernel<17>
                                            : doppler_exact_kernel<kTaperTerms>;
  return launch_pdl(kern, grid, dim3(256), 0, a.stream, a.x, a.y, a.n, a.taps, a.pp, a.pulse_base,
                    a.carrier_cycles_per_sample, a.tc);
}

// Path choice from the largest |beta - 1| among the launched pulses (host-known):
//   drift = |beta - 1| * (R + 1) / 2 is the largest Taylor step delta of the fast kernels (R = 13, the
//   largest R any of them uses for W <= 32, so the choice holds for every kernel that may run).
//   first order  if drift <= 5e-4 (truncation delta^2 / 2 |w''| <= 4.1e-7 per tap weight; summed over the
//                window's sum |w''| ~ 25 it stays below 1e-6 of the output rms -- round 2 raised the
//                bound from 2e-4, which sent the C4 train's largest |v| ~ 5 km/s to the second order)
//   second order if drift <= 2e-3 (truncation <= 1.3 delta^3 <= 1.1e-8)
//   exact taps otherwise.
// The tapered weights have the first-order path only (h'' of sinc K is not formed): second-order
// drifts take the exact path.
int doppler_path(double max_abs_beta_m1, bool taper, int W) {
  const int R = (W == 128) ? dop_r(128) : (W == 64 ? kDopR : 13);  // the largest R of the kernels for this W
  const double drift = max_abs_beta_m1 * (R / 2 + 0.5);
#ifndef DC_DOP_FAST1
#define DC_DOP_FAST1 5.0e-4
#endif
  if (drift <= DC_DOP_FAST1) return 1;
  if (drift <= kDopMaxDrift && !taper) return 2;
  return 0;
}

cudaError_t launch_doppler(const DopplerArgs &a, double max_abs_beta_m1) {
  const int path = doppler_path(max_abs_beta_m1, a.taper, a.taps);
  if (path == 0) return launch_doppler_exact(a);
  return launch_doppler_fast(a, path == 2);
}

}  // namespace dc
