// tile_fft.cuh -- persistent, prefetching tile kernels for the ionospheric stage (Eq. 15).
//
// Every regime is expressed as a stream of 8192-sample TILES, each processed by one CTA:
//   SMALL  rows = whole pulses (n <= 8192): forward FFT -> Eq. 15 phase -> inverse FFT
//   COLA   four-step pass A: [N1][C] column tile, forward N1-point DFTs, times w_n^(k1 t2)
//   ROWB   four-step pass B: [NB][N2] row tile, forward DFT -> phase -> inverse DFT, times w_n^(-k1 t2)
//   COLC   four-step pass C: [N1][C] column tile, inverse N1-point DFTs
// A CTA is persistent: while it computes tile i, the input of tile i + gridDim.x streams
// into a shared-memory staging buffer with cp.async (16-byte LDGSTS, L1-bypassing), so the
// HBM/L2 latency of the next tile overlaps this tile's FFT passes.  Twiddle tables are copied
// into shared memory once per CTA.  The first FFT pass reads the staging buffer, the
// exchanges between passes use a separate padded work buffer, the last pass stores straight
// from registers to global memory.
#pragma once
#include "doppler_tile.cuh"
#include "fft_engine.cuh"

namespace dc {

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16_zfill(void *smem_dst, const void *gsrc, bool valid) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gsrc), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit_() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

enum TileMode { MODE_SMALL = 0, MODE_COLA = 1, MODE_ROWB = 2, MODE_COLC = 3 };

// What the frequency-domain step does between the forward and inverse DFTs (bins X_k):
//   VAR_CORRECT   X_k e^{-i 2 pi nu_k}                 Eq. 15
//   VAR_DISTORT   X_k e^{+i 2 pi nu_k}                 Eq. 14 forward model
//   VAR_COMPRESS  X_k e^{-i 2 pi nu_k} T_k             Eq. 15 then the matched filter (reading R16);
//                                                      T = conj(R) of the reference (per pulse: table ref_idx[p])
//   VAR_REFERENCE store conj(X_k) to ref_out, no inverse (builds the T tables of VAR_COMPRESS; the FFT P/Q
//                 path's forward transform)
// Bin tables (T, ref_out) use the "row layout": bin k = k1 + N1 k2 at index k1 N2 + k2 (N1 = n / N2; natural
// order k for single-CTA pulses, N1 = 1).
enum RowVar { VAR_CORRECT = 0, VAR_DISTORT = 1, VAR_COMPRESS = 2, VAR_REFERENCE = 3 };

struct TileArgs {
  const float2 *src;  // tile input (pulse-major, pulse_stride apart)
  float2 *dst;        // tile output
  int64_t pulses;     // pulses in this launch
  int64_t pulse_stride;
  int64_t pulse_base;  // first pulse's index in pp[]
  int log2n;
  const PulseParams *pp;
  const float2 *twf, *twi;  // pass tables of the tile's FFT size (global; copied to smem)
  const float2 *twh, *twl;  // four-step outer twiddles (global; copied to smem)
  int H;
  double fs_over_n, fc;
  const float2 *ref;    // VAR_COMPRESS: T tables (row layout), n entries each
  const int *ref_idx;   // VAR_COMPRESS: per-pulse table index (indexed like pp), or null = table 0
  float2 *ref_out;      // VAR_REFERENCE: conj(X) per pulse (row layout), n entries each
  float2 *dop_y;        // fused dc_correct (DOPW > 0): Doppler output y[pulses][n]
  double dop_carrier;   // fused dc_correct: fc / fs (reading R10)
};

// Fused single-round-trip dc_correct for single-CTA pulses (NEXT-1; DOPW = compile-time Doppler W > 0):
// the Eq. 15 result of the tile's pulses lands in a zero-margined shared-memory buffer that aliases the
// work buffer, and the Doppler tile code (doppler_tile.cuh) resamples it straight from there -- x is
// read and y written once, 16 B/sample for both stages.  Margins of kCsPad zeros on each side hold the
// window's reach outside [0, n) (R12): W/2 + 1 below, W/2 + R + (n - 1)|beta - 1| above (W <= 64).
constexpr int kCsPad = 64;

// Shared-memory layout (float2 units): [staging ELEMS][work SMEM_ELEMS][twf][twi][twh][twl]
template <int P, int LOGE, int NB, bool ROW, int MODE>
struct TileCfg {
  using TL = Tile<P, (1 << LOGE), NB, ROW>;
  using PP = PassPlan<P, LOGE>;
  static constexpr int L = 1 << P;
  static constexpr int T = TL::T;
  // pass tables live in shared memory when small (four-step sizes); the regime-0 tables of
  // large pulses (~L entries per direction) stay in global memory (L1-cached)
  static constexpr int TWF_ALL = (MODE == MODE_COLC) ? 0 : PP::tw_off_fwd(PP::npass);
  static constexpr int TWI_ALL = (MODE == MODE_COLA) ? 0 : PP::tw_off_inv(PP::npass);
  static constexpr bool SMEM_TW = (TWF_ALL + TWI_ALL) * 8 <= 40 * 1024;
  static constexpr int TWF = SMEM_TW ? TWF_ALL : 0;
  static constexpr int TWI = SMEM_TW ? TWI_ALL : 0;
  static constexpr int TWF_PAD = (TWF + 1) & ~1;
  static constexpr int TWI_PAD = (TWI + 1) & ~1;
  static __host__ __device__ constexpr int outer_elems(int H, int log2n) {
    return (MODE == MODE_COLA || MODE == MODE_ROWB) ? ((1 << H) + (1 << (log2n - H))) : 0;
  }
  static __host__ __device__ constexpr size_t smem_bytes(int H, int log2n, bool fused = false) {
    return sizeof(float2) * ((size_t)TL::ELEMS + TL::SMEM_ELEMS + TWF_PAD + TWI_PAD + outer_elems(H, log2n) +
                             (fused ? (size_t)(T / 32) * kDopSeg : 0));
  }
  static constexpr int DSTRIDE = L + 2 * kCsPad;  // fused dc_correct: one zero-margined pulse
};

template <int P, int LOGE, int NB, bool ROW, int MODE, int VAR, int DOPW = 0, bool DSECOND = false>
__global__ void __launch_bounds__(TileCfg<P, LOGE, NB, ROW, MODE>::T, 1) tile_fft_kernel(const TileArgs a) {
  static_assert(DOPW == 0 || (MODE == MODE_SMALL && VAR == VAR_CORRECT && DOPW <= 64), "fused dc_correct");
  static_assert(DOPW == 0 || NB * TileCfg<P, LOGE, NB, ROW, MODE>::DSTRIDE <= TileCfg<P, LOGE, NB, ROW, MODE>::TL::SMEM_ELEMS,
                "the Doppler buffer aliases the work buffer");
  pdl_wait();  // programmatic dependent launch (dc_common.cuh); the trigger is implicit at exit
  using CFG = TileCfg<P, LOGE, NB, ROW, MODE>;
  using TL = typename CFG::TL;
  using PP = typename CFG::PP;
  constexpr int L = CFG::L;
  constexpr int E = 1 << LOGE;
  constexpr int T = CFG::T;
  constexpr int NP = PP::npass;
  constexpr bool FWD = (MODE != MODE_COLC);
  constexpr bool INVP = (MODE != MODE_COLA) && VAR != VAR_REFERENCE;
  constexpr bool DISTORT = (VAR == VAR_DISTORT);
  constexpr int R0 = 1 << (FWD ? PP::log_radix_fwd(0) : PP::log_radix_inv(0));
  extern __shared__ float4 smem4[];
  float2 *S = reinterpret_cast<float2 *>(smem4);
  float2 *Wk = S + TL::ELEMS;
  float2 *Tf = Wk + TL::SMEM_ELEMS;
  float2 *Ti = Tf + CFG::TWF_PAD;
  float2 *Th = Ti + CFG::TWI_PAD;
  const int H = a.H;
  float2 *Tl = Th + ((MODE == MODE_COLA || MODE == MODE_ROWB) ? (1 << (a.log2n - H)) : 0);
  float2 *Ob = Tl + ((MODE == MODE_COLA || MODE == MODE_ROWB) ? (1 << H) : 0);  // fused: output staging
  float2 *D = Wk;  // fused: zero-margined iono result, NB x DSTRIDE (aliases the work buffer)
  const int tid = threadIdx.x;

  // ---- geometry of the tile stream
  const int log2n = a.log2n;
  const int n = 1 << log2n;
  int64_t tiles_per_pulse;
  int n2 = 0;
  if constexpr (MODE == MODE_SMALL) {
    tiles_per_pulse = 1;  // (NB pulses per tile; see below)
  } else if constexpr (ROW) {
    tiles_per_pulse = (n >> P) / NB;  // rows k1 of N2 = L samples, NB per tile
  } else {
    n2 = n >> P;
    tiles_per_pulse = n2 / NB;  // column groups of NB columns
  }
  const int64_t total = (MODE == MODE_SMALL) ? (a.pulses + NB - 1) / NB : a.pulses * tiles_per_pulse;
  int64_t item = blockIdx.x;
  if (item >= total) return;

  // staging: issue the cp.async for tile `it` into S
  auto stage = [&](int64_t it) {
    if constexpr (MODE == MODE_SMALL) {
      const int64_t p0 = it * NB;
      const int64_t valid = min((int64_t)NB, a.pulses - p0) * L;  // samples of real pulses in the tile
      const float4 *g = reinterpret_cast<const float4 *>(a.src + p0 * L);
      float4 *s4 = reinterpret_cast<float4 *>(S);
      for (int i = tid; i < TL::ELEMS / 2; i += T) {
        const bool ok = 2 * (int64_t)i < valid;
        cp_async16_zfill(s4 + i, ok ? (const void *)(g + i) : (const void *)a.src, ok);
      }
    } else if constexpr (ROW) {
      const int64_t pulse = it / tiles_per_pulse;
      const int64_t r0 = (it - pulse * tiles_per_pulse) * NB;
      const float4 *g = reinterpret_cast<const float4 *>(a.src + pulse * a.pulse_stride + r0 * L);
      float4 *s4 = reinterpret_cast<float4 *>(S);
#pragma unroll 4
      for (int i = tid; i < TL::ELEMS / 2; i += T) cp_async16(s4 + i, g + i);
    } else {
      const int64_t pulse = it / tiles_per_pulse;
      const int64_t c0 = (it - pulse * tiles_per_pulse) * NB;
      const float2 *g = a.src + pulse * a.pulse_stride + c0;
      constexpr int V = NB / 2;  // float4 per row segment
      float4 *s4 = reinterpret_cast<float4 *>(S);
#pragma unroll 4
      for (int i = tid; i < L * V; i += T) {
        const int row = i / V, v = i - row * V;
        cp_async16(s4 + i, reinterpret_cast<const float4 *>(g + (int64_t)row * n2) + v);
      }
    }
  };
  stage(item);
  cp_async_commit_();

  // ---- tables into shared memory (once)
  for (int i = tid; i < CFG::TWF; i += T) Tf[i] = a.twf[i];
  for (int i = tid; i < CFG::TWI; i += T) Ti[i] = a.twi[i];
  if constexpr (MODE == MODE_COLA || MODE == MODE_ROWB) {
    for (int i = tid; i < (n >> H); i += T) Th[i] = a.twh[i];
    for (int i = tid; i < (1 << H); i += T) Tl[i] = a.twl[i];
  }
  const uint32_t nmask = (uint32_t)n - 1u;
  const uint32_t hmask = (1u << H) - 1u;

  for (; item < total; item += gridDim.x) {
    cp_async_wait_all();
    __syncthreads();
    // ---- first pass inputs from the staging buffer
    float2 v[E];
#pragma unroll
    for (int q = 0; q < E / R0; ++q) {
      int b, j;
      TL::template bmap<R0>(tid + q * T, b, j);
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int i = j + r * (L / R0);
        v[q * R0 + r] = ROW ? S[b * L + i] : S[i * NB + b];
      }
    }
    __syncthreads();  // staging buffer free: prefetch the next tile
    const int64_t nitem = item + gridDim.x;
    if (nitem < total) stage(nitem);
    cp_async_commit_();

    int64_t pulse, base;  // pulse of the tile; first row / column / pulse index
    if constexpr (MODE == MODE_SMALL) {
      pulse = item * NB;
      base = 0;
    } else {
      pulse = item / tiles_per_pulse;
      base = (item - pulse * tiles_per_pulse) * NB;
    }

    if constexpr (FWD) run_passes<TL, PP, 0, NP - 1, false>(v, Wk, tid, CFG::SMEM_TW ? Tf : a.twf);

    if constexpr (MODE == MODE_SMALL || MODE == MODE_ROWB) {
      // ---- frequency domain (Eq. 15): registers hold bins k2 = j + r L/RL of FFT b
      constexpr int RL = 1 << PP::log_radix_fwd(NP - 1);
      const float inv_n = (MODE == MODE_ROWB) ? 1.0f : 1.0f / (float)n;  // ROWB: 1/n applied in pass A
      const int P1 = log2n - P;
#pragma unroll
      for (int q = 0; q < E / RL; ++q) {
        int b, j;
        TL::template bmap<RL>(tid + q * T, b, j);
        int64_t p;
        int k1 = 0;
        if constexpr (MODE == MODE_SMALL) {
          p = pulse + b;
        } else {
          p = pulse;
          k1 = (int)base + b;
        }
        if constexpr (VAR == VAR_REFERENCE) {
          // conj(X_k) in the row layout (index k1 L + k2); ROWB undoes pass A's 1/n (exact: a power of two)
          const float sc = (MODE == MODE_ROWB) ? (float)n : 1.0f;
          if (p < a.pulses) {
#pragma unroll
            for (int r = 0; r < RL; ++r) {
              const int k2 = j + r * (L / RL);
              const float2 x = v[q * RL + r];
              a.ref_out[p * (int64_t)n + (int64_t)k1 * L + k2] = make_float2(x.x * sc, -x.y * sc);
            }
          }
          continue;
        }
        const double nu_coef = (p < a.pulses) ? a.pp[a.pulse_base + p].nu_coef : 0.0;
        const float2 *tab = nullptr;
        if constexpr (VAR == VAR_COMPRESS)
          tab = a.ref + ((a.ref_idx && p < a.pulses) ? (int64_t)a.ref_idx[a.pulse_base + p] * n : 0) + (int64_t)k1 * L;
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          const int k2 = j + r * (L / RL);
          const int k = (MODE == MODE_SMALL) ? k2 : (k1 + (k2 << P1));
          const int kk = (k >= n / 2) ? k - n : k;
          const double f = a.fc + a.fs_over_n * (double)kk;
          float2 m = make_float2(inv_n, 0.f);
          if (f > 0.0 && nu_coef != 0.0) {
            const double nu = nu_coef * drcp(f);
            float rf = __double2float_rn(nu - rint(nu));
            if (fabs(nu) >= (double)kPhaseExactCycles)  // huge |nu|: the oracle's binary64 operations
              rf = phase_frac_exact(a.pp[a.pulse_base + p].k2, a.fc, a.fs_over_n, kk);
            const float2 w = expm2pi(DISTORT ? -rf : rf);
            m = make_float2(w.x * inv_n, w.y * inv_n);
          }
          if constexpr (VAR == VAR_COMPRESS) m = cmul(m, (p < a.pulses) ? tab[k2] : make_float2(0.f, 0.f));
          v[q * RL + r] = cmul(v[q * RL + r], m);
        }
      }
      if constexpr (VAR == VAR_REFERENCE) continue;
    }

    if constexpr (INVP) run_passes<TL, PP, 0, NP - 1, true>(v, Wk, tid, CFG::SMEM_TW ? Ti : a.twi);

    // ---- last pass outputs straight to global memory (fused dc_correct: to the Doppler buffer)
    constexpr int RO = 1 << (INVP ? PP::log_radix_inv(NP - 1) : PP::log_radix_fwd(NP - 1));
    if constexpr (DOPW > 0) __syncthreads();  // every thread has loaded its last-pass inputs from Wk = D
#pragma unroll
    for (int q = 0; q < E / RO; ++q) {
      int b, j;
      TL::template bmap<RO>(tid + q * T, b, j);
#pragma unroll
      for (int r = 0; r < RO; ++r) {
        const int i = j + r * (L / RO);  // output index within FFT b
        float2 val = v[q * RO + r];
        if constexpr (MODE == MODE_SMALL && DOPW > 0) {
          D[b * CFG::DSTRIDE + kCsPad + i] = val;
        } else if constexpr (MODE == MODE_SMALL) {
          const int64_t p = pulse + b;
          if (p < a.pulses) __stcs(a.dst + p * L + i, val);
        } else if constexpr (MODE == MODE_ROWB) {
          const uint32_t k1 = (uint32_t)base + b;
          const uint32_t m = (k1 * (uint32_t)i) & nmask;
          val = cmulc(val, cmul(Th[m >> H], Tl[m & hmask]));
          __stcg(a.dst + pulse * a.pulse_stride + (int64_t)k1 * L + i, val);
        } else if constexpr (MODE == MODE_COLA) {
          const uint32_t t2 = (uint32_t)base + b;
          const uint32_t m = ((uint32_t)i * t2) & nmask;
          val = cscale(cmul(val, cmul(Th[m >> H], Tl[m & hmask])), 1.0f / (float)n);  // 1/n (R6) folded here
          __stcg(a.dst + pulse * a.pulse_stride + (int64_t)i * n2 + t2, val);
        } else {
          __stcg(a.dst + pulse * a.pulse_stride + (int64_t)i * n2 + base + b, val);
        }
      }
    }
    if constexpr (DOPW > 0) {
      // ---- Doppler (Eq. 16 windowed, D1-D4) of the tile's pulses straight from shared memory
      for (int e = tid; e < NB * 2 * kCsPad; e += T) {
        const int b = e / (2 * kCsPad), j = e - b * 2 * kCsPad;
        D[b * CFG::DSTRIDE + (j < kCsPad ? j : L + j)] = make_float2(0.f, 0.f);
      }
      __syncthreads();
      float2 *obw = Ob + (tid >> 5) * kDopSeg;
      for (int b = 0; b < NB; ++b) {
        const int64_t p = pulse + b;
        if (p >= a.pulses) break;
        DopTile cur;
        cur.pulse = p;
        cur.Bcta = -kCsPad;
        cur.beta = a.pp[a.pulse_base + p].beta;
        cur.span = CFG::DSTRIDE;  // the zero-margined pulse
        cur.pad0 = 0;
        cur.pad1 = 0;
        for (int m0 = 0; m0 < L; m0 += T * kDopR) {
          cur.m0 = m0;
          if (m0 + (tid >> 5) * kDopSeg < L)  // warps wholly past the pulse end skip
            dop_tile_compute<DSECOND, DOPW, 0>(D + b * CFG::DSTRIDE, cur, DOPW, obw, a.dop_y, L, a.dop_carrier);
        }
      }
      __syncthreads();  // D is the next item's exchange buffer
    }
  }
  cp_async_wait_all();
  if constexpr (DOPW > 0) {
    if ((tid & 31) == 0) bulk_store_wait_all();  // the warp's last output segment has left shared memory
  }
}

}  // namespace dc
