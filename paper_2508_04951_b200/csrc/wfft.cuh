// wfft.cuh -- warp-level 1024-point FFT kernels for the four-step passes of n = 2^17..2^21
// (and whole 1024-sample pulses).
//
// One warp owns one 1024-point FFT: lane j holds the 32 samples x[j + 32 r] in registers,
// pass 1 is a radix-32 DFT over r (Stockham NS = 1, outputs to j*32 + s), a warp-private
// padded shared-memory exchange (stride 33: conflict-free) and pass 2 a twiddled radix-32 DFT
// over the other index; the result X[j + 32 s] is in natural order with the same register
// ownership that the first inverse pass needs, so forward FFT -> Eq. 15 phase -> inverse FFT
// never leave the warp.  Warps synchronise only with __syncwarp(), so the 8 warps of a CTA run
// out of phase and hide each other's shared-memory and FP64 latency (the barrier-lockstep
// CTA design of tile_fft.cuh left ~2 warps per scheduler stalled in the same phase).
#pragma once
#include "tile_fft.cuh"
#include "tma.cuh"

namespace dc {

constexpr int kWW = 8;  // warps per CTA
constexpr int kWPad = 1058;  // padded exchange buffer (index i + (i >> 5) < 1056; 2*1058 = 4 mod 16 spreads the CTA store reads)

__device__ __forceinline__ int wpad(int i) { return i + (i >> 5); }

// twiddle of pass 2: w1024^(k r), table layout [r/2][k] float4 (k = lane): conflict-free
template <bool INV>
__device__ __forceinline__ void wfft1024(float2 (&v)[32], float2 *__restrict__ wk, const float4 *__restrict__ tw,
                                         int lane) {
  DFT<32, INV>::run(v);
  __syncwarp();
#pragma unroll
  for (int s = 0; s < 32; ++s) wk[wpad(lane * 32 + s)] = v[s];
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = wk[wpad(lane + 32 * r)];
#pragma unroll
  for (int h = 0; h < 16; ++h) {
    const float4 p = tw[h * 32 + lane];
    if (h > 0) v[2 * h] = INV ? cmulc(v[2 * h], make_float2(p.x, p.y)) : cmul(v[2 * h], make_float2(p.x, p.y));
    v[2 * h + 1] = INV ? cmulc(v[2 * h + 1], make_float2(p.z, p.w)) : cmul(v[2 * h + 1], make_float2(p.z, p.w));
  }
  DFT<32, INV>::run(v);
}

// w_n^m = exp(-2 pi i m / n) for 0 <= m < n = 2^log2n via sincospif of the exact FP32 argument
// 2 m / n (m < 2^24 is exact in FP32): ~1 ulp, no table, no shared-memory bank conflicts.
__device__ __forceinline__ float2 twn(uint32_t m, int log2n) {
  const float x = __uint2float_rn(m) * __int_as_float((127 + 1 - log2n) << 23);  // 2 m / n
  float sn, cs;
  sincospif(x, &sn, &cs);
  return make_float2(cs, -sn);
}

// Rare path of the Eq. 15 phase (bins with |nu| >= kPhaseExactCycles, i.e. within ~1 MHz of DC at
// 100-200 TECU): bit s of `ex` marks element lane + 32 s of this lane, which the main loop rotated by
// the FP32-pair phase; it is re-rotated by (exact binary64 phase - FP32-pair phase).  The warp's
// samples go through its exchange buffer (each lane touches only its own slots) so that the
// out-of-line binary64 routine is called from a loop with no sample registers live -- 32 inline
// call sites in the phase loop cost the row pass 2.4x (measured, round 2).
template <bool DISTORT, class GOF, class KB>
__device__ __forceinline__ void phase_exact_fixup_g(float2 (&v)[32], uint32_t ex, float2 *__restrict__ wk, int lane,
                                                    const PulseParams &pr, GOF g_of, KB kb_of, long long n,
                                                    double fc, double fs_over_n) {
  if (!__any_sync(0xffffffffu, ex != 0u)) return;
  __syncwarp();
#pragma unroll
  for (int s = 0; s < 32; ++s) wk[wpad(lane + 32 * s)] = v[s];
#pragma unroll 1
  while (ex != 0u) {
    const int s = __ffs(ex) - 1;
    ex &= ex - 1u;
    const float2 g = g_of(s);
    const long long k = kb_of(s);
    float d = phase_frac_exact(pr.k2, fc, fs_over_n, k >= n / 2 ? k - n : k) - phase_frac(pr.nu_hi, pr.nu_lo, g);
    d -= rintf(d);
    float2 &e = wk[wpad(lane + 32 * s)];
    e = cmul(e, expm2pi(DISTORT ? -d : d));
  }
  __syncwarp();
#pragma unroll
  for (int s = 0; s < 32; ++s) v[s] = wk[wpad(lane + 32 * s)];
}

// the common case: element s of this lane reads its g entry at grow[lane + 32 s]
template <bool DISTORT, class KB>
__device__ __forceinline__ void phase_exact_fixup(float2 (&v)[32], uint32_t ex, float2 *__restrict__ wk, int lane,
                                                  const PulseParams &pr, const float2 *grow, KB kb_of, long long n,
                                                  double fc, double fs_over_n) {
  phase_exact_fixup_g<DISTORT>(v, ex, wk, lane, pr, [&](int s) { return grow[lane + 32 * s]; }, kb_of, n, fc, fs_over_n);
}

struct WarpArgs {
  const float2 *src;
  float2 *dst;
  int64_t pulses;
  int64_t pulse_stride;
  int64_t pulse_base;
  int log2n;
  const PulseParams *pp;
  const float2 *tw;  // 1024-entry pass-2 table, float4 [r/2][k] layout
  const float2 *twh, *twl;
  int H;
  double fs_over_n, fc;
  float scale;  // pass A: 1/n (inverse-transform normalisation folded into the outer twiddle)
  const float2 *gtab;  // per-bin 1/f_k FP32 pairs, row layout [k1][k2] (MODE_SMALL: natural order)
  const float2 *ref;   // VAR_COMPRESS: T = conj(R_k) tables (n entries each, same layout as gtab)
  const int *ref_idx;  // VAR_COMPRESS: per-pulse table index (indexed like pp), or null = table 0
  float2 *ref_out;     // VAR_REFERENCE: conj(X_k) per pulse (n entries each, same layout as gtab)
  int outer_c;         // the conj outer twiddle of pass B is applied by pass C on load (n = 2^20: both warp-level)
};

// (RowVar: what the row kernel does between its forward and inverse DFTs -- tile_fft.cuh)

// MODE_ROWB: four-step pass B on rows k1 of Z (N2 = 1024).  MODE_SMALL: whole pulses of 1024.
// NW warps per CTA.  STAGE: each warp prefetches its next row into a private shared buffer with
// cp.async; !STAGE: rows are loaded straight into registers.  Default NW = 12 (168 registers, Z row
// staged, g row read from L2): +14% over NW = 8 (255 registers, Z and g staged); NW = 16 spills.
#ifndef DC_ROW_NW
#define DC_ROW_NW 12
#endif
template <int NW, bool STAGE>
struct RowCfg {
  // staging per warp (float2): Z row, plus the g row when it fits (NW <= 8; NW = 12 reads g from L2)
  static constexpr bool SG = STAGE && NW <= 8;
  static constexpr int STG = STAGE ? (SG ? 2048 : 1024) : 0;
  static __host__ __device__ constexpr size_t elems(bool outer, int log2n, int H) {
    // (outer twiddles come from twn(), so no outer-twiddle table is staged)
    return (void)outer, (void)log2n, (void)H, (size_t)NW * (STG + kWPad + 32) + 1024;
  }
};

template <int MODE, int VAR, int NW, bool STAGE>
__global__ void __launch_bounds__(NW * 32, 1) warp_row_kernel(const WarpArgs a) {
  pdl_wait();  // programmatic dependent launch (dc_common.cuh); the trigger is implicit at exit
  using CFG = RowCfg<NW, STAGE>;
  constexpr bool SG = CFG::SG;
  extern __shared__ float4 smem4[];
  float2 *sm = reinterpret_cast<float2 *>(smem4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float2 *stg = sm + warp * CFG::STG;                        // per-warp staging (8 KB) if STAGE
  float2 *wk = sm + NW * CFG::STG + warp * kWPad;            // per-warp exchange
  float2 *Pw = sm + NW * (CFG::STG + kWPad) + warp * 32;     // per-warp outer-twiddle powers
  float4 *Tw = reinterpret_cast<float4 *>(sm + NW * (CFG::STG + kWPad + 32));
  const int log2n = a.log2n;
  const int n = 1 << log2n;
  const uint32_t nmask = (uint32_t)n - 1u;
  const int P1 = log2n - 10;
  const int64_t rows_per_pulse = (MODE == MODE_ROWB) ? ((int64_t)1 << P1) : 1;
  const int64_t total = a.pulses * rows_per_pulse;
  const int64_t gw = (int64_t)blockIdx.x * NW + warp, G = (int64_t)gridDim.x * NW;

  // tables (once per CTA)
  for (int i = threadIdx.x; i < 512; i += NW * 32) Tw[i] = reinterpret_cast<const float4 *>(a.tw)[i];
  auto row_ptr = [&](const float2 *base, int64_t it) {
    const int64_t p = it / rows_per_pulse, k1 = it - p * rows_per_pulse;
    return base + p * a.pulse_stride + k1 * 1024;
  };
  // two cp.async groups per row: the Z row (needed first) and the g row (needed at the phase)
  auto stage_z = [&](int64_t it) {
    const float4 *g = reinterpret_cast<const float4 *>(row_ptr(a.src, it));
    float4 *s4 = reinterpret_cast<float4 *>(stg);
#pragma unroll
    for (int i = 0; i < 16; ++i) cp_async16(s4 + lane + 32 * i, g + lane + 32 * i);
  };
  auto stage_g = [&](int64_t it) {
    const int64_t k1 = it - (it / rows_per_pulse) * rows_per_pulse;
    const float4 *gt = reinterpret_cast<const float4 *>(a.gtab + k1 * 1024);
    float4 *s4 = reinterpret_cast<float4 *>(stg);
#pragma unroll
    for (int i = 0; i < 16; ++i) cp_async16(s4 + 512 + lane + 32 * i, gt + lane + 32 * i);
  };
  int64_t it = gw;
  if constexpr (STAGE) {
    if (it < total) stage_z(it);
    cp_async_commit_();
    if constexpr (SG) {
      if (it < total) stage_g(it);
      cp_async_commit_();
    }
  }
  __syncthreads();  // tables visible

  for (; it < total; it += G) {
    float2 v[32];
    if constexpr (STAGE) {
      if constexpr (SG) {
        cp_async_wait_1();  // Z row of this item landed (its g row may still be in flight)
      } else {
        cp_async_wait_all();  // the only group in flight is this item's Z row
      }
      __syncwarp();
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = stg[lane + 32 * r];
      __syncwarp();  // Z staging consumed: prefetch the next Z row now
      if (it + G < total) stage_z(it + G);
      cp_async_commit_();
    } else {
      const float2 *g = row_ptr(a.src, it);
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = (MODE == MODE_ROWB) ? __ldcg(g + lane + 32 * r) : __ldcs(g + lane + 32 * r);
    }
    const int64_t p = it / rows_per_pulse;
    const uint32_t k1 = (uint32_t)(it - p * rows_per_pulse);

    wfft1024<false>(v, wk, Tw, lane);

    // ---- Eq. 15 phase of bins k = k1 + N1 k2, k2 = lane + 32 s (MODE_SMALL: k = k2):
    // nu = nu_coef * g_k with g_k = 1/f_k from the plan table (0 for f_k <= 0, R3), FP32-pair math
    {
      const float inv_n = (MODE == MODE_ROWB) ? 1.0f : 1.0f / (float)n;  // ROWB: 1/n applied in pass A
      if constexpr (SG) {
        cp_async_wait_1();  // this item's g row landed (the next Z row may still be in flight)
        __syncwarp();
      }
      if constexpr (VAR == VAR_REFERENCE) {
        // reference spectrum: X_k of the zero-padded reference pulse, stored conjugated; ROWB undoes
        // the 1/n that pass A folded in (exact: a power of two)
        const float sc = (MODE == MODE_ROWB) ? (float)n : 1.0f;
        float2 *ro = a.ref_out + p * (int64_t)n + (int64_t)k1 * 1024;
#pragma unroll
        for (int s = 0; s < 32; ++s) ro[lane + 32 * s] = make_float2(v[s].x * sc, -v[s].y * sc);
      } else {
        const PulseParams pr = a.pp[a.pulse_base + p];
        const float2 *grow = SG ? (stg + 1024) : (a.gtab + (int64_t)k1 * 1024);
        float2 rc[VAR == VAR_COMPRESS ? 32 : 1];
        if constexpr (VAR == VAR_COMPRESS) {
          const float2 *rtab = a.ref + (a.ref_idx ? (int64_t)a.ref_idx[a.pulse_base + p] * n : 0) + (int64_t)k1 * 1024;
#pragma unroll
          for (int s = 0; s < 32; ++s) rc[s] = __ldg(rtab + lane + 32 * s);
        }
        uint32_t ex = 0u;  // elements needing the exact binary64 phase (phase_exact_fixup)
#pragma unroll
        for (int s = 0; s < 32; ++s) {
          if (!SG && s % 8 == 0) asm volatile("" ::: "memory");  // table loads in chunks of 8 (registers)
          const float2 g = SG ? grow[lane + 32 * s] : __ldg(grow + lane + 32 * s);
          const float rf = phase_frac(pr.nu_hi, pr.nu_lo, g);
          ex |= phase_needs_exact(pr.nu_hi, g) ? (1u << s) : 0u;
          const float2 w = expm2pi((VAR == VAR_DISTORT) ? -rf : rf);
          v[s] = cmul(v[s], make_float2(w.x * inv_n, w.y * inv_n));
          if constexpr (VAR == VAR_COMPRESS) v[s] = cmul(v[s], rc[s]);
        }
        phase_exact_fixup<VAR == VAR_DISTORT>(
            v, ex, wk, lane, pr, grow,
            [&](int s) {
              return (long long)((MODE == MODE_ROWB) ? k1 + ((uint32_t)(lane + 32 * s) << P1) : (uint32_t)(lane + 32 * s));
            },
            n, a.fc, a.fs_over_n);
      }
      if constexpr (SG) {
        __syncwarp();  // g staging consumed: prefetch the next g row
        if (it + G < total) stage_g(it + G);
        cp_async_commit_();
      }
      if constexpr (VAR == VAR_REFERENCE) continue;
    }

    wfft1024<true>(v, wk, Tw, lane);

    // ---- outputs t2 = lane + 32 s: conj outer twiddle (ROWB) and coalesced stores
    float2 *out = const_cast<float2 *>(row_ptr(a.dst, it));
    if (MODE == MODE_ROWB && a.outer_c) {
      // the compute-bound row pass leaves the conj outer twiddle to the memory-bound pass C
#pragma unroll
      for (int s = 0; s < 32; ++s) __stcg(out + lane + 32 * s, v[s]);
    } else if constexpr (MODE == MODE_ROWB) {
      __syncwarp();
      Pw[lane] = twn((32u * k1 * (uint32_t)lane) & nmask, log2n);
      const float2 base = twn((k1 * (uint32_t)lane) & nmask, log2n);
      __syncwarp();
#pragma unroll
      for (int s = 0; s < 32; ++s) __stcg(out + lane + 32 * s, cmulc(v[s], cmul(base, Pw[s])));
    } else {
#pragma unroll
      for (int s = 0; s < 32; ++s) __stcs(out + lane + 32 * s, v[s]);
    }
  }
  if constexpr (STAGE) cp_async_wait_all();
}

// Four-step column passes with N1 = 1024: a CTA stages a [1024][8] tile (8 columns t2, 64-byte
// row segments, coalesced) into padded row-major shared memory (row stride 10 samples); warp w
// transforms column w entirely in registers (forward + outer twiddle for pass A, inverse for
// pass C), writes its column into its exchange buffer, and the CTA stores the tile back
// row-major with 16-byte coalesced stores.
// staging layout: dense 64-byte rows [1024][8]; the 16-byte chunk c of row r is stored at
// chunk c ^ ((r >> 1) & 3), so cp.async writes are conflict-free and column reads are 2-way.
__device__ __forceinline__ int col_sw(int row, int col) {
  return row * 8 + 2 * ((col >> 1) ^ ((row >> 1) & 3)) + (col & 1);
}

// Staging: the TMA engine loads the [1024][8] tile as four 256-row boxes of a 3-D tensor map
// {t2 (n2), t1 (1024), pulse} with SWIZZLE_64B, which is exactly the col_sw() layout (16-byte
// chunk index XOR address bits 7-8), so column reads are 2-way and no LSU instructions are spent
// on staging.
// Column pass, default variant: one CTA of TWO 8-warp consumer groups per SM and THREE staging
// slots.  Local tile i of the CTA goes to group i mod 2 and slot i mod 3; a slot holds the 64 KiB
// [1024][8] tile and is then reused in place as its group's padded exchange space (8 x 1058
// samples), so the CTA needs 3 x 68 KiB.  When group g finishes tile i (tile stored, group
// barrier) it issues the TMA load of tile i + 3 into the freed slot, so two tiles are computed
// while the third streams in.  (The round-1 single-group variant -- one 8-warp group, two staging
// tiles plus separate exchange buffers -- left the load latency exposed between tiles: 64 / 71 %.)
constexpr int kColSlot = ((kWW * kWPad * 8 + 1023) / 1024) * 1024 / 8;  // float2 elements
constexpr int kColSlots = 3;
__host__ __device__ constexpr size_t warp_col3_smem_bytes() {
  return (size_t)kColSlots * kColSlot * 8 + 2 * kWW * 32 * 8 + 512 * 16 + kColSlots * 8 + 1024;
}
template <bool INV>
__global__ void __launch_bounds__(2 * kWW * 32, 1) warp_col3_kernel(const WarpArgs a, const __grid_constant__ CUtensorMap smap) {
  pdl_wait();  // programmatic dependent launch (dc_common.cuh); the trigger is implicit at exit
  extern __shared__ __align__(1024) float4 smem4[];
  float2 *slots = reinterpret_cast<float2 *>(smem4);
  const int tid = threadIdx.x, grp = tid >> 8, gtid = tid & 255, warp = gtid >> 5, lane = tid & 31;
  float2 *Pw = slots + kColSlots * kColSlot + (grp * kWW + warp) * 32;
  float4 *Tw = reinterpret_cast<float4 *>(slots + kColSlots * kColSlot + 2 * kWW * 32);
  uint64_t *full = reinterpret_cast<uint64_t *>(Tw + 512);
  const int log2n = a.log2n;
  const int n = 1 << log2n;
  const uint32_t nmask = (uint32_t)n - 1u;
  const int n2 = n >> 10;
  const int64_t tiles_per_pulse = n2 / kWW;
  const int64_t total = a.pulses * tiles_per_pulse;
  auto tile_of = [&](int64_t i) { return (int64_t)blockIdx.x + i * (int64_t)gridDim.x; };
  // pass C walks the tiles last-to-first: the last pulses the row pass wrote are still in L2
  auto tile_id = [&](int64_t i) { return INV ? total - 1 - tile_of(i) : tile_of(i); };

  for (int i = tid; i < 512; i += 2 * kWW * 32) Tw[i] = reinterpret_cast<const float4 *>(a.tw)[i];
  auto stage = [&](int64_t i) {  // one thread; every generic access to the slot is ordered before it
    const int64_t it = tile_id(i);
    const int64_t p = it / tiles_per_pulse, c0 = (it - p * tiles_per_pulse) * kWW;
    float2 *sb = slots + (i % kColSlots) * kColSlot;
    uint64_t *bar = &full[i % kColSlots];
    fence_proxy_async();
    mbar_arrive_expect_tx(bar, 1024 * 8 * sizeof(float2));
#pragma unroll
    for (int b = 0; b < 4; ++b) tma_load_3d(sb + b * 256 * 8, &smap, (int)c0, b * 256, (int)p, bar);
  };
  if (tid == 0) {
    for (int s = 0; s < kColSlots; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
    for (int64_t i = 0; i < kColSlots; ++i)
      if (tile_of(i) < total) stage(i);
  }
  __syncthreads();
  auto group_sync = [grp] { asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "n"(kWW * 32) : "memory"); };

  for (int64_t i = grp; tile_of(i) < total; i += 2) {
    const int64_t it = tile_id(i);
    float2 *sb = slots + (i % kColSlots) * kColSlot;
    float2 *wk = sb + warp * kWPad;
    mbar_wait(&full[i % kColSlots], (unsigned)((i / kColSlots) & 1));
    float2 v[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) v[r] = sb[col_sw(lane + 32 * r, warp)];
    group_sync();  // the whole tile is in the group's registers: the slot becomes exchange space
    const int64_t p = it / tiles_per_pulse, c0 = (it - p * tiles_per_pulse) * kWW;
    if constexpr (!INV) {
      wfft1024<false>(v, wk, Tw, lane);
      const uint32_t t2 = (uint32_t)(c0 + warp);
      __syncwarp();
      Pw[lane] = twn((32u * t2 * (uint32_t)lane) & nmask, log2n);
      const float2 base = cscale(twn((t2 * (uint32_t)lane) & nmask, log2n), a.scale);
      __syncwarp();
#pragma unroll
      for (int s = 0; s < 32; ++s) v[s] = cmul(v[s], cmul(base, Pw[s]));
    } else {
      if (a.outer_c) {
        // pass B's conj outer twiddle w_n^(-k1 t2) on the inputs k1 = lane + 32 r of column t2
        const uint32_t t2 = (uint32_t)(c0 + warp);
        __syncwarp();
        Pw[lane] = twn((32u * t2 * (uint32_t)lane) & nmask, log2n);
        const float2 base = twn((t2 * (uint32_t)lane) & nmask, log2n);
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = cmulc(v[r], cmul(base, Pw[r]));
      }
      wfft1024<true>(v, wk, Tw, lane);
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < 32; ++s) wk[wpad(lane + 32 * s)] = v[s];
    group_sync();
    float2 *g = a.dst + p * a.pulse_stride + c0;
#pragma unroll 4
    for (int j = gtid; j < 1024 * 4; j += kWW * 32) {
      const int row = j >> 2, v4 = j & 3;
      const float2 e0 = sb[(2 * v4) * kWPad + wpad(row)];
      const float2 e1 = sb[(2 * v4 + 1) * kWPad + wpad(row)];
      __stcg(reinterpret_cast<float4 *>(g + (int64_t)row * n2 + 2 * v4), make_float4(e0.x, e0.y, e1.x, e1.y));
    }
    group_sync();  // slot drained: stream tile i + 3 into it
    if (gtid == 0 && tile_of(i + kColSlots) < total) stage(i + kColSlots);
  }
}

}  // namespace dc
