// wsmall.cuh -- single-kernel ionospheric correction (Eq. 15) of pulses of
// n = N1 x 1024 samples, N1 = 2, 4, 8 (n = 2^11 .. 2^13): one HBM round trip per pulse, the
// four-step decomposition t = 1024 t1 + t2, k = k1 + N1 k2 done entirely in shared memory.
//
// Tiles of 8192 contiguous samples (8 / N1 whole pulses) arrive with one bulk copy each
// (cp.async.bulk + transaction mbarrier).  Per tile:
//   A  thread per column (pulse, t2): N1-point DFT over t1 in registers, x w_n^(k1 t2) / n, in place
//   B  warp per row (pulse, k1): 1024-point forward DFT, the Eq. 15 phase of bin k1 + N1 k2
//      (FP32-pair nu from the plan's row-layout 1/f table), inverse DFT, x conj w_n^(k1 t2), in place
//   C  thread per column: inverse N1-point DFT over k1, stored straight to y (coalesced rows)
// The arithmetic is the three-pass four-step of the n > 8192 regime with the intermediate kept in
// shared memory, so it matches the warp row pass bit for bit in the row stage.
#pragma once
#include "tma.cuh"
#include "doppler_tile.cuh"
#include "wfft.cuh"

namespace dc {

// Two consumer groups of 8 warps, three staging slots (the column-pass pipeline of
// warp_col3_kernel applied to whole pulses).  Local tile i (8192 contiguous samples = 8 / N1 pulses)
// goes to group i mod 2 and slot i mod 3; phases A / B / C are separated by the GROUP's named barrier
// only, so the two groups run out of phase and one group's barrier waits are covered by the other's
// work, while the third slot streams in.  The warp FFT's exchange space is the row itself (XOR-swizzled
// in place: wfft1024_ip), so the CTA needs 3 x 64 KiB and no per-warp exchange buffers.  Arithmetic
// identical to warp_small_kernel (same DFTs, twiddles, phase and rounding order).
constexpr int kWs3T = 512;  // threads per CTA: two 8-warp groups (one 16-warp group at n = 2^14)
// slot of 8192 samples; the fused dc_correct variant (DOPW > 0) gives every pulse kCsPad zeros on each
// side (R12: x = 0 outside [0, n)) for the Doppler stage that runs on the slot after pass C
// n = 2^14 (N1 = 16): one pulse is a 128 KiB tile, so the CTA runs ONE 16-warp group on ONE slot (the
// next pulse streams in once pass C has drained the slot)
__host__ __device__ constexpr int wsmall3_ppt(int N1) { return N1 >= 8 ? 1 : 8 / N1; }
__host__ __device__ constexpr int wsmall3_nslot(int N1) { return N1 == 16 ? 1 : 3; }
__host__ __device__ constexpr int wsmall3_slot(int N1, int dopw) {
  return (N1 == 16 ? 16384 : 8192) + (dopw ? wsmall3_ppt(N1) * 2 * kCsPad : 0);
}
__host__ __device__ constexpr size_t wsmall3_smem_bytes(int N1 = 8, int dopw = 0) {
  return (size_t)wsmall3_nslot(N1) * wsmall3_slot(N1, dopw) * 8 + (size_t)kWs3T * 8 + 512 * 16 + 1024 * 8 + 3 * 8 + 128;
}

// physical slot of logical element i = 32 row + col of a 1024-sample row: 32 row + (col ^ row) --
// lane-distinct banks both for the Stockham write (row = lane) and the transposed read (col = lane)
__device__ __forceinline__ int wxor(int i) { return (i & ~31) | ((i ^ (i >> 5)) & 31); }

// wfft1024 with the exchange in the row's own 1024 slots (the caller has every sample in registers)
template <bool INV>
__device__ __forceinline__ void wfft1024_ip(float2 (&v)[32], float2 *__restrict__ row, const float4 *__restrict__ tw,
                                            int lane) {
  DFT<32, INV>::run(v);
  __syncwarp();
#pragma unroll
  for (int s = 0; s < 32; ++s) row[wxor(lane * 32 + s)] = v[s];
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = row[wxor(lane + 32 * r)];
#pragma unroll
  for (int h = 0; h < 16; ++h) {
    const float4 p = tw[h * 32 + lane];
    if (h > 0) v[2 * h] = INV ? cmulc(v[2 * h], make_float2(p.x, p.y)) : cmul(v[2 * h], make_float2(p.x, p.y));
    v[2 * h + 1] = INV ? cmulc(v[2 * h + 1], make_float2(p.z, p.w)) : cmul(v[2 * h + 1], make_float2(p.z, p.w));
  }
  DFT<32, INV>::run(v);
}

// DOPW > 0: fused single-round-trip dc_correct (NEXT-1): pass C leaves the ionospheric result in the
// slot (zero-margined) and the group resamples it there (Eq. 16, doppler_tile.cuh, W = DOPW, direct
// stores of R outputs per thread); x is read and y written once, 16 B/sample for both stages.
template <int N1, int VAR, int DOPW = 0, bool DSECOND = false>
__global__ void __launch_bounds__(kWs3T, 1) warp_small3_kernel(const WarpArgs a, float2 *__restrict__ y = nullptr,
                                                                double carrier = 0.0) {
  pdl_wait();  // programmatic dependent launch (dc_common.cuh); the trigger is implicit at exit
  static_assert(N1 == 2 || N1 == 4 || N1 == 8 || N1 == 16, "n = 2^11 .. 2^14");
  constexpr int P1 = (N1 == 2) ? 1 : (N1 == 4) ? 2 : (N1 == 8) ? 3 : 4;
  constexpr int log2n = P1 + 10;
  constexpr int n = 1 << log2n;
  constexpr uint32_t nmask = n - 1u;
  constexpr int PPT = wsmall3_ppt(N1);  // pulses per tile
  constexpr int NSLOT = wsmall3_nslot(N1), NGRP = (N1 == 16) ? 1 : 2, GT = kWs3T / NGRP, GW = GT / 32;
  constexpr int PAD = DOPW ? kCsPad : 0, PS = n + 2 * PAD, SLOT = wsmall3_slot(N1, DOPW);  // pulse pl at slot + pl PS + PAD
  extern __shared__ __align__(1024) float4 smem4[];
  float2 *slots = reinterpret_cast<float2 *>(smem4);  // NSLOT x SLOT samples
  const int tid = threadIdx.x, grp = tid / GT, gtid = tid - grp * GT, warp = gtid >> 5, lane = tid & 31;
  float2 *Pw = slots + NSLOT * SLOT + (tid >> 5) * 32;
  float4 *Tw = reinterpret_cast<float4 *>(slots + NSLOT * SLOT + kWs3T);
  float2 *T1 = reinterpret_cast<float2 *>(Tw + 512);  // w_n^t2, t2 < 1024 (pass A's column twiddle)
  uint64_t *full = reinterpret_cast<uint64_t *>(T1 + 1024);
  const int64_t tiles = (a.pulses + PPT - 1) / PPT;
  auto tile_of = [&](int64_t i) { return (int64_t)blockIdx.x + i * (int64_t)gridDim.x; };
  for (int i = tid; i < 512; i += kWs3T) Tw[i] = reinterpret_cast<const float4 *>(a.tw)[i];
  for (int i = tid; i < 1024; i += kWs3T) T1[i] = twn((uint32_t)i, log2n);
  if constexpr (PAD > 0) {  // the margins are never written again
    for (int i = tid; i < NSLOT * PPT * 2 * PAD; i += kWs3T) {
      const int sl = i / (PPT * 2 * PAD), j = i - sl * (PPT * 2 * PAD), pl = j / (2 * PAD), e = j - pl * 2 * PAD;
      slots[sl * SLOT + pl * PS + (e < PAD ? e : n + e)] = make_float2(0.f, 0.f);
    }
  }
  auto stage = [&](int64_t i) {  // one thread; every generic access to the slot is ordered before it
    const int64_t p0 = tile_of(i) * PPT;
    const int np = (int)min((int64_t)PPT, a.pulses - p0);
    const unsigned bytes = (unsigned)(np * n * sizeof(float2));
    fence_proxy_async();
    mbar_arrive_expect_tx(&full[i % NSLOT], bytes);
    if constexpr (PAD == 0) {
      bulk_load(slots + (i % NSLOT) * SLOT, a.src + p0 * (int64_t)n, bytes, &full[i % NSLOT]);
    } else {
      for (int pl = 0; pl < np; ++pl)
        bulk_load(slots + (i % NSLOT) * SLOT + pl * PS + PAD, a.src + (p0 + pl) * (int64_t)n, n * sizeof(float2),
                  &full[i % NSLOT]);
    }
  };
  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
    for (int64_t i = 0; i < NSLOT; ++i)
      if (tile_of(i) < tiles) stage(i);
  }
  __syncthreads();
  auto group_sync = [grp] { asm volatile("bar.sync %0, %1;\n" ::"r"(1 + grp), "n"(GT) : "memory"); };

  for (int64_t i = grp; tile_of(i) < tiles; i += NGRP) {
    float2 *sb = slots + (i % NSLOT) * SLOT;
    mbar_wait(&full[i % NSLOT], (unsigned)((i / NSLOT) & 1));
    const int64_t p0 = tile_of(i) * PPT;
    const int np = (int)min((int64_t)PPT, a.pulses - p0);
    // ---- A: columns (pulse pl, t2), forward N1-point DFT, x w_n^(k1 t2) / n
#pragma unroll 1
    for (int c = gtid; c < np * 1024; c += GT) {
      float2 *col = sb + (c >> 10) * PS + PAD + (c & 1023);
      const uint32_t t2 = (uint32_t)(c & 1023);
      float2 v[N1];
#pragma unroll
      for (int r = 0; r < N1; ++r) v[r] = col[1024 * r];
      DFT<N1, false>::run(v);
      const float2 w1 = T1[t2];  // = twn(t2, log2n)
      float2 w = cscale(make_float2(1.f, 0.f), a.scale);
#pragma unroll
      for (int k1 = 0; k1 < N1; ++k1) {
        col[1024 * k1] = cmul(v[k1], w);
        w = cmul(w, w1);  // w_n^(k1 t2): at most 7 products of correctly rounded twiddles
      }
    }
    group_sync();
    // ---- B: rows (pulse pl, k1): forward DFT -> phase -> inverse DFT -> x conj w_n^(k1 t2)
#pragma unroll 1
    for (int rw = warp; rw < np * N1; rw += GW) {
      const int pl = rw / N1, k1 = rw - pl * N1;
      float2 *row = sb + pl * PS + PAD + 1024 * k1;
      float2 v[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = row[lane + 32 * r];
      wfft1024_ip<false>(v, row, Tw, lane);
      const PulseParams pr = a.pp[a.pulse_base + p0 + pl];
      const float2 *grow = a.gtab + 1024 * k1;
      uint32_t ex = 0u;  // elements needing the exact binary64 phase
#pragma unroll
      for (int s = 0; s < 32; ++s) {
        if (s % 8 == 0) asm volatile("" ::: "memory");  // table loads in chunks of 8 (registers)
        const float2 g = __ldg(grow + lane + 32 * s);
        const float rf = phase_frac(pr.nu_hi, pr.nu_lo, g);
        ex |= phase_needs_exact(pr.nu_hi, g) ? (1u << s) : 0u;
        v[s] = cmul(v[s], expm2pi((VAR == VAR_DISTORT) ? -rf : rf));
      }
      if (__any_sync(0xffffffffu, ex != 0u)) {  // rare: the exact binary64 phase (phase_exact_fixup_g)
        __syncwarp();
#pragma unroll
        for (int s = 0; s < 32; ++s) row[lane + 32 * s] = v[s];
#pragma unroll 1
        while (ex != 0u) {
          const int s = __ffs(ex) - 1;
          ex &= ex - 1u;
          const float2 g = grow[lane + 32 * s];
          const long long k = (long long)k1 + (long long)N1 * (lane + 32 * s);
          float d = phase_frac_exact(pr.k2, a.fc, a.fs_over_n, k >= n / 2 ? k - n : k) - phase_frac(pr.nu_hi, pr.nu_lo, g);
          d -= rintf(d);
          float2 &e = row[lane + 32 * s];
          e = cmul(e, expm2pi((VAR == VAR_DISTORT) ? -d : d));
        }
        __syncwarp();
#pragma unroll
        for (int s = 0; s < 32; ++s) v[s] = row[lane + 32 * s];
      }
      wfft1024_ip<true>(v, row, Tw, lane);
      __syncwarp();
      Pw[lane] = twn((32u * (uint32_t)k1 * (uint32_t)lane) & nmask, log2n);
      const float2 base = T1[k1 * lane];  // = twn(k1 lane, log2n): k1 lane < 256
      __syncwarp();
#pragma unroll
      for (int s = 0; s < 32; ++s) row[lane + 32 * s] = cmulc(v[s], cmul(base, Pw[s]));
    }
    group_sync();
    // ---- C: columns, inverse N1-point DFT over k1 -> y[1024 t1 + t2]
#pragma unroll 1
    for (int c = gtid; c < np * 1024; c += GT) {
      const int pl = c >> 10;
      float2 *col = sb + pl * PS + PAD + (c & 1023);
      float2 v[N1];
#pragma unroll
      for (int r = 0; r < N1; ++r) v[r] = col[1024 * r];
      DFT<N1, true>::run(v);
      if constexpr (DOPW > 0) {
#pragma unroll
        for (int r = 0; r < N1; ++r) col[1024 * r] = v[r];
      } else {
        float2 *yp = a.dst + (p0 + pl) * (int64_t)n + (c & 1023);
#pragma unroll
        for (int r = 0; r < N1; ++r) __stcs(yp + 1024 * r, v[r]);
      }
    }
    if constexpr (DOPW > 0) {
      // ---- D: Doppler (Eq. 16 windowed, D1-D4) of the tile's pulses from the slot, 32 R outputs per warp
      // and item; dop_tile_compute places thread t at m0 + t R, so m0 undoes the CTA-wide warp offset
      constexpr int R = dop_r(DOPW), SEG = 32 * R, NSEG = (n + SEG - 1) / SEG;
      group_sync();
#pragma unroll 1
      for (int q = warp; q < np * NSEG; q += GW) {
        const int pl = q / NSEG, sg = q - pl * NSEG;
        DopTile cur;
        cur.pulse = p0 + pl;
        cur.m0 = (int64_t)sg * SEG - (int64_t)(tid >> 5) * SEG;
        cur.Bcta = -PAD;
        cur.beta = a.pp[a.pulse_base + p0 + pl].beta;
        cur.span = PS;  // the zero-margined pulse: x[k] at slot[pl PS + PAD + k]
        cur.pad0 = 0;
        cur.pad1 = 0;
        dop_tile_compute<DSECOND, DOPW, 0, R, true>(sb + pl * PS, cur, DOPW, nullptr, y, n, carrier);
      }
    }
    group_sync();  // slot drained: stream tile i + NSLOT into it
    if (gtid == 0 && tile_of(i + NSLOT) < tiles) stage(i + NSLOT);
  }
}

}  // namespace dc
