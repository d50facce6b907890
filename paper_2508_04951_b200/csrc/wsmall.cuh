// wsmall.cuh -- single-kernel ionospheric correction (Eq. 15) of pulses of
// n = N1 x 1024 samples, N1 = 2, 4, 8 (n = 2^11 .. 2^13): one HBM round trip per pulse, the
// four-step decomposition t = 1024 t1 + t2, k = k1 + N1 k2 done entirely in shared memory.
//
// A CTA (8 warps) owns tiles of 8192 contiguous samples (8 / N1 whole pulses), double-buffered:
// the next tile streams in with one bulk copy (cp.async.bulk + transaction mbarrier) while the
// current one computes.  Per tile:
//   A  thread per column (pulse, t2): N1-point DFT over t1 in registers, x w_n^(k1 t2) / n, in place
//   B  warp per row (pulse, k1): 1024-point forward DFT (wfft1024), the Eq. 15 phase of bin
//      k1 + N1 k2 (FP32-pair nu from the plan's row-layout 1/f table), inverse DFT,
//      x conj w_n^(k1 t2), in place
//   C  thread per column: inverse N1-point DFT over k1, stored straight to y (coalesced rows)
// The arithmetic is the three-pass four-step of iono_kernels.cu with the intermediate kept in
// shared memory, so it matches the warp row pass bit for bit in the row stage.
#pragma once
#include "tma.cuh"
#include "wfft.cuh"

namespace dc {

constexpr int kWsT = 8 * 32;  // threads per CTA
__host__ __device__ constexpr size_t wsmall_smem_bytes() {
  return (size_t)2 * 8192 * 8 + (size_t)8 * (kWPad + 32) * 8 + 512 * 16 + 2 * 8 + 128;
}

template <int N1, int VAR>
__global__ void __launch_bounds__(kWsT, 1) warp_small_kernel(const WarpArgs a) {
  pdl_wait();  // programmatic dependent launch (dc_common.cuh); the trigger is implicit at exit
  static_assert(N1 == 2 || N1 == 4 || N1 == 8, "n = 2^11 .. 2^13");
  constexpr int P1 = (N1 == 2) ? 1 : (N1 == 4) ? 2 : 3;
  constexpr int log2n = P1 + 10;
  constexpr int n = 1 << log2n;
  constexpr uint32_t nmask = n - 1u;
  constexpr int PPT = 8 / N1;  // pulses per tile
  extern __shared__ __align__(128) float4 smem4[];
  float2 *bufs = reinterpret_cast<float2 *>(smem4);  // 2 x 8192 samples
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float2 *wk = bufs + 2 * 8192 + warp * kWPad;
  float2 *Pw = bufs + 2 * 8192 + 8 * kWPad + warp * 32;
  float4 *Tw = reinterpret_cast<float4 *>(bufs + 2 * 8192 + 8 * (kWPad + 32));
  uint64_t *bars = reinterpret_cast<uint64_t *>(Tw + 512);
  const int64_t tiles = (a.pulses + PPT - 1) / PPT;
  for (int i = tid; i < 512; i += kWsT) Tw[i] = reinterpret_cast<const float4 *>(a.tw)[i];
  auto stage = [&](int64_t t, int b) {  // thread 0: the tile's valid pulses, one bulk copy
    const int64_t p0 = t * PPT;
    const int np = (int)min((int64_t)PPT, a.pulses - p0);
    const unsigned bytes = (unsigned)(np * n * sizeof(float2));
    mbar_arrive_expect_tx(&bars[b], bytes);
    bulk_load(bufs + b * 8192, a.src + p0 * (int64_t)n, bytes, &bars[b]);
  };
  int64_t t = blockIdx.x;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
    if (t < tiles) stage(t, 0);
  }
  __syncthreads();
  unsigned phase[2] = {0u, 0u};
  for (int b = 0; t < tiles; t += gridDim.x, b ^= 1) {
    if (tid == 0 && t + gridDim.x < tiles) {
      fence_proxy_async();  // buffer b ^ 1 was last read by generic loads before the trailing barrier
      stage(t + gridDim.x, b ^ 1);
    }
    mbar_wait(&bars[b], phase[b]);
    phase[b] ^= 1u;
    float2 *sb = bufs + b * 8192;
    const int64_t p0 = t * PPT;
    const int np = (int)min((int64_t)PPT, a.pulses - p0);
    // ---- A: columns (pulse pl, t2), forward N1-point DFT, x w_n^(k1 t2) / n
#pragma unroll 1
    for (int c = tid; c < np * 1024; c += kWsT) {
      float2 *col = sb + (c >> 10) * n + (c & 1023);
      const uint32_t t2 = (uint32_t)(c & 1023);
      float2 v[N1];
#pragma unroll
      for (int r = 0; r < N1; ++r) v[r] = col[1024 * r];
      DFT<N1, false>::run(v);
      const float2 w1 = twn(t2 & nmask, log2n);
      float2 w = cscale(make_float2(1.f, 0.f), a.scale);
      const float2 w1s = w1;
#pragma unroll
      for (int k1 = 0; k1 < N1; ++k1) {
        col[1024 * k1] = cmul(v[k1], w);
        w = cmul(w, w1s);  // w_n^(k1 t2): at most 7 products of correctly rounded twiddles
      }
    }
    __syncthreads();
    // ---- B: rows (pulse pl, k1): forward DFT -> phase -> inverse DFT -> x conj w_n^(k1 t2)
    if (warp < np * N1) {
      const int pl = warp / N1, k1 = warp - pl * N1;
      float2 *row = sb + pl * n + 1024 * k1;
      float2 v[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = row[lane + 32 * r];
      wfft1024<false>(v, wk, Tw, lane);
      const PulseParams pr = a.pp[a.pulse_base + p0 + pl];
      const float2 *grow = a.gtab + 1024 * k1;
      uint32_t ex = 0u;  // elements needing the exact binary64 phase (phase_exact_fixup)
#pragma unroll
      for (int s = 0; s < 32; ++s) {
        if (s % 8 == 0) asm volatile("" ::: "memory");  // table loads in chunks of 8 (registers)
        const float2 g = __ldg(grow + lane + 32 * s);
        const float rf = phase_frac(pr.nu_hi, pr.nu_lo, g);
        ex |= phase_needs_exact(pr.nu_hi, g) ? (1u << s) : 0u;
        v[s] = cmul(v[s], expm2pi((VAR == VAR_DISTORT) ? -rf : rf));
      }
      phase_exact_fixup<VAR == VAR_DISTORT>(
          v, ex, wk, lane, pr, grow, [&](int s) { return (long long)k1 + (long long)N1 * (lane + 32 * s); }, n, a.fc,
          a.fs_over_n);
      wfft1024<true>(v, wk, Tw, lane);
      __syncwarp();
      Pw[lane] = twn((32u * (uint32_t)k1 * (uint32_t)lane) & nmask, log2n);
      const float2 base = twn(((uint32_t)k1 * (uint32_t)lane) & nmask, log2n);
      __syncwarp();
#pragma unroll
      for (int s = 0; s < 32; ++s) row[lane + 32 * s] = cmulc(v[s], cmul(base, Pw[s]));
    }
    __syncthreads();
    // ---- C: columns, inverse N1-point DFT over k1 -> y[1024 t1 + t2]
#pragma unroll 1
    for (int c = tid; c < np * 1024; c += kWsT) {
      const int pl = c >> 10;
      const float2 *col = sb + pl * n + (c & 1023);
      float2 v[N1];
#pragma unroll
      for (int r = 0; r < N1; ++r) v[r] = col[1024 * r];
      DFT<N1, true>::run(v);
      float2 *yp = a.dst + (p0 + pl) * (int64_t)n + (c & 1023);
#pragma unroll
      for (int r = 0; r < N1; ++r) __stcs(yp + 1024 * r, v[r]);
    }
    __syncthreads();  // buffer b consumed
  }
}

}  // namespace dc
