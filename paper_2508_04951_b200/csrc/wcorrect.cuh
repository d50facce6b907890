// wcorrect.cuh -- fused single-round-trip dc_correct (NEXT-1) of 1024-sample pulses on the warp-level FFT:
// one warp per pulse runs the forward FFT, the Eq. 15 phase and the inverse FFT in registers (as
// warp_row_kernel<MODE_SMALL>), drops the result into its zero-margined shared-memory buffer (which
// aliases the FFT's exchange space) and resamples it there with the Doppler tile code (doppler_tile.cuh,
// three rounds of 32 x R outputs).  x is read and y written once: 16 B/sample for both stages.
#pragma once
#include "doppler_tile.cuh"
#include "tile_fft.cuh"  // kCsPad
#include "wfft.cuh"

namespace dc {

constexpr int kWcNW = 12;                    // warps per CTA
constexpr int kWcD = 1024 + 2 * kCsPad;      // per-warp buffer: exchange (kWPad) or the padded pulse
static_assert(kWcD >= kWPad, "the Doppler buffer aliases the exchange space");
template <int WT>
__host__ __device__ constexpr size_t wcorrect_smem_bytes() {
  return ((size_t)kWcNW * (kWcD + 32 * dop_r(WT))) * sizeof(float2) + 512 * 16;
}

template <int WT, bool SECOND>
__global__ void __launch_bounds__(kWcNW * 32, 1) warp_correct1024_kernel(const WarpArgs a, float2 *__restrict__ y,
                                                                          double carrier) {
  pdl_wait();  // programmatic dependent launch (dc_common.cuh); the trigger is implicit at exit
  constexpr int n = 1024, R = dop_r(WT), SEG = 32 * R;
  extern __shared__ float4 smem4[];
  float2 *sm = reinterpret_cast<float2 *>(smem4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float2 *wk = sm + warp * kWcD;                         // exchange, then the padded pulse
  float2 *ob = sm + kWcNW * kWcD + warp * SEG;           // the warp's output segment (bulk stores)
  float4 *Tw = reinterpret_cast<float4 *>(sm + kWcNW * (kWcD + SEG));
  for (int i = threadIdx.x; i < 512; i += kWcNW * 32) Tw[i] = reinterpret_cast<const float4 *>(a.tw)[i];
  __syncthreads();
  const float inv_n = 1.0f / (float)n;
  for (int64_t it = (int64_t)blockIdx.x * kWcNW + warp; it < a.pulses; it += (int64_t)gridDim.x * kWcNW) {
    float2 v[32];
    const float2 *xp = a.src + it * n;
#pragma unroll
    for (int r = 0; r < 32; ++r) v[r] = __ldcs(xp + lane + 32 * r);
    wfft1024<false>(v, wk, Tw, lane);
    // ---- Eq. 15 phase of bin k = lane + 32 s
    const PulseParams pr = a.pp[a.pulse_base + it];
    uint32_t ex = 0u;
#pragma unroll
    for (int s = 0; s < 32; ++s) {
      if (s % 8 == 0) asm volatile("" ::: "memory");  // table loads in chunks of 8 (registers)
      const float2 g = __ldg(a.gtab + lane + 32 * s);
      const float rf = phase_frac(pr.nu_hi, pr.nu_lo, g);
      ex |= phase_needs_exact(pr.nu_hi, g) ? (1u << s) : 0u;
      const float2 w = expm2pi(rf);
      v[s] = cmul(v[s], make_float2(w.x * inv_n, w.y * inv_n));
    }
    phase_exact_fixup<false>(v, ex, wk, lane, pr, a.gtab, [&](int s) { return (long long)(lane + 32 * s); }, n, a.fc,
                             a.fs_over_n);
    wfft1024<true>(v, wk, Tw, lane);
    // ---- the iono result into the zero-margined buffer (R12: x = 0 outside [0, n))
    __syncwarp();  // every lane is done with the exchange space
#pragma unroll
    for (int i = 0; i < 2 * kCsPad / 32; ++i) {
      const int e = lane + 32 * i;
      wk[e < kCsPad ? e : n + e] = make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int s = 0; s < 32; ++s) wk[kCsPad + lane + 32 * s] = v[s];
    __syncwarp();
    // ---- Doppler (Eq. 16 windowed, D1-D4) of this pulse from shared memory, 32 R outputs per round
    DopTile cur;
    cur.pulse = it;
    cur.Bcta = -kCsPad;
    cur.beta = pr.beta;
    cur.span = kWcD;  // the zero-margined pulse: x[k] at wk[kCsPad + k]
    cur.pad0 = 0;
    cur.pad1 = 0;
#pragma unroll 1
    for (int m0 = 0; m0 < n; m0 += SEG) {
      cur.m0 = m0 - (int64_t)warp * SEG;  // dop_tile_compute places thread t at m0 + t R: undo the warp offset
      dop_tile_compute<SECOND, WT, 0, R>(wk, cur, WT, ob, y, n, carrier);
    }
    __syncwarp();  // the buffer is the next pulse's exchange space
  }
  if (lane == 0) bulk_store_wait_all();  // the warp's last output segment has left shared memory
}

}  // namespace dc
