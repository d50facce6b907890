// wtiny.cuh -- warp-level ionospheric correction (Eq. 15) of short pulses n = 32 Q,
// Q = 4, 8, 16 (n = 128, 256, 512): one HBM round trip per pulse, everything in registers plus one
// warp-private shared-memory exchange per direction.
//
// A warp owns P = 32 / Q pulses; lane (pl, j), j < Q, holds x[j + Q r] (r = 0..31) of pulse pl.
// Forward DFT, split n = 32 x Q (k = s + 32 t, s < 32, t < Q):
//   stage 1  V_j[s] = sum_r x[j + Q r] w_32^(r s)                  (DFT32 in registers)
//   exchange lane (pl, j) takes s = j + Q u, u < 32 / Q, and V_j'[s] for all j' < Q
//   stage 2  X[s + 32 t] = sum_j' (V_j'[s] w_n^(j' s)) w_Q^(j' t)   (32 / Q DFT_Q in registers)
// then the Eq. 15 phase of bin k (FP32-pair nu from the plan's natural-order 1/f table, the exact
// binary64 path for huge |nu|, 1/n folded in) and the same stages in reverse for the inverse.  The
// round-1 tile kernel reached 0.43 / 0.36 of HBM at n = 256 / 512 (barrier-synchronised passes).
#pragma once
#include "wfft.cuh"

namespace dc {

constexpr int kTinyNW = 8;  // warps per CTA
__host__ __device__ constexpr size_t wtiny_smem_bytes(int n) { return ((size_t)kTinyNW * kWPad + n) * sizeof(float2); }

template <int Q, int VAR>
__global__ void __launch_bounds__(kTinyNW * 32) warp_tiny_kernel(const WarpArgs a) {
  pdl_wait();  // programmatic dependent launch (dc_common.cuh); the trigger is implicit at exit
  static_assert(Q == 4 || Q == 8 || Q == 16, "n = 128 .. 512");
  constexpr int n = 32 * Q, P = 32 / Q, U = 32 / Q;
  constexpr int log2n = (Q == 4) ? 7 : (Q == 8) ? 8 : 9;
  constexpr bool DISTORT = (VAR == VAR_DISTORT);
  extern __shared__ float4 smem4[];
  float2 *sm = reinterpret_cast<float2 *>(smem4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float2 *wk = sm + warp * kWPad;
  float2 *Tn = sm + kTinyNW * kWPad;  // w_n^m, m < n (sincospif of the exact FP32 argument 2m/n)
  for (int m = threadIdx.x; m < n; m += kTinyNW * 32) Tn[m] = twn((uint32_t)m, log2n);
  __syncthreads();
  const int pl = lane / Q, j = lane - (lane / Q) * Q;
  auto pad = [](int e) { return e + (e >> 5); };
  const int64_t items = (a.pulses + P - 1) / P;
  const float inv_n = 1.0f / (float)n;
  for (int64_t it = (int64_t)blockIdx.x * kTinyNW + warp; it < items; it += (int64_t)gridDim.x * kTinyNW) {
    const int64_t p = it * P + pl;
    const bool ok = p < a.pulses;
    float2 v[32];
    const float2 *xp = a.src + (ok ? p : 0) * (int64_t)n;
#pragma unroll
    for (int r = 0; r < 32; ++r) v[r] = ok ? __ldcs(xp + j + Q * r) : make_float2(0.f, 0.f);
    // ---- forward
    DFT<32, false>::run(v);
    __syncwarp();
#pragma unroll
    for (int s = 0; s < 32; ++s) wk[pad(pl * n + 32 * j + s)] = v[s];
    __syncwarp();
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int s = j + Q * u;
        v[u * Q + q] = cmul(wk[pad(pl * n + 32 * q + s)], Tn[(q * s) & (n - 1)]);
      }
#pragma unroll
    for (int u = 0; u < U; ++u) DFT<Q, false>::run(v + u * Q);
    // ---- Eq. 15 phase of bin k = s + 32 t (s = j + Q u, t = element index within DFT u)
    const PulseParams pr = a.pp[a.pulse_base + (ok ? p : 0)];
    auto kb_of = [&](int e) { return (long long)(j + Q * (e / Q) + 32 * (e % Q)); };
    uint32_t ex = 0u;
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      const float2 g = __ldg(a.gtab + kb_of(e));
      const float rf = phase_frac(pr.nu_hi, pr.nu_lo, g);
      ex |= phase_needs_exact(pr.nu_hi, g) ? (1u << e) : 0u;
      const float2 w = expm2pi(DISTORT ? -rf : rf);
      v[e] = cmul(v[e], make_float2(w.x * inv_n, w.y * inv_n));
    }
    __syncwarp();  // wk free: the fix-up uses it as lane-private scratch
    phase_exact_fixup_g<DISTORT>(
        v, ex, wk, lane, pr, [&](int e) { return __ldg(a.gtab + kb_of(e)); }, kb_of, n, a.fc, a.fs_over_n);
    // ---- inverse: stage 2 then stage 1
#pragma unroll
    for (int u = 0; u < U; ++u) DFT<Q, true>::run(v + u * Q);
    __syncwarp();
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int s = j + Q * u;
        wk[pad(pl * n + 32 * q + s)] = cmulc(v[u * Q + q], Tn[(q * s) & (n - 1)]);
      }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < 32; ++s) v[s] = wk[pad(pl * n + 32 * j + s)];
    DFT<32, true>::run(v);
    if (ok) {
      float2 *yp = a.dst + p * (int64_t)n;
#pragma unroll
      for (int r = 0; r < 32; ++r) __stcs(yp + j + Q * r, v[r]);
    }
    __syncwarp();  // wk is reused by the next item
  }
}

}  // namespace dc
