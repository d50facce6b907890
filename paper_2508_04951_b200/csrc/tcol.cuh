// tcol.cuh -- four-step column passes for short columns (N1 = 16, 32, 64; n = N1 x 1024 =
// 2^14 .. 2^16, config C2): ONE THREAD PER COLUMN.  A warp takes 32 adjacent columns t2, so each
// of its N1 row loads is one coalesced 256-byte segment; the thread holds its whole column in
// registers and runs the N1-point DFT there (no shared memory, no barriers).  Pass A multiplies by
// w_n^(k1 t2) / n (exact arguments through sincospif) and writes Z[k1][t2]; pass C reads the row
// pass's output column and writes y[1024 t1 + t2].  The row pass between them is the warp-level
// 1024-point kernel (wfft.cuh).
#pragma once
#include "wfft.cuh"

namespace dc {

__device__ __forceinline__ constexpr float cos64(int k) {
  constexpr float t[64] = {
    1.00000000000000000000f,
    0.99518472667219692873f,
    0.98078528040323043058f,
    0.95694033573220882438f,
    0.92387953251128673848f,
    0.88192126434835504956f,
    0.83146961230254523567f,
    0.77301045336273699338f,
    0.70710678118654757274f,
    0.63439328416364548779f,
    0.55557023301960228867f,
    0.47139673682599780857f,
    0.38268343236508983729f,
    0.29028467725446233105f,
    0.19509032201612833135f,
    0.09801714032956077016f,
    0.00000000000000006123f,
    -0.09801714032956064526f,
    -0.19509032201612819257f,
    -0.29028467725446216452f,
    -0.38268343236508972627f,
    -0.47139673682599769755f,
    -0.55557023301960195560f,
    -0.63439328416364537677f,
    -0.70710678118654746172f,
    -0.77301045336273699338f,
    -0.83146961230254534669f,
    -0.88192126434835493853f,
    -0.92387953251128673848f,
    -0.95694033573220882438f,
    -0.98078528040323043058f,
    -0.99518472667219681771f,
    -1.00000000000000000000f,
    -0.99518472667219692873f,
    -0.98078528040323043058f,
    -0.95694033573220893540f,
    -0.92387953251128684951f,
    -0.88192126434835504956f,
    -0.83146961230254545772f,
    -0.77301045336273710440f,
    -0.70710678118654768376f,
    -0.63439328416364593188f,
    -0.55557023301960217765f,
    -0.47139673682599786408f,
    -0.38268343236509033689f,
    -0.29028467725446244208f,
    -0.19509032201612866442f,
    -0.09801714032956045097f,
    -0.00000000000000018370f,
    0.09801714032956009015f,
    0.19509032201612830359f,
    0.29028467725446205350f,
    0.38268343236509000382f,
    0.47139673682599758653f,
    0.55557023301960184458f,
    0.63439328416364559882f,
    0.70710678118654735069f,
    0.77301045336273666031f,
    0.83146961230254523567f,
    0.88192126434835482751f,
    0.92387953251128651644f,
    0.95694033573220882438f,
    0.98078528040323031956f,
    0.99518472667219692873f
  };
  return t[k & 63];
}
// v * exp(-+ 2 pi i K / 64), K = 1 .. 31 (compile-time constants)
template <int K, bool INV>
__device__ __forceinline__ float2 rot64(float2 v) {
  if constexpr ((K & 1) == 0) {
    return rot<32, K / 2, INV>(v);
  } else {
    constexpr float c = cos64(K);
    constexpr float sn = cos64(K - 16);  // sin(2 pi K / 64)
    constexpr float s = INV ? sn : -sn;
    return make_float2(fmaf(v.x, c, -v.y * s), fmaf(v.x, s, v.y * c));
  }
}
template <bool INV, int K = 1>
__device__ __forceinline__ void rot64_all(float2 *o) {
  if constexpr (K < 32) {
    o[K] = rot64<K, INV>(o[K]);
    rot64_all<INV, K + 1>(o);
  }
}
// in-place natural-order DFT of N = 16, 32 or 64 points held by one thread
template <int N, bool INV>
__device__ __forceinline__ void dft_thread(float2 *v) {
  if constexpr (N == 64) {  // radix-2 DIT over two DFT-32s
    float2 e[32], o[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      e[i] = v[2 * i];
      o[i] = v[2 * i + 1];
    }
    DFT<32, INV>::run(e);
    DFT<32, INV>::run(o);
    rot64_all<INV>(o);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      v[k] = cadd(e[k], o[k]);
      v[k + 32] = csub(e[k], o[k]);
    }
  } else {
    DFT<N, INV>::run(v);
  }
}

constexpr int kTcolT = 256;  // threads per CTA (8 warps x 32 columns)

template <int N1, bool INV>
__global__ void __launch_bounds__(kTcolT, 1) thread_col_kernel(const WarpArgs a) {
  pdl_wait();  // programmatic dependent launch (dc_common.cuh); the trigger is implicit at exit
  constexpr int log2n = (N1 == 16 ? 4 : N1 == 32 ? 5 : 6) + 10;
  constexpr int n = 1 << log2n;
  constexpr uint32_t nmask = n - 1u;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * kTcolT + threadIdx.x) >> 5, G = ((int64_t)gridDim.x * kTcolT) >> 5;
  const int64_t total = a.pulses * (1024 / 32);  // warp items: 32 columns of one pulse
  for (int64_t it = gw; it < total; it += G) {
    const int64_t p = it >> 5;
    const uint32_t t2 = (uint32_t)((it & 31) * 32 + lane);
    const float2 *src = a.src + p * a.pulse_stride + t2;
    float2 *dst = a.dst + p * a.pulse_stride + t2;
    float2 v[N1];
#pragma unroll
    for (int r = 0; r < N1; ++r) v[r] = INV ? __ldcg(src + 1024 * r) : __ldcs(src + 1024 * r);
    if (INV && a.outer_c) {
      // pass B's conj outer twiddle w_n^(-k1 t2), applied on load (the row pass is the compute-bound one)
      uint32_t tz;
      asm volatile("mov.u32 %0, 0;\n" : "=r"(tz));
      tz += t2;
#pragma unroll
      for (int h = 0; h < N1 / 8; ++h) {
        const float2 hi = twn((uint32_t)(8 * h) * tz & nmask, log2n);
#pragma unroll
        for (int c = 0; c < 8; ++c) v[8 * h + c] = cmulc(v[8 * h + c], cmul(hi, twn((uint32_t)c * tz & nmask, log2n)));
      }
    }
    dft_thread<N1, INV>(v);
    if constexpr (!INV) {
      // w_n^(k1 t2) / n = hi(k1 >> 3) lo(k1 & 7); an opaque zero keeps the compiler from hoisting
      // the N1 twiddles of this column out of the loop (they would spill)
      uint32_t tz;
      asm volatile("mov.u32 %0, 0;\n" : "=r"(tz));
      tz += t2;
#pragma unroll
      for (int h = 0; h < N1 / 8; ++h) {
        const float2 hi = cscale(twn((uint32_t)(8 * h) * tz & nmask, log2n), a.scale);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float2 lo = twn((uint32_t)c * tz & nmask, log2n);
          __stcg(dst + 1024 * (8 * h + c), cmul(v[8 * h + c], cmul(hi, lo)));
        }
      }
    } else {
#pragma unroll
      for (int r = 0; r < N1; ++r) __stcg(dst + 1024 * r, v[r]);
    }
  }
}

}  // namespace dc
