// dc_common.cuh -- shared device helpers of libdispcorr (product path only).
//
// Nothing here is shared with oracle/ (the FP64 CPU oracle): the two
// implementations are independent by construction.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace dc {

// ----------------------------------------------------------------------------- programmatic dependent launch
// Every kernel is launched with programmatic stream serialisation and executes griddepcontrol.wait
// -- which returns once the previous grid has completed and its memory is visible -- before it
// touches any global data.  The dependent launch is triggered implicitly as this grid's CTAs exit,
// so the next kernel's launch latency overlaps this kernel's tail (measured: -2 us per single-pulse
// call).  An explicit trigger at kernel entry was measured 3 % slower on the C4 train (the next
// grid's CTAs then take SMs from this grid's tail).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
#ifdef DC_NO_PDL  // diagnostics build: plain stream-ordered launches
  cfg.numAttrs = 0;
#else
  cfg.numAttrs = 1;
#endif
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ----------------------------------------------------------------------------- physics
// CODATA 2018 (SI).  Eq. 1 names the symbols only; reading R5.
constexpr double kQe = 1.602176634e-19;
constexpr double kMe = 9.1093837015e-31;
constexpr double kEps0 = 8.8541878128e-12;
constexpr double kC = 299792458.0;
constexpr double kPi = 3.14159265358979323846264338327950288;

// K2 / TEC = q_e^2 / (8 pi^2 m_e eps0)   (Eq. 1)
__host__ __device__ inline double k2_per_tec() { return (kQe * kQe) / (8.0 * kPi * kPi * kMe * kEps0); }

// ----------------------------------------------------------------------------- per-pulse parameters
// Staged from the host once per call (16 B / pulse).
struct PulseParams {
  double nu_coef;  // 2 K2 / c = 2 * k2_per_tec * tec / c  [cycles * Hz]; nu_k = nu_coef / f_k  (Eq. 14/15)
  double beta;     // 1 / alpha (binary64, computed on the host exactly as the oracle does)
  double k2;       // K2 = k2_per_tec * tec (Eq. 1), for the exact binary64 phase of huge-|nu| bins
  float nu_hi, nu_lo;  // nu_coef as an unevaluated FP32 pair (hi + lo), for the FP32 phase path
};
static_assert(sizeof(PulseParams) == 32, "PulseParams is 32 bytes per pulse");

// Eq. 15 phase cycles nu = nu_coef * g (g = 1/f_k from the plan's per-bin FP32-pair table) reduced
// mod 1, entirely in FP32 pair arithmetic: p + e = hi*gh exactly (FMA), lo terms in FP32.  Returns
// r in [-1/2, 1/2] with |error| <~ 1e-12 cycles for |nu| ~ 1e3 (and ~1e-6 at the extreme near-DC
// bins where |nu| ~ 1e8); DESIGN.md "Precision".
__device__ __forceinline__ float phase_frac(float hi, float lo, float2 g) {
  const float p = hi * g.x;
  const float e = fmaf(hi, g.x, -p);
  const float l = fmaf(hi, g.y, fmaf(lo, g.x, e));
  const float fr = p - rintf(p);  // exact; 0 when |p| >= 2^23 (p is then an integer)
  const float t = fr + l;
  return t - rintf(t);
}

// Bins whose |nu| reaches 2^19 cycles (f_k within ~0.3 MHz of DC at 100 TECU -- far outside the
// model's validity, but accepted by the ABI) take the exact binary64 path below: there the
// FP32-pair product (~2^-46 relative) would leave > 1e-8 cycles of phase error.
constexpr float kPhaseExactCycles = 524288.0f;

// Eq. 15 phase cycles of signed bin kk reduced mod 1, in binary64 with the oracle's operations term
// for term (f_k = fc + (fs/n) kk, nu = 2 K2 / (c f_k), r = nu - rint(nu); R2-R4), so the result
// equals the oracle's to the FP32 rounding of r even where |nu| ~ 1e10.  Out of line: rare path.
static __device__ __noinline__ float phase_frac_exact(double k2, double fc, double fs_over_n, long long kk) {
  const double f = __dadd_rn(fc, __dmul_rn(fs_over_n, (double)kk));
  if (!(f > 0.0)) return 0.f;
  const double nu = __ddiv_rn(__dmul_rn(2.0, k2), __dmul_rn(kC, f));
  return __double2float_rn(nu - rint(nu));
}

// the FP32-pair path is exact enough for this bin unless |nu| ~ |nu_hi g_hi| reaches kPhaseExactCycles
__device__ __forceinline__ bool phase_needs_exact(float nu_hi, float2 g) { return fabsf(nu_hi * g.x) >= kPhaseExactCycles; }

// ----------------------------------------------------------------------------- complex float
// sm_100a has packed f32x2 FADD2/FMUL2/FFMA2: one issue slot per complex add / half a complex
// multiply.  The FMA pipe throughput is unchanged (128 lanes/clk/SM, measured), but issue slots
// are freed for the LDS/ALU work of the FFT passes.
#ifndef DC_X2
#define DC_X2 1
#endif
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
#if DC_X2
  return __fadd2_rn(a, b);
#else
  return make_float2(a.x + b.x, a.y + b.y);
#endif
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
#if DC_X2
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
#else
  return make_float2(a.x - b.x, a.y - b.y);
#endif
}
// a * b
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
#if DC_X2
  const float2 t = __fmul2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x));
  return __ffma2_rn(make_float2(a.x, a.x), b, t);
#else
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
#endif
}
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
#if DC_X2
  const float2 t = __fmul2_rn(make_float2(a.y, a.y), make_float2(b.y, b.x));
  return __ffma2_rn(make_float2(a.x, a.x), make_float2(b.x, -b.y), t);
#else
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
#endif
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ float2 mul_mi(float2 a) {
  return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

// exp(-i 2 pi r) for |r| <= 1/2 via the SFU sin/cos (abs. error ~4e-7).
__device__ __forceinline__ float2 expm2pi(float r) {
  float s, c;
  __sincosf(6.283185307179586f * r, &s, &c);
  return make_float2(c, -s);
}

// Reciprocal of a positive-or-negative binary64 value to ~1 ulp: FP32 SFU seed + 2 Newton steps.
__device__ __forceinline__ double drcp(double f) {
  float ff = __double2float_rn(f);
  float r0;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(ff));
  double r = (double)r0;
  double e = fma(-f, r, 1.0);
  r = fma(r, e, r);
  e = fma(-f, r, 1.0);
  r = fma(r, e, r);
  return r;
}

}  // namespace dc
