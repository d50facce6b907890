// pq_kernels.cu -- FFT P/Q resampling (the paper's second Doppler method; NEXT-4, reading R18).
//
// "The Fourier transform of the signal has terms removed or added followed by an inverse Fourier
// transform"; the box filter has N/alpha samples and the method is exact only when N - N/alpha
// is an even integer.  With M = n + 2 round((n alpha - n) / 2) (R18):
//   X = DFT_n(x);  A_kappa = X_kappa for |kappa| < h = min(n, M)/2, the Nyquist bin folded (M < n) or
//   split (M > n);  y_m = (1/n) sum_kappa A_kappa e^{+i 2 pi kappa m / M}  (m < min(n, M); 0 beyond),
//   then the carrier term of R10 with beta_eff = n / M.
// M is not a power of two (it is n +- an even number), so the length-M inverse DFT is evaluated as a
// chirp-z (Bluestein) convolution: kappa m = (kappa^2 + m^2 - (m - kappa)^2) / 2 gives
//   y_m = (1/n) e^{i pi m^2/M} sum_kappa a_kappa b_{m-kappa},  a_kappa = A_kappa e^{i pi kappa^2/M},
//   b_j = e^{-i pi j^2/M},
// a linear convolution over m - kappa in [-h, min(n,M) - 1 + h], i.e. a cyclic one of length L = 2n.  The
// cyclic convolution runs on the ionospheric kernels of a plan of size L in their pulse-compression mode
// (forward FFT, times the per-M table T_M = DFT_L(b), inverse FFT; tec = 0), so every step is one of:
//   pq_gather_kernel   conj(X) (row layout of the n-plan's forward spectra) -> a (natural order, length L)
//   pq_chirp_kernel    r_s = conj(b_{-s mod L}) of one M (its DFT, conjugated, is T_M)
//   pq_post_kernel     y_m = e^{i pi m^2/M} c_m / n, carrier, zero tail; y = x where M == n (identity)
// Chirp phases: pi (j^2 mod 2M) / M with j^2 mod 2M in exact 64-bit integer arithmetic.
#include "dc_kernels.h"

#include <algorithm>

namespace dc {

// e^{+i pi j^2 / M} for |j| < 2^26, M <= 2^26: q = j^2 mod 2M exactly, then sincospi of q/M in [-1, 1)
__device__ __forceinline__ float2 chirp_pos(int64_t j, int64_t M) {
  const uint64_t twoM = 2ull * (uint64_t)M;
  const uint64_t a = (uint64_t)(j < 0 ? -j : j) % twoM;
  const uint64_t q = (a * a) % twoM;
  double x = (double)q / (double)M;  // [0, 2)
  if (x >= 1.0) x -= 2.0;
  float s, c;
  sincospif((float)x, &s, &c);
  return make_float2(c, s);
}

// bin k of an n-point spectrum stored in the row layout: k = k1 + N1 k2 at index k1 N2 + k2
__device__ __forceinline__ int64_t row_index(int64_t k, int log2n, int P1) {
  return ((k & ((1ll << P1) - 1)) << (log2n - P1)) + (k >> P1);
}

__global__ void __launch_bounds__(256) pq_gather_kernel(const float2 *__restrict__ Xc, float2 *__restrict__ a,
                                                        int64_t pulses, int log2n, int P1, const int *__restrict__ Mv) {
  pdl_wait();
  const int64_t n = 1ll << log2n, L = 2 * n;
  const int64_t total = pulses * L;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i >> (log2n + 1), j = i & (L - 1);
    const int64_t M = Mv[p];
    const int64_t Nm = M < n ? M : n, h = Nm / 2;
    // identity pulses (M == n) are copied by pq_post_kernel: their a is zero
    float2 v = make_float2(0.f, 0.f);
    const bool on = M != n && (j <= h || j >= L - h);
    if (on) {
      const int64_t kap = (j <= h) ? j : j - L;
      const float2 *Xp = Xc + p * n;
      auto X = [&](int64_t k) {  // X_k (signed k), from the conjugated spectrum
        const float2 c = Xp[row_index(k < 0 ? k + n : k, log2n, P1)];
        return make_float2(c.x, -c.y);
      };
      float2 A;
      if (kap == h && M < n) {  // truncation: fold X_{-h} into +h
        const float2 u = X(h), w = X(-h);
        A = make_float2(u.x + w.x, u.y + w.y);
      } else if (kap == h || kap == -h) {
        // padding: X_{n/2} split over +h and -h; truncation keeps kappa in [-(h - 1), h]
        const float2 u = X(h);
        A = (M > n) ? make_float2(0.5f * u.x, 0.5f * u.y) : make_float2(0.f, 0.f);
      } else {
        A = X(kap);
      }
      v = cmul(A, chirp_pos(kap, M));
    }
    a[i] = v;
  }
}

// r_s = conj(b_{(-s) mod L}) for one M: b_j = e^{-i pi j^2/M} on the residues j in [-h, Nm - 1 + h], 0 elsewhere
__global__ void __launch_bounds__(256) pq_chirp_kernel(float2 *__restrict__ r, int64_t n, int64_t M) {
  pdl_wait();
  const int64_t L = 2 * n;
  const int64_t Nm = M < n ? M : n, h = Nm / 2;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < L; s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rho = (L - s) & (L - 1);
    float2 v = make_float2(0.f, 0.f);
    if (rho <= Nm - 1 + h) v = chirp_pos(rho, M);
    else if (rho >= L - h) v = chirp_pos(rho - L, M);
    r[s] = v;
  }
}

__global__ void __launch_bounds__(256) pq_post_kernel(const float2 *__restrict__ c, const float2 *__restrict__ x,
                                                      float2 *__restrict__ y, int64_t pulses, int log2n,
                                                      const int *__restrict__ Mv, double fc, double fs) {
  pdl_wait();
  const int64_t n = 1ll << log2n, L = 2 * n;
  const int64_t total = pulses * n;
  const float inv_n = 1.0f / (float)n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i >> log2n, m = i & (n - 1);
    const int64_t M = Mv[p];
    float2 v;
    if (M == n) {
      v = x[i];  // box filter of the pulse's own length: nothing removed or added
    } else if (m < M) {
      const float2 z = c[p * L + m];
      v = cmul(z, chirp_pos(m, M));
      v = make_float2(v.x * inv_n, v.y * inv_n);
      // carrier term (R10) with beta_eff = n / M, the oracle's operations: ((fc (1 - beta)) m) / fs
      const double beta = __ddiv_rn((double)n, (double)M);
      const double psi = __ddiv_rn(__dmul_rn(__dmul_rn(fc, __dsub_rn(1.0, beta)), (double)m), fs);
      if (psi != 0.0) v = cmul(v, expm2pi(__double2float_rn(psi - rint(psi))));
    } else {
      v = make_float2(0.f, 0.f);
    }
    y[i] = v;
  }
}

static int ew_grid(int64_t total) {
  LaunchShape ls{148, 8};
  launch_shape(pq_post_kernel, 256, 0, &ls);  // (cached) SM count of the current device
  const int64_t want = (total + 255) / 256;
  return (int)std::min<int64_t>(want, (int64_t)ls.sms * 8);
}

cudaError_t launch_pq_gather(const float2 *Xc, float2 *a, int64_t pulses, int log2n, int P1, const int *Mv,
                             cudaStream_t st) {
  return launch_pdl(pq_gather_kernel, dim3(ew_grid(pulses << (log2n + 1))), dim3(256), 0, st, Xc, a, pulses, log2n, P1, Mv);
}

cudaError_t launch_pq_chirp(float2 *r, int64_t n, int64_t M, cudaStream_t st) {
  return launch_pdl(pq_chirp_kernel, dim3(ew_grid(2 * n)), dim3(256), 0, st, r, n, M);
}

cudaError_t launch_pq_post(const float2 *c, const float2 *x, float2 *y, int64_t pulses, int log2n, const int *Mv,
                           double fc, double fs, cudaStream_t st) {
  return launch_pdl(pq_post_kernel, dim3(ew_grid(pulses << log2n)), dim3(256), 0, st, c, x, y, pulses, log2n, Mv, fc,
                    fs);
}

}  // namespace dc
