/*
 * oracle.c -- plain, slow, obviously-correct FP64 CPU oracle for the
 * dispersion-correction hot path of arXiv 2508.04951 (Vickers, Mack,
 * Osaretin, "Real-Time Doppler and Ionospheric Dispersion Correction
 * Techniques for Arbitrary Waveforms Utilizing GPU Compute").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load or call this
 * library.  The product path (paper_2508_04951_b200/, libdispcorr) shares no
 * code, header, table or constant generator with this file and never calls it.
 *
 * Citations: "P:Lnnn" = line nnn of the paper text; equation numbers
 * follow source order (Eq. 1 at P:L89 ... Eq. 16 at P:L285).  Readings of
 * silent/ambiguous passages are the ones listed in DESIGN.md section
 * "Readings of the paper" (R1..R12); each use below names its reading.
 *
 * Arithmetic: IEEE binary64 throughout, no fast-math, no reassociation beyond
 * what the definitions state.  Complex numbers are interleaved (re, im) pairs.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_PI 3.14159265358979323846264338327950288

/* CODATA 2018 exact / recommended values (SI).  P:L91 Eq. 1 names the
 * symbols; the paper gives no numbers (reading R5). */
static const double ORC_QE = 1.602176634e-19;    /* electron charge, C (exact) */
static const double ORC_ME = 9.1093837015e-31;   /* electron mass, kg          */
static const double ORC_EPS0 = 8.8541878128e-12; /* vacuum permittivity, F/m   */
static const double ORC_C = 299792458.0;         /* speed of light, m/s (exact) */

/* ---------------------------------------------------------------------------
 * Physical model
 * ------------------------------------------------------------------------- */

/* K2 / E = q_e^2 / (8 pi^2 m_e eps0)   [m^3/s^2 per (el/m^2)]
 * Eq. 1 and Appendix A Eq. 21. */
double orc_k2_per_tec(void) {
  return (ORC_QE * ORC_QE) / (8.0 * ORC_PI * ORC_PI * ORC_ME * ORC_EPS0);
}

double orc_speed_of_light(void) { return ORC_C; }

/* One-way group delay tau(f) = K2 / (c f^2), Eq. 1. */
double orc_group_delay(double f_hz, double tec) {
  double k2 = orc_k2_per_tec() * tec;
  return k2 / (ORC_C * f_hz * f_hz);
}

/* alpha = (1 + v/c) / (1 - v/c), v > 0 approaching.  Eq. 13 context. */
double orc_alpha_from_velocity(double v_mps) {
  return (1.0 + v_mps / ORC_C) / (1.0 - v_mps / ORC_C);
}

/* ---------------------------------------------------------------------------
 * Discrete Fourier transform.  X_k = sum_t x_t exp(sign * i 2 pi k t / n).
 * sign = -1 is the forward transform (numpy / textbook convention, reading R1).
 * ------------------------------------------------------------------------- */

/* Direct O(n^2) DFT, the definition written out.  The exponent k*t is reduced
 * modulo n in exact integer arithmetic (exp is 2 pi-periodic in the angle), so
 * the angle stays in [0, 2 pi). */
void orc_dft(int64_t n, const double *x, double *X, int sign) {
  for (int64_t k = 0; k < n; ++k) {
    double re = 0.0, im = 0.0;
    for (int64_t t = 0; t < n; ++t) {
      int64_t kt = (int64_t)(((__int128)k * t) % n);
      double ang = (double)sign * 2.0 * ORC_PI * (double)kt / (double)n;
      double c = cos(ang), s = sin(ang);
      double xr = x[2 * t], xi = x[2 * t + 1];
      re += xr * c - xi * s;
      im += xr * s + xi * c;
    }
    X[2 * k] = re;
    X[2 * k + 1] = im;
  }
}

/* Textbook iterative radix-2 decimation-in-time FFT, in place, n = 2^p.
 * Bit-reversal permutation followed by log2(n) butterfly stages with twiddles
 * exp(sign * i 2 pi j / len) from cos/sin.  Unnormalised. */
void orc_fft(int64_t n, double *x, int sign) {
  /* bit reversal */
  for (int64_t i = 1, j = 0; i < n; ++i) {
    int64_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      double tr = x[2 * i], ti = x[2 * i + 1];
      x[2 * i] = x[2 * j];
      x[2 * i + 1] = x[2 * j + 1];
      x[2 * j] = tr;
      x[2 * j + 1] = ti;
    }
  }
  for (int64_t len = 2; len <= n; len <<= 1) {
    int64_t half = len >> 1;
    for (int64_t j = 0; j < half; ++j) {
      double ang = (double)sign * 2.0 * ORC_PI * (double)j / (double)len;
      double wr = cos(ang), wi = sin(ang);
      for (int64_t s = 0; s < n; s += len) {
        int64_t a = s + j, b = s + j + half;
        double br = x[2 * b] * wr - x[2 * b + 1] * wi;
        double bi = x[2 * b] * wi + x[2 * b + 1] * wr;
        double ar = x[2 * a], ai = x[2 * a + 1];
        x[2 * a] = ar + br;
        x[2 * a + 1] = ai + bi;
        x[2 * b] = ar - br;
        x[2 * b + 1] = ai - bi;
      }
    }
  }
}

/* ---------------------------------------------------------------------------
 * Ionospheric correction, Eq. 15:
 *   S_Tx = F^-1[ F(S_Rx) exp(-4 pi i K2 / (c f)) ]
 * and the forward (distortion) model, Eq. 14, with the opposite
 * sign.  Steps (SURVEY O-IONO):
 *   1. X = DFT(x)                                    (forward, e^{-i}; R1)
 *   2. f_k = fc + fs (k - n [k >= n/2]) / n          (bin -> absolute RF; R2)
 *   3. nu_k = 2 K2 / (c f_k) cycles if f_k > 0 else 0 (two-way 2 tau f; R3, R4)
 *   4. Y_k = X_k exp(dir * i 2 pi nu_k), dir = -1 correct (Eq. 15), +1 distort (Eq. 14)
 *   5. y = (1/n) IDFT(Y)                             (R6)
 * exp(i 2 pi nu) is evaluated as exp(i 2 pi (nu - nearbyint(nu))): the same
 * number (period 1 in nu), with the subtraction exact in binary64.
 * method: 0 = radix-2 FFT (n must be a power of two), 1 = direct DFT.
 * ------------------------------------------------------------------------- */
double orc_bin_frequency(int64_t k, int64_t n, double fs, double fc) {
  int64_t kk = (k >= n / 2) ? k - n : k; /* Nyquist bin n/2 is negative (R2) */
  return fc + fs * (double)kk / (double)n;
}

double orc_iono_phase_cycles(double f_hz, double tec) {
  if (!(f_hz > 0.0)) return 0.0; /* unit multiplier at f <= 0 (R3) */
  double k2 = orc_k2_per_tec() * tec;
  return 2.0 * k2 / (ORC_C * f_hz); /* 2 tau(f) f = 2 K2 / (c f), Eq. 14 */
}

int orc_iono_dir(int64_t n, double fs, double fc, double tec, int dir, int method,
                 const double *x, double *y) {
  if (n < 1) return -1;
  double *X = (double *)malloc(sizeof(double) * 2 * (size_t)n);
  if (!X) return -2;
  if (method == 1) {
    orc_dft(n, x, X, -1);
  } else {
    memcpy(X, x, sizeof(double) * 2 * (size_t)n);
    orc_fft(n, X, -1);
  }
  for (int64_t k = 0; k < n; ++k) {
    double f = orc_bin_frequency(k, n, fs, fc);
    double nu = orc_iono_phase_cycles(f, tec);
    double r = nu - nearbyint(nu);
    double ang = (double)dir * 2.0 * ORC_PI * r;
    double c = cos(ang), s = sin(ang);
    double xr = X[2 * k], xi = X[2 * k + 1];
    X[2 * k] = xr * c - xi * s;
    X[2 * k + 1] = xr * s + xi * c;
  }
  if (method == 1) {
    orc_dft(n, X, y, +1);
  } else {
    memcpy(y, X, sizeof(double) * 2 * (size_t)n);
    orc_fft(n, y, +1);
  }
  for (int64_t t = 0; t < 2 * n; ++t) y[t] /= (double)n;
  free(X);
  return 0;
}

/* Correction (Eq. 15). */
int orc_iono(int64_t n, double fs, double fc, double tec, int method, const double *x,
             double *y) {
  return orc_iono_dir(n, fs, fc, tec, -1, method, x, y);
}

/* ---------------------------------------------------------------------------
 * Pulse compression after the ionospheric correction (the
 * paper's pulse-compression path, fig:pulse_compression_path P:L246-251, whose
 * headline timing is "during pulse compression").  The corrected pulse
 * y = iono(x) (Eq. 15) is matched-filtered against a reference r_0 .. r_{L-1}
 * (L <= n), circularly over the n-sample window (reading R16):
 *   z_m = sum_{s=0}^{L-1} y_{(s+m) mod n} conj(r_s)
 * i.e. the circular cross-correlation, which equals IDFT_n(Y_k conj(R_k)) with
 * R = DFT_n of r zero-padded to n.  Written here as the direct sum (the
 * definition), for the outputs listed in idx (all n when idx == NULL).
 * ------------------------------------------------------------------------- */
int orc_correlate(int64_t n, const double *y, int64_t L, const double *r, int64_t nidx,
                  const int64_t *idx, double *z) {
  if (n < 1 || L < 1 || L > n) return -1;
  const int64_t cnt = idx ? nidx : n;
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
  for (int64_t i = 0; i < cnt; ++i) {
    const int64_t m = idx ? idx[i] : i;
    double ar = 0.0, ai = 0.0;
    for (int64_t s = 0; s < L; ++s) {
      const int64_t t = (s + m) % n;
      const double yr = y[2 * t], yi = y[2 * t + 1], rr = r[2 * s], ri = r[2 * s + 1];
      ar += yr * rr + yi * ri; /* y conj(r) */
      ai += yi * rr - yr * ri;
    }
    z[2 * i] = ar;
    z[2 * i + 1] = ai;
  }
  return 0;
}

int orc_compress(int64_t n, double fs, double fc, double tec, const double *x, int64_t L,
                 const double *r, int64_t nidx, const int64_t *idx, double *z) {
  if (n < 1 || L < 1 || L > n) return -1;
  double *y = (double *)malloc(sizeof(double) * 2 * (size_t)n);
  if (!y) return -2;
  int rc = orc_iono(n, fs, fc, tec, (n & (n - 1)) ? 1 : 0, x, y);
  if (rc == 0) rc = orc_correlate(n, y, L, r, nidx, idx, z);
  free(y);
  return rc;
}

/* ---------------------------------------------------------------------------
 * Doppler time-dilation correction by windowed Whittaker-Shannon
 * interpolation, Eq. 16 restricted to a window of W samples
 * (Alg. 1, window P:L533).  Resampling onto t/alpha
 * undoes S(alpha t) (Eq. 13; reading R8).  Steps (SURVEY O-DOPP):
 *   beta = 1/alpha; for m in [0, n):
 *     t = m beta; k_lo = floor(t - W/2) + 1               (window {k: -W/2 < k - t <= W/2}; R9)
 *     acc = sum_{k=k_lo}^{k_lo+W-1} [0 <= k < n] x_k sinc(t - k)   (zero outside; R12)
 *     y_m = acc exp(-i 2 pi fc (1 - beta) m / fs)            (carrier term; R10)
 * sinc(d) = 1 at d = 0, 0 at nonzero integer d, sin(pi d)/(pi d) otherwise
 * (normalised sinc, Eq. 16; rectangular window, reading R11).
 * ------------------------------------------------------------------------- */
double orc_sinc(double d) {
  if (d == 0.0) return 1.0;
  if (d == floor(d)) return 0.0;
  return sin(ORC_PI * d) / (ORC_PI * d);
}

/* ---------------------------------------------------------------------------
 * Optional taper of the sinc window ("taper window size, taper"; SURVEY
 * 8(f) NEXT-3; reading R17): Kaiser window of shape parameter kb >= 0 over the
 * W-sample window, half-width L = W/2,
 *   taper(d) = I0(kb sqrt(1 - (d/L)^2)) / I0(kb),   d = t - k in [-L, L),
 * so h(d) = sinc(d) taper(d).  kb = 0 gives taper = 1 exactly (the rectangular
 * window of R11).  I0 by its power series sum_j ((z/2)^2)^j / (j!)^2.
 * ------------------------------------------------------------------------- */
double orc_bessel_i0(double z) {
  double q = 0.25 * z * z, term = 1.0, sum = 1.0;
  for (int j = 1; j < 500; ++j) {
    term *= q / ((double)j * (double)j);
    sum += term;
    if (term < 1e-17 * sum) break;
  }
  return sum;
}

double orc_kaiser(double d, double L, double kb) {
  if (kb == 0.0) return 1.0;
  double x = d / L;
  double r = 1.0 - x * x;
  if (r < 0.0) r = 0.0;
  return orc_bessel_i0(kb * sqrt(r)) / orc_bessel_i0(kb);
}

/* Hann taper (reading R17, the second taper option): taper(d) = (1 + cos(pi d / L)) / 2, selected by
 * passing kb = ORC_HANN (-1) wherever a Kaiser kb is taken. */
#define ORC_HANN (-1.0)
double orc_hann(double d, double L) { return 0.5 * (1.0 + cos(ORC_PI * d / L)); }
static double orc_taper(double d, double L, double kb) { return (kb == ORC_HANN) ? orc_hann(d, L) : orc_kaiser(d, L, kb); }

/* one output m of the windowed, optionally tapered Eq. 16 with the R10 carrier (the steps above) */
static void orc_doppler_one(int64_t n, int W, double fs, double fc, double beta, double kb, const double *x,
                            int64_t m, double *ym) {
  double L = 0.5 * (double)W;
  double t = (double)m * beta;
  int64_t k_lo = (int64_t)floor(t - 0.5 * (double)W) + 1;
  double re = 0.0, im = 0.0;
  for (int64_t k = k_lo; k < k_lo + W; ++k) {
    if (k < 0 || k >= n) continue;
    double h = orc_sinc(t - (double)k) * orc_taper(t - (double)k, L, kb);
    re += x[2 * k] * h;
    im += x[2 * k + 1] * h;
  }
  /* carrier rotation; cycles reduced mod 1 (period 1) before the angle */
  double psi = fc * (1.0 - beta) * (double)m / fs;
  double r = psi - nearbyint(psi);
  double ang = -2.0 * ORC_PI * r;
  double c = cos(ang), s = sin(ang);
  ym[0] = re * c - im * s;
  ym[1] = re * s + im * c;
}

int orc_doppler_win(int64_t n, int W, double fs, double fc, double alpha, double kb,
                    const double *x, double *y) {
  if (n < 1 || W < 1 || !(alpha > 0.0) || !(kb >= 0.0 || kb == ORC_HANN)) return -1;
  double beta = 1.0 / alpha;
  for (int64_t m = 0; m < n; ++m) orc_doppler_one(n, W, fs, fc, beta, kb, x, m, y + 2 * m);
  return 0;
}

/* The same outputs at the nidx sample positions idx[] only (parity at sizes where the whole
 * pulse would take too long); OpenMP over the samples. */
int orc_doppler_at(int64_t n, int W, double fs, double fc, double alpha, double kb, const double *x,
                   int64_t nidx, const int64_t *idx, double *y) {
  if (n < 1 || W < 1 || !(alpha > 0.0) || !(kb >= 0.0 || kb == ORC_HANN)) return -1;
  double beta = 1.0 / alpha;
  int err = 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) reduction(| : err)
#endif
  for (int64_t i = 0; i < nidx; ++i) {
    if (idx[i] < 0 || idx[i] >= n) {
      err |= 1;
      continue;
    }
    orc_doppler_one(n, W, fs, fc, beta, kb, x, idx[i], y + 2 * i);
  }
  return err ? -1 : 0;
}

/* rectangular window (reading R11) */
int orc_doppler(int64_t n, int W, double fs, double fc, double alpha, const double *x,
                double *y) {
  return orc_doppler_win(n, W, fs, fc, alpha, 0.0, x, y);
}

/* Exact (unwindowed) Whittaker-Shannon sum over the whole record, Eq. 16,
 * O(n^2).  Used only as a brute-force pin for orc_doppler. */
int orc_doppler_exact(int64_t n, double fs, double fc, double alpha, const double *x,
                      double *y) {
  double beta = 1.0 / alpha;
  for (int64_t m = 0; m < n; ++m) {
    double t = (double)m * beta;
    double re = 0.0, im = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      double h = orc_sinc(t - (double)k);
      re += x[2 * k] * h;
      im += x[2 * k + 1] * h;
    }
    double psi = fc * (1.0 - beta) * (double)m / fs;
    double r = psi - nearbyint(psi);
    double ang = -2.0 * ORC_PI * r;
    double c = cos(ang), s = sin(ang);
    y[2 * m] = re * c - im * s;
    y[2 * m + 1] = re * s + im * c;
  }
  return 0;
}

/* ---------------------------------------------------------------------------
 * FFT P/Q resampling (Table 2): "the Fourier
 * transform of the signal has terms removed or added followed by an inverse Fourier
 * transform" -- the sinc filter becomes a box filter; exact for Nyquist-limited signals
 * when the number of added/removed samples is an even integer.  Reading R18:
 *   X = DFT_n(x);  Y (length M) takes the bins of X with |signed frequency| < min(n, M)/2,
 *   the bin at min(n, M)/2 (even min) is split in half when padding (M > n) and the two
 *   bins at +-n'/2 are folded together when truncating (M < n);
 *   y_m = (1/n) sum_{k<M} Y_k exp(+i 2 pi k m / M),  m < min(n, M); zero for M <= m < n,
 * i.e. the band-limited periodic interpolant of x at t = m n / M (scipy.signal.resample's
 * convention).  Direct transforms of any length (the definitions written out).
 * ------------------------------------------------------------------------- */
/* The length-M spectrum Y of the P/Q resampler from the length-n spectrum X (reading R18): bins
 * 0 .. Nm/2 and -1 .. -(Nm - Nm/2 - 1) copied (Nm = min(n, M)); for even Nm the Nyquist bin is folded
 * (M < n: X[-h] added into Y[+h]) or split in half over Y[+h] and Y[-h] (M > n).  Y: 2M doubles, zeroed. */
static void pq_bins(int64_t n, int64_t M, const double *X, double *Y) {
  const int64_t Nm = (n < M) ? n : M;
  const int64_t nyq = Nm / 2 + 1;               /* bins 0 .. nyq-1: DC, positive (and +Nm/2 when even) */
  for (int64_t k = 0; k < nyq; ++k) {
    Y[2 * k] = X[2 * k];
    Y[2 * k + 1] = X[2 * k + 1];
  }
  for (int64_t j = 1; j <= Nm - nyq; ++j) {     /* negative frequencies -1 .. -(Nm - nyq) */
    Y[2 * (M - j)] = X[2 * (n - j)];
    Y[2 * (M - j) + 1] = X[2 * (n - j) + 1];
  }
  if (Nm % 2 == 0) {
    const int64_t h = Nm / 2;
    if (M < n) {                                /* truncation: fold X[-h] into Y[+h] */
      Y[2 * h] += X[2 * (n - h)];
      Y[2 * h + 1] += X[2 * (n - h) + 1];
    } else if (M > n) {                         /* padding: split X[+h] over Y[+h] and Y[-h] */
      Y[2 * h] *= 0.5;
      Y[2 * h + 1] *= 0.5;
      Y[2 * (M - h)] = Y[2 * h];
      Y[2 * (M - h) + 1] = Y[2 * h + 1];
    }
  }
}

int orc_pq_resample(int64_t n, int64_t M, const double *x, double *y) {
  if (n < 1 || M < 1) return -1;
  double *X = (double *)malloc(sizeof(double) * 2 * (size_t)n);
  double *Y = (double *)calloc(2 * (size_t)M, sizeof(double));
  if (!X || !Y) {
    free(X);
    free(Y);
    return -2;
  }
  orc_dft(n, x, X, -1);
  pq_bins(n, M, X, Y);
  double *z = (double *)malloc(sizeof(double) * 2 * (size_t)M);
  if (!z) {
    free(X);
    free(Y);
    return -2;
  }
  orc_dft(M, Y, z, +1);
  for (int64_t m = 0; m < n; ++m) {
    y[2 * m] = (m < M) ? z[2 * m] / (double)n : 0.0;
    y[2 * m + 1] = (m < M) ? z[2 * m + 1] / (double)n : 0.0;
  }
  free(X);
  free(Y);
  free(z);
  return 0;
}

/* orc_pq_resample at the `count` output indices idx[] only (for pulses too long for the O(n^2) DFTs):
 * X by the radix-2 FFT (n a power of two), Y as above, then each requested output as the length-M
 * inverse DFT sum written out, y_m = (1/n) sum_k Y_k e^{+i 2 pi (k m mod M) / M} (0 for m >= M). */
int orc_pq_resample_at(int64_t n, int64_t M, const double *x, int64_t count, const int64_t *idx, double *y) {
  if (n < 1 || M < 1 || (n & (n - 1))) return -1;
  double *X = (double *)malloc(sizeof(double) * 2 * (size_t)n);
  double *Y = (double *)calloc(2 * (size_t)M, sizeof(double));
  if (!X || !Y) {
    free(X);
    free(Y);
    return -2;
  }
  memcpy(X, x, sizeof(double) * 2 * (size_t)n);
  orc_fft(n, X, -1);
  pq_bins(n, M, X, Y);
  for (int64_t i = 0; i < count; ++i) {
    const int64_t m = idx[i];
    double re = 0.0, im = 0.0;
    if (m < M) {
      for (int64_t k = 0; k < M; ++k) {
        const int64_t km = (int64_t)(((__int128)k * m) % M);
        const double ang = 2.0 * ORC_PI * (double)km / (double)M;
        const double c = cos(ang), s = sin(ang);
        re += Y[2 * k] * c - Y[2 * k + 1] * s;
        im += Y[2 * k] * s + Y[2 * k + 1] * c;
      }
    }
    y[2 * i] = re / (double)n;
    y[2 * i + 1] = im / (double)n;
  }
  free(X);
  free(Y);
  return 0;
}

/* Doppler correction by FFT P/Q resampling (reading R18): output m samples the input at
 * t = m n / M with M = n + 2 round((n alpha - n) / 2) (an even number of samples added or
 * removed, the paper's exact case), then the carrier term of R10 with beta_eff = n / M. */
int64_t orc_pq_length(int64_t n, double alpha) {
  return n + 2 * (int64_t)llround(0.5 * ((double)n * alpha - (double)n));
}

int orc_doppler_pq(int64_t n, double fs, double fc, double alpha, const double *x, double *y) {
  if (n < 1 || !(alpha > 0.0)) return -1;
  const int64_t M = orc_pq_length(n, alpha);
  if (M < 1) return -1;
  int rc = orc_pq_resample(n, M, x, y);
  if (rc) return rc;
  const double beta_eff = (double)n / (double)M;
  for (int64_t m = 0; m < n; ++m) {
    double psi = fc * (1.0 - beta_eff) * (double)m / fs;
    double r = psi - nearbyint(psi);
    double ang = -2.0 * ORC_PI * r;
    double c = cos(ang), sn = sin(ang);
    double re = y[2 * m], im = y[2 * m + 1];
    y[2 * m] = re * c - im * sn;
    y[2 * m + 1] = re * sn + im * c;
  }
  return 0;
}

/* orc_doppler_pq at the output indices idx[] only (orc_pq_resample_at, then the same carrier term). */
int orc_doppler_pq_at(int64_t n, double fs, double fc, double alpha, const double *x, int64_t count, const int64_t *idx,
                      double *y) {
  if (n < 1 || !(alpha > 0.0)) return -1;
  const int64_t M = orc_pq_length(n, alpha);
  if (M < 1) return -1;
  int rc = orc_pq_resample_at(n, M, x, count, idx, y);
  if (rc) return rc;
  const double beta_eff = (double)n / (double)M;
  for (int64_t i = 0; i < count; ++i) {
    const int64_t m = idx[i];
    double psi = fc * (1.0 - beta_eff) * (double)m / fs;
    double r = psi - nearbyint(psi);
    double ang = -2.0 * ORC_PI * r;
    double c = cos(ang), sn = sin(ang);
    double re = y[2 * i], im = y[2 * i + 1];
    y[2 * i] = re * c - im * sn;
    y[2 * i + 1] = re * sn + im * c;
  }
  return 0;
}

/* ---------------------------------------------------------------------------
 * Batched entry points on complex64 inputs (the GPU's input type),
 * upcast exactly to binary64; pulses are independent and may be run
 * on several host threads (nthreads <= 0: OpenMP default).  Output binary64.
 * stage: 1 = iono, 2 = doppler, 3 = correct = doppler(iono(x)) with a binary64
 * intermediate (reading R7: iono first).
 * ------------------------------------------------------------------------- */
int orc_run_batch_win(int stage, int64_t n, int64_t batch, double fs, double fc, int W, double kb,
                      const double *tec, const double *alpha, const float *x, double *y,
                      int nthreads, int method) {
  int err = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) reduction(| : err)
#endif
  for (int64_t p = 0; p < batch; ++p) {
    double *xin = (double *)malloc(sizeof(double) * 2 * (size_t)n);
    double *tmp = (double *)malloc(sizeof(double) * 2 * (size_t)n);
    if (!xin || !tmp) {
      err |= 1;
      free(xin);
      free(tmp);
      continue;
    }
    const float *xp = x + (size_t)p * 2 * (size_t)n;
    for (int64_t i = 0; i < 2 * n; ++i) xin[i] = (double)xp[i];
    double *yp = y + (size_t)p * 2 * (size_t)n;
    if (stage == 1) {
      err |= orc_iono(n, fs, fc, tec[p], method, xin, yp) != 0;
    } else if (stage == 2) {
      err |= orc_doppler_win(n, W, fs, fc, alpha[p], kb, xin, yp) != 0;
    } else {
      err |= orc_iono(n, fs, fc, tec[p], method, xin, tmp) != 0;
      err |= orc_doppler_win(n, W, fs, fc, alpha[p], kb, tmp, yp) != 0;
    }
    free(xin);
    free(tmp);
  }
  return err ? -1 : 0;
}

int orc_run_batch(int stage, int64_t n, int64_t batch, double fs, double fc, int W,
                  const double *tec, const double *alpha, const float *x, double *y,
                  int nthreads, int method) {
  return orc_run_batch_win(stage, n, batch, fs, fc, W, 0.0, tec, alpha, x, y, nthreads, method);
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
