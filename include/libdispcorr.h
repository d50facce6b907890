/*
 * libdispcorr -- B200-native (sm_100a) per-pulse dispersion correction.
 *
 * C ABI of the hot path of arXiv 2508.04951 (Vickers, Mack, Osaretin):
 *   stage 1, ionospheric correction (Eq. 15):
 *       S_Tx = F^-1[ F(S_Rx) exp(-4 pi i K2 / (c f)) ],   K2 = 40.308193022 * TEC   (Eq. 1)
 *   stage 2, Doppler time-dilation correction (Eq. 13; Eq. 16):
 *       windowed Whittaker-Shannon (sinc) resampling of each pulse onto t/alpha
 *       using the W samples around each output.
 * Readings of silent passages (bin -> frequency map, window membership, carrier
 * term, ...) are DESIGN.md R1..R13; they are restated at each call below.
 *
 * Conventions shared by every call
 *   - Samples are complex64: interleaved (re, im) IEEE float32 pairs,
 *     laid out pulse-major, float2[batch][n]; pulse p starts at x + p*n.
 *   - Device pointers must be CUDA device (or managed) memory of the plan's
 *     device, 16-byte aligned (torch allocations are 256-byte aligned).
 *   - Per-pulse parameter arrays (tec, alpha) are HOST arrays of `batch`
 *     binary64 values; they are validated and copied before the call returns,
 *     so the caller may reuse them immediately.
 *   - Calls are asynchronous on the plan's stream: DC_OK means "validated and
 *     enqueued".  Asynchronous faults surface as DC_ERR_CUDA from the next call
 *     or from dc_sync().  dc_correct_host() is the one synchronous call.
 *   - A plan must not be used from two host threads at once (it owns scratch and
 *     a parameter staging ring).  Distinct plans are independent.
 *   - Errors are synchronous and nothing is enqueued when a call returns an
 *     error; dc_last_error_message() gives a one-line explanation.
 */
#ifndef LIBDISPCORR_H
#define LIBDISPCORR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DC_VERSION 100 /* 1.0.0 */

typedef struct dc_plan_s *dc_plan_t; /* opaque; created by dc_plan, destroyed by dc_plan_destroy */

typedef enum {
  DC_OK = 0,
  DC_ERR_INVALID_VALUE = 1,      /* a size / rate / parameter outside its documented range */
  DC_ERR_NULL_POINTER = 2,       /* a required pointer is NULL */
  DC_ERR_MISALIGNED = 3,         /* a sample pointer is not 16-byte aligned */
  DC_ERR_ALIASING = 4,           /* y overlaps x where the call requires distinct buffers */
  DC_ERR_OUT_OF_MEMORY = 5,      /* device or pinned-host allocation failed */
  DC_ERR_CUDA = 6,               /* a CUDA runtime error (incl. an earlier asynchronous fault) */
  DC_ERR_UNSUPPORTED_DEVICE = 7, /* device is not compute capability 10.0 (B200, sm_100a) */
  DC_ERR_NOT_DEVICE_MEMORY = 8   /* a sample pointer is not device/managed memory of the plan's device */
} dc_status;

/* Plan for pulses of n complex samples at sample rate fs_hz whose DFT bin k
 * represents absolute frequency f_k = fc_hz + fs_hz*(k - n*[k >= n/2])/n
 * (reading R2; fc_hz = 0 for absolute-RF complex samples as in P:L311), with a
 * W = taps sample sinc window for the Doppler stage.
 *   n      power of two, 2 <= n <= 2^24 (O(N log N) for N = 2^k)
 *   fs_hz  > 0, finite;  fc_hz >= 0, finite
 *   taps   2 <= taps <= 128 and taps <= n (odd or even)
 *   device CUDA device ordinal (must be sm_100)
 *   cuda_stream  cudaStream_t to enqueue on; NULL = legacy default stream
 * Allocates the plan's device scratch, twiddle tables and pinned staging; no
 * kernel runs.  On error *out is set to NULL. */
dc_status dc_plan(dc_plan_t *out, int64_t n, double fs_hz, double fc_hz, int taps, int device,
                  void *cuda_stream);

/* Release everything the plan owns (synchronises the plan's stream first). */
dc_status dc_plan_destroy(dc_plan_t plan);

/* Re-target the plan to another stream of the same device. */
dc_status dc_set_stream(dc_plan_t plan, void *cuda_stream);

/* Block until all work enqueued by this plan is done; reports asynchronous faults. */
dc_status dc_sync(dc_plan_t plan);

/* Ionospheric correction, Eq. 15, IN PLACE on device x[batch][n]:
 *   X = DFT(x) (forward kernel e^{-i 2 pi k t / n});  X_k *= exp(-i 2 pi nu_k) / n with
 *   nu_k = 2 K2 / (c f_k), K2 = dc_k2_per_tec() * tec[p]  (two-way), nu_k = 0 if f_k <= 0
 *   (reading R3); x = IDFT(X).  tec: host double[batch], el/m^2, each finite and >= 0.
 * batch >= 1.  One HBM round trip per pulse for n <= 2^14 (n = 2^14: the in-CTA four-step kernel of
 * regime 1); n > 2^14 uses a three-pass four-step decomposition in place on x. */
dc_status dc_iono(dc_plan_t plan, void *x, int64_t batch, const double *tec);

/* Forward ionospheric model, Eq. 14: the same with exp(+i 2 pi nu_k).
 * Used to synthesise dispersed echoes and the matched-filter reference. */
dc_status dc_iono_distort(dc_plan_t plan, void *x, int64_t batch, const double *tec);

/* Matched-filter reference for dc_compress (the paper's pulse-compression path,
 * fig:pulse_compression_path P:L246-251; "46 us ... during pulse compression").
 * r: device float2[L], 1 <= L <= n, the transmitted reference r_0 .. r_{L-1}; it is
 * zero-padded to n and its DFT R_k is computed on the device and kept (conjugated) in
 * the plan (8n bytes), replacing any earlier reference.  r may be reused as soon as
 * the plan's stream has passed this call.  Any plan size n. */
dc_status dc_set_reference(dc_plan_t plan, const void *r, int64_t L);

/* Pulse compression after the ionospheric correction (reading R16):
 *   z[p][m] = sum_{s=0}^{L-1} y[p][(s + m) mod n] conj(r_s),   y[p] = dc_iono(x[p], tec[p]),
 * i.e. z = F^-1[ F(x) e^{-i 2 pi nu_k} conj(R_k) ] -- the conj(R_k) multiply is fused into the
 * Eq. 15 phase step, so compression costs no HBM bytes beyond dc_iono's.
 * x, z: device float2[batch][n]; z == x (in place) or z disjoint from x (else
 * DC_ERR_ALIASING).  tec: host double[batch] as dc_iono.  DC_ERR_INVALID_VALUE when no
 * reference has been set. */
dc_status dc_compress(dc_plan_t plan, const void *x, void *z, int64_t batch, const double *tec);

/* Doppler correction: y[p][m] = e^{-i 2 pi fc (1 - beta) m / fs} *
 *   sum_{k : -W/2 < k - t_m <= W/2, 0 <= k < n} x[p][k] sinc(t_m - k),   t_m = m * beta,
 *   beta = 1/alpha[p] (binary64), sinc(d) = sin(pi d)/(pi d), sinc(0) = 1   (Eq. 16 windowed;
 *   readings R8-R12).  Output length n; samples outside [0, n) are zero.
 * x, y: device float2[batch][n], must not overlap.  alpha: host double[batch], each finite > 0.
 * alpha[p] == 1 reproduces x[p] bit-exactly. */
dc_status dc_doppler(dc_plan_t plan, const void *x, void *y, int64_t batch, const double *alpha);

/* Doppler correction by FFT P/Q resampling, the paper's second resampling method ("the Fourier
 * transform of the signal has terms removed or added followed by an inverse Fourier transform",
 * P:L206; box filter of N/alpha samples, exact when N - N/alpha is an even integer, P:L292-294;
 * benchmarked in fig:pqbenchmark).  Reading R18, per pulse p:
 *   M = n + 2 round((n alpha[p] - n) / 2)   (an even number of samples added or removed)
 *   X = DFT_n(x[p]);  Y = X with the bins of |signed frequency| >= min(n, M)/2 removed (M < n: the
 *   -Nyquist bin folded into +Nyquist) or zeros added (M > n: the Nyquist bin split in half over +-);
 *   y[p][m] = (1/n) sum_k Y_k e^{+i 2 pi k m / M} * e^{-i 2 pi fc (1 - n/M) m / fs}  for m < min(n, M),
 *   0 for min(n, M) <= m < n.  M == n (|n alpha - n| < 1) returns x[p] bit-exactly (no work).
 * The length-M inverse DFT is a chirp-z (Bluestein) convolution of length 2n on the device.
 * x, y: device float2[batch][n], must not overlap.  alpha: host double[batch], finite > 0, with
 * 2 <= M <= 8n.  n <= 2^23.  The plan keeps a cache of per-M convolution tables (16n bytes each,
 * <= 1 GiB) and 1 GiB-bounded group buffers, allocated on the first call. */
dc_status dc_doppler_pq(dc_plan_t plan, const void *x, void *y, int64_t batch, const double *alpha);

/* Taper of the Doppler stage's sinc window (reading R17; "taper window size, taper"):
 * Kaiser window of shape `kaiser` over the W = taps window, half-width L = W/2,
 *   h(d) = sinc(d) I0(kaiser sqrt(1 - (d/L)^2)) / I0(kaiser),  d = t_m - k,
 * used by dc_doppler and dc_correct from the next call on.  kaiser = 0 (the default) is the
 * rectangular window of R11.  kaiser must be finite and in [0, 12] (else DC_ERR_INVALID_VALUE).
 * The centre tap keeps weight 1, so alpha = 1 still reproduces x exactly. */
dc_status dc_set_taper(dc_plan_t plan, double kaiser);

/* Window of the Doppler stage's sinc taps (reading R17; "taper"), used by dc_doppler and
 * dc_correct from the next call on, over the W = taps window with half-width L = W/2, d = t_m - k:
 *   DC_WINDOW_RECT    h(d) = sinc(d)                                   (R11, the default; param ignored)
 *   DC_WINDOW_KAISER  h(d) = sinc(d) I0(param sqrt(1 - (d/L)^2)) / I0(param), param in [0, 12]
 *                     (dc_set_taper(plan, param))
 *   DC_WINDOW_HANN    h(d) = sinc(d) (1 + cos(pi d / L)) / 2           (param ignored)
 * The centre tap keeps weight 1, so alpha = 1 still reproduces x exactly.  DC_ERR_INVALID_VALUE for an
 * unknown kind or a Kaiser param outside [0, 12]. */
enum { DC_WINDOW_RECT = 0, DC_WINDOW_KAISER = 1, DC_WINDOW_HANN = 2 };
dc_status dc_set_window(dc_plan_t plan, int kind, double param);

/* dc_correct = dc_doppler(dc_iono(x)) (iono first, reading R7), x left unchanged,
 * result in y (must not overlap x).  Pulses run in launch groups of <= 2 GiB; the
 * ionospheric result of a group is kept in a plan-owned device buffer (allocated on the
 * first call, sized to min(batch, group)) between the stages -- except for single-CTA pulses
 * (n = 2^10 .. 2^14) with W = 16 or 32, the rectangular window and |1/alpha - 1| within the
 * first/second-order range, where one fused kernel reads x and writes y once (16 B/sample). */
dc_status dc_correct(dc_plan_t plan, const void *x, void *y, int64_t batch, const double *tec,
                     const double *alpha);

/* dc_correct on HOST buffers (pageable or pinned), synchronous: chunks of pulses are
 * copied host->device, corrected and copied back with copy/compute overlap on the
 * plan's stream plus an internal copy stream.  x_host, y_host: complex64[batch][n]. */
dc_status dc_correct_host(dc_plan_t plan, const void *x_host, void *y_host, int64_t batch,
                          const double *tec, const double *alpha);

/* Plan introspection (for tests and the benchmark). */
typedef struct {
  int64_t n;             /* samples per pulse */
  int log2n;
  int taps;              /* sinc window W */
  int regime;            /* 0 = single-CTA fused FFT (n <= 8192), 1 = four-step (n = 2^14: in one CTA, one HBM round trip) */
  int64_t n1, n2;        /* four-step split n = n1 * n2 (t = n2 t1 + t2, k = k1 + n1 k2); 0 if regime 0 */
  int64_t chunk_pulses;  /* pulses per dc_correct chunk (scratch = chunk_pulses * n * 8 bytes) */
  int64_t scratch_bytes; /* device scratch owned by the plan */
  int sm_count;          /* multiprocessors of the plan's device */
  int64_t kernel_launches; /* kernels this plan has launched so far */
} dc_plan_info_t;
dc_status dc_plan_info(dc_plan_t plan, dc_plan_info_t *info);

/* Per-kernel-class timing (for the benchmark's roofline figures).  When enabled, every kernel
 * the plan launches is bracketed by CUDA events on the plan's stream; dc_profile_read()
 * synchronises the stream and returns, per class, the launches, summed device milliseconds and
 * samples processed since the last reset.  Classes: DC_K_IONO_SMALL (regime-0 fused FFT ->
 * phase -> IFFT; also n = 2^14's in-CTA four-step), DC_K_FOURSTEP_A/B/C (regime-1 passes), DC_K_DOPPLER (sinc resampler),
 * DC_K_PQ (one record per dc_doppler_pq launch group: all of its kernels), DC_K_CORRECT_FUSED (the
 * single-round-trip dc_correct kernel of short pulses: n = 2^10 .. 2^14, W = 16 or 32, no taper). */
enum { DC_K_IONO_SMALL = 0, DC_K_FOURSTEP_A = 1, DC_K_FOURSTEP_B = 2, DC_K_FOURSTEP_C = 3, DC_K_DOPPLER = 4,
       DC_K_PQ = 5, DC_K_CORRECT_FUSED = 6, DC_K_CLASSES = 7 };
typedef struct {
  int64_t launches[DC_K_CLASSES];
  double ms[DC_K_CLASSES];
  int64_t samples[DC_K_CLASSES];
} dc_profile_t;
dc_status dc_profile_enable(dc_plan_t plan, int enable); /* also resets the counters */
dc_status dc_profile_read(dc_plan_t plan, dc_profile_t *out);

/* Human-readable name of a status code (static string). */
const char *dc_status_string(dc_status s);

/* One-line explanation of the most recent error on the calling thread ("" if none). */
const char *dc_last_error_message(void);

/* alpha = (1 + v/c) / (1 - v/c), v > 0 approaching; NaN if |v| >= c or v not finite. */
double dc_alpha_from_velocity(double v_r_mps);

/* K2 / TEC = q_e^2 / (8 pi^2 m_e eps0) (Eq. 1, CODATA 2018) = 40.308193022 m^3 s^-2 per el/m^2. */
double dc_k2_per_tec(void);

int dc_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LIBDISPCORR_H */
