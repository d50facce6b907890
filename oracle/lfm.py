"""LFM analytic truth and matched-filter metric used to pin the oracle.

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py header).  Plain numpy, FP64.

* cubic_frequency: the paper's closed-form real root of the predistortion cubic,
  Eq. 9-12 of Eq. 2.
* cubic_frequency_newton: the same root of Eq. 2 by Newton iteration (a second,
  independent evaluation used to pin the closed form).
* cubic_waveform: phase by trapezoidal integration of f(t) at dt = 1/fs
  (Fig. 2 caption P:L311).
* matched_filter_loss: cross-correlation peak loss (the paper's metric is
  "SNR loss" from matched filtering; its formula is unstated, we
  use the Cauchy-Schwarz-normalised peak, reading R13 in DESIGN.md).
"""
from __future__ import annotations

import numpy as np

C_LIGHT = 299792458.0


def _A_D(t, f0, B, T, k2):
    A = f0 + B * t / T - 2.0 * k2 * B / (C_LIGHT * f0 * f0 * T)
    D = 2.0 * k2 * B / (C_LIGHT * T)
    return A, D


def cubic_frequency(t, f0: float, B: float, T: float, k2: float) -> np.ndarray:
    """f(t) = (1/3)(A - omega - chi/omega), Eq. 9 with chi (Eq. 10), psi (Eq. 11), omega (Eq. 12)."""
    t = np.asarray(t, dtype=np.float64)
    A, D = _A_D(t, f0, B, T, k2)
    if k2 == 0.0:
        return A.copy() if isinstance(A, np.ndarray) else np.float64(A)
    chi = A * A                                     # Eq. 10
    psi = -2.0 * A ** 3 - 27.0 * D                  # Eq. 11
    omega = np.cbrt((psi + np.sqrt(psi * psi - 4.0 * chi ** 3)) / 2.0)  # Eq. 12 (real cube root)
    return (A - omega - chi / omega) / 3.0          # Eq. 9


def cubic_residual(f, t, f0, B, T, k2):
    """Left-hand side of Eq. 2: f^3 - A f^2 - D."""
    A, D = _A_D(np.asarray(t, dtype=np.float64), f0, B, T, k2)
    return f ** 3 - A * f ** 2 - D


def cubic_frequency_newton(t, f0: float, B: float, T: float, k2: float, iters: int = 60) -> np.ndarray:
    """Root of Eq. 2 by Newton's method started at the undistorted chirp f0 + B t / T."""
    t = np.asarray(t, dtype=np.float64)
    A, D = _A_D(t, f0, B, T, k2)
    f = f0 + B * t / T
    for _ in range(iters):
        g = f ** 3 - A * f ** 2 - D
        dg = 3.0 * f ** 2 - 2.0 * A * f
        f = f - g / dg
    return f


def cubic_waveform(f0: float, B: float, T: float, k2: float, fs: float, n_samples: int | None = None) -> np.ndarray:
    """Unit-amplitude predistorted LFM: phase = 2 pi * trapezoidal integral of f(t), dt = 1/fs."""
    if n_samples is None:
        n_samples = int(round(T * fs))
    t = np.arange(n_samples, dtype=np.float64) / fs
    f = cubic_frequency(t, f0, B, T, k2)
    # trapezoid: phi_i = sum_{j<i} (f_j + f_{j+1}) / 2 * dt, in cycles, kept mod 1 via cumulative sum of increments
    inc = 0.5 * (f[:-1] + f[1:]) / fs
    cyc = np.concatenate([[0.0], np.cumsum(inc)])
    cyc = cyc - np.floor(cyc)
    return np.exp(2j * np.pi * cyc)


def xcorr_peak(a: np.ndarray, b: np.ndarray) -> float:
    """max over all lags of |sum_t a[t+l] conj(b[t])| (linear correlation via zero-padded FFT)."""
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    L = 1 << int(np.ceil(np.log2(a.size + b.size - 1)))
    A = np.fft.fft(a, L)
    Bf = np.fft.fft(b, L)
    return float(np.max(np.abs(np.fft.ifft(A * np.conj(Bf)))))


def matched_filter_loss_db(received: np.ndarray, reference: np.ndarray) -> float:
    """SNR loss of `received` against `reference`: -20 log10(peak / (|rx| |ref|)).

    0 dB iff received is a delayed, phase-rotated, scaled copy of the reference."""
    p = xcorr_peak(received, reference)
    norm = np.linalg.norm(received) * np.linalg.norm(reference)
    return float(-20.0 * np.log10(p / norm))


def envelope_peak(x: np.ndarray) -> float:
    """Sub-sample location of the |x| maximum (parabolic fit of log|x| around the max)."""
    m = np.abs(np.asarray(x))
    i = int(np.argmax(m))
    if 0 < i < m.size - 1:
        y0, y1, y2 = np.log(m[i - 1]), np.log(m[i]), np.log(m[i + 1])
        den = y0 - 2 * y1 + y2
        if den != 0:
            return i + 0.5 * (y0 - y2) / den
    return float(i)
