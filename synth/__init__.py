"""Seeded synthetic workload generators shared by the tests, smoke() and bench.py.

This module holds input generation only -- waveform synthesis (chirps, codes,
noise) and per-pulse parameter draws.  It contains none of the correction
method's arithmetic (no ionospheric phase, no resampling), so both the CUDA
path and the FP64 oracle can consume identical complex64 inputs without sharing
method code.  Recipes are the ones stated in DESIGN.md section "Input recipe"
(SURVEY section 8(d)): absolute-RF complex samples at fs = 2.048 GHz,
waveform bank seed 4951, per-pulse parameter seed 4952.
"""
from __future__ import annotations

import numpy as np

FS_PAPER = 2.048e9          # P:L311 / P:L333
TECU = 1e16                 # 1 TEC unit in electrons / m^2
BANK_SEED = 4951
PARAM_SEED = 4952
# alpha range for |v| <= 5 km/s (Eq. 13 with v = +-5000 m/s): 1 +- 3.33569658541e-5
ALPHA_SPAN_5KMS = 3.33569658541e-5  # alpha(5 km/s) - 1
C_LIGHT = 299792458.0


def _t(n: int, fs: float) -> np.ndarray:
    return np.arange(n, dtype=np.float64) / fs


def lfm(n: int, fs: float, f0: float, B: float, T: float, offset: int = 0, fc: float = 0.0,
        time_scale: float = 1.0, extra_phase_hz: float = 0.0) -> np.ndarray:
    """Unit-amplitude LFM exp(i 2 pi ((f0-fc) tau + B tau^2/(2T))) for tau in [0, T), zero elsewhere.

    tau = time_scale * (t - offset/fs).  time_scale != 1 evaluates the chirp on a
    scaled time axis (used to synthesise an analytically dilated echo S(alpha t));
    extra_phase_hz adds exp(i 2 pi extra t) (a downconversion residue)."""
    t = _t(n, fs)
    tau = time_scale * (t - offset / fs)
    inside = (tau >= 0) & (tau < T)
    cyc = (f0 - fc) * tau + 0.5 * B * tau * tau / T + extra_phase_hz * t
    x = np.exp(2j * np.pi * (cyc - np.floor(cyc)))
    x[~inside] = 0
    return x


def tukey(n_win: int, frac: float = 0.1) -> np.ndarray:
    """Tukey (tapered cosine) window with total taper fraction `frac`."""
    if n_win <= 1:
        return np.ones(max(n_win, 0))
    w = np.ones(n_win)
    m = int(np.floor(frac * (n_win - 1) / 2.0))
    if m > 0:
        k = np.arange(m + 1)
        ramp = 0.5 * (1 - np.cos(np.pi * k / m))
        w[: m + 1] = ramp
        w[-(m + 1):] = ramp[::-1]
    return w


def tukey_lfm(n: int, fs: float, f0: float, B: float, T: float, offset: int, time_scale: float = 1.0,
              frac: float = 0.1) -> np.ndarray:
    """LFM with a Tukey envelope evaluated at tau = time_scale (t - offset/fs) (analytic dilation)."""
    t = _t(n, fs)
    tau = time_scale * (t - offset / fs)
    inside = (tau >= 0) & (tau < T)
    cyc = f0 * tau + 0.5 * B * tau * tau / T
    x = np.exp(2j * np.pi * (cyc - np.floor(cyc)))
    # continuous Tukey envelope
    u = np.clip(tau / T, 0, 1)
    env = np.ones(n)
    a = frac / 2
    lo = u < a
    hi = u > 1 - a
    env[lo] = 0.5 * (1 - np.cos(np.pi * u[lo] / a))
    env[hi] = 0.5 * (1 - np.cos(np.pi * (1 - u[hi]) / a))
    x = x * env
    x[~inside] = 0
    return x


def tone(n: int, fs: float, f: float) -> np.ndarray:
    cyc = f * _t(n, fs)
    return np.exp(2j * np.pi * (cyc - np.floor(cyc)))


def bin_tone(n: int, k0: int) -> np.ndarray:
    """exp(i 2 pi k0 t / n) with the exponent reduced in integers (exact bin-centred tone)."""
    t = np.arange(n, dtype=np.int64)
    return np.exp(2j * np.pi * ((k0 * t) % n) / n)


def gaussian_packet(n: int, fs: float, f: float, sigma: float, center: float) -> np.ndarray:
    t = np.arange(n, dtype=np.float64)
    cyc = f * t / fs
    return np.exp(-0.5 * ((t - center) / sigma) ** 2) * np.exp(2j * np.pi * (cyc - np.floor(cyc)))


def complex_gaussian(n: int, seed: int, batch: int | None = None) -> np.ndarray:
    rng = np.random.default_rng(seed)
    shape = (n,) if batch is None else (batch, n)
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2.0)


def bandlimited_noise(n: int, fs: float, f_lo: float, f_hi: float, seed: int, fc: float = 0.0) -> np.ndarray:
    """Complex Gaussian noise brick-wall limited to [f_lo, f_hi] (absolute RF, bin k -> fc + fftfreq)."""
    X = np.fft.fft(complex_gaussian(n, seed))
    f = fc + np.fft.fftfreq(n, 1.0 / fs)
    X[(f < f_lo) | (f > f_hi)] = 0
    x = np.fft.ifft(X)
    return x / np.sqrt(np.mean(np.abs(x) ** 2))


def raised_cosine(t_over_Tc: np.ndarray, rolloff: float) -> np.ndarray:
    x = np.asarray(t_over_Tc, dtype=np.float64)
    out = np.sinc(x) * np.cos(np.pi * rolloff * x)
    den = 1 - (2 * rolloff * x) ** 2
    sing = np.abs(den) < 1e-10
    out = np.where(sing, np.pi / 4 * np.sinc(1 / (2 * rolloff)), out / np.where(sing, 1, den))
    return out


def bpsk(n: int, fs: float, chip_rate: float, carrier: float, duration: float, offset: int,
         seed: int, rolloff: float = 0.25, fc: float = 0.0) -> np.ndarray:
    """Random BPSK code, raised-cosine shaped, on `carrier` (absolute RF when fc = 0)."""
    rng = np.random.default_rng(seed)
    nchips = int(round(duration * chip_rate))
    chips = rng.integers(0, 2, nchips) * 2.0 - 1.0
    L = int(round(duration * fs))
    t = np.arange(L) / fs
    u = t * chip_rate
    env = np.zeros(L)
    span = 8
    for c in range(nchips):
        lo = max(0, int((c - span) * fs / chip_rate))
        hi = min(L, int((c + span + 1) * fs / chip_rate) + 1)
        env[lo:hi] += chips[c] * raised_cosine(u[lo:hi] - c - 0.5, rolloff)
    x = np.zeros(n, dtype=np.complex128)
    tt = np.arange(n) / fs
    cyc = (carrier - fc) * tt
    seg = slice(offset, min(n, offset + L))
    x[seg] = env[: seg.stop - seg.start]
    return x * np.exp(2j * np.pi * (cyc - np.floor(cyc)))


def p4(n: int, fs: float, nchips: int, carrier: float, duration: float, offset: int, fc: float = 0.0) -> np.ndarray:
    """P4 polyphase code: phase_k = pi (k-1)^2 / N - pi (k-1), rectangular chips."""
    L = int(round(duration * fs))
    idx = np.minimum((np.arange(L) * nchips) // L, nchips - 1)
    ph = np.pi * idx.astype(np.float64) ** 2 / nchips - np.pi * idx
    x = np.zeros(n, dtype=np.complex128)
    seg = slice(offset, min(n, offset + L))
    x[seg] = np.exp(1j * ph[: seg.stop - seg.start])
    cyc = (carrier - fc) * np.arange(n) / fs
    return x * np.exp(2j * np.pi * (cyc - np.floor(cyc)))


# ----------------------------------------------------------------------------- configs
def c1_pulse(variant: str = "a") -> dict:
    """C1: n = 4096, one LFM pulse.  (a) abs-RF fs = 2.048 GHz, f0 = 413 MHz, B = 18 MHz,
    T = 1 us at offset 1024; (b) baseband fs = 51.2 MHz, fc = 422 MHz, T = 40 us."""
    n = 4096
    if variant == "a":
        fs, fc = FS_PAPER, 0.0
        x = lfm(n, fs, 413e6, 18e6, 1e-6, offset=1024)
    else:
        fs, fc = 51.2e6, 422e6
        x = lfm(n, fs, 413e6, 18e6, 40e-6, offset=1024, fc=fc)
    return dict(n=n, fs=fs, fc=fc, x=x.astype(np.complex64), tec=1e18, alpha=1 + 1e-5, W=16)


def c2_batch(batch: int = 256, n: int = 1 << 16) -> dict:
    """C2: phase-coded (BPSK, raised cosine 0.25, 18 Mchip/s, 422 MHz carrier, 16 us at offset n/4),
    TEC sweep tec_p = p TECU."""
    fs = FS_PAPER
    dur = 16e-6 * n / (1 << 16)
    x = bpsk(n, fs, 18e6, 422e6, dur, n // 4, seed=BANK_SEED).astype(np.complex64)
    xb = np.broadcast_to(x, (batch, n)).copy()
    tec = np.arange(batch, dtype=np.float64) * TECU
    return dict(n=n, fs=fs, fc=0.0, x=xb, tec=tec)


def waveform_bank(n: int, fs: float = FS_PAPER, count: int = 16, T: float = 100e-6, seed: int = BANK_SEED) -> np.ndarray:
    """C4 mixed bank: LFM up / LFM down / BPSK / P4 / band-limited noise (413-431 MHz), T at a
    seeded random offset inside the n-sample window.  Returns complex64 [count, n]."""
    rng = np.random.default_rng(seed)
    L = int(round(T * fs))
    if L >= n:
        T = 0.5 * n / fs
        L = int(round(T * fs))
    bank = np.zeros((count, n), dtype=np.complex64)
    for i in range(count):
        off = int(rng.integers(0, max(1, n - L)))
        kind = i % 5
        if kind == 0:
            x = lfm(n, fs, 413e6, 18e6, T, off)
        elif kind == 1:
            x = lfm(n, fs, 431e6, -18e6, T, off)
        elif kind == 2:
            x = bpsk(n, fs, 18e6, 422e6, T, off, seed=seed + i)
        elif kind == 3:
            x = p4(n, fs, 1800, 422e6, T, off)
        else:
            x = bandlimited_noise(n, fs, 413e6, 431e6, seed=seed + i)
        bank[i] = x.astype(np.complex64)
    return bank


def pulse_params(batch: int, seed: int = PARAM_SEED, tec_max_tecu: float = 200.0,
                 v_max_mps: float = 5000.0) -> tuple[np.ndarray, np.ndarray]:
    """SURVEY 8(d) C4 recipe: per-pulse TEC ~ U[0, tec_max] TECU and radial velocity
    v ~ U[-v_max, +v_max] mapped to alpha = (1 + v/c) / (1 - v/c) (the Doppler model of Eq. 13's
    context) -- the workload's parameters, not part of the correction."""
    rng = np.random.default_rng(seed)
    tec = rng.uniform(0.0, tec_max_tecu, batch) * TECU
    v = rng.uniform(-v_max_mps, v_max_mps, batch)
    alpha = (1.0 + v / C_LIGHT) / (1.0 - v / C_LIGHT)
    return tec, alpha


def pulse_train(batch: int, n: int, bank_count: int = 16, fs: float = FS_PAPER) -> dict:
    """C4 pulse train: pulse p is bank[p % bank_count]."""
    bank = waveform_bank(n, fs, bank_count)
    tec, alpha = pulse_params(batch)
    return dict(n=n, fs=fs, fc=0.0, bank=bank, index=np.arange(batch) % bank_count, tec=tec, alpha=alpha, W=32)
