"""Pins of the FP64 oracle against what the paper and mathematics fix (CPU only).

Each test names the passage it pins.  These tests must catch a dropped term,
a wrong sign, a wrong index or a transposed operand anywhere in oracle/.
"""
import os

import numpy as np
import pytest

import synth
from oracle import lfm as L
from oracle import oracle as O
from golden_io import read_golden

C = 299792458.0


# --------------------------------------------------------------------------- constants (Eq. 1, Eq. 13)
def test_k2_constant_standard_value(golden_dir):
    rows = dict((r[0], r[1]) for r in read_golden(os.path.join(golden_dir, "paper_values.txt")))
    approx, tol = float(rows["k2_per_tec_approx"]), float(rows["k2_per_tec_reltol"])
    k = O.k2_per_tec()
    assert abs(k / approx - 1) < tol                       # ~40.31
    assert abs(k - 40.308193022) < 1e-8                     # CODATA 2018 closed form


def test_group_delay_values():
    # tau(413 MHz, 1e18) ~ 7.88e-7 s
    assert abs(O.group_delay(413e6, 1e18) - 7.882655e-7) < 1e-12
    # f^-2 scaling (Eq. 1): tau(2f) = tau(f)/4 and linear in TEC
    assert O.group_delay(826e6, 1e18) == pytest.approx(O.group_delay(413e6, 1e18) / 4, rel=1e-15)
    assert O.group_delay(413e6, 2e18) == pytest.approx(2 * O.group_delay(413e6, 1e18), rel=1e-15)
    assert O.group_delay(413e6, 0.0) == 0.0
    # phase scale nu(413 MHz, 100 TECU) = 651.107 cycles = 2 tau f (two-way)
    assert O.iono_phase_cycles(413e6, 1e18) == pytest.approx(651.1073, abs=1e-3)
    assert O.iono_phase_cycles(-1e6, 1e18) == 0.0 and O.iono_phase_cycles(0.0, 1e18) == 0.0


def test_alpha_from_velocity():
    assert O.alpha_from_velocity(0.0) == 1.0
    assert O.alpha_from_velocity(5000.0) - 1 == pytest.approx(3.33569658541e-5, rel=1e-9)
    for v in (1e3, 1e4, 1e5, 1e6):
        assert abs(O.alpha_from_velocity(v) * O.alpha_from_velocity(-v) - 1) < 1e-15
    assert O.alpha_from_velocity(1000.0) > 1  # approaching => alpha > 1


# --------------------------------------------------------------------------- DFT core
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 12, 16, 64, 100])
def test_direct_dft_vs_numpy(n):
    x = synth.complex_gaussian(n, seed=n)
    assert np.allclose(O.dft(x, -1), np.fft.fft(x), rtol=0, atol=1e-12 * max(1, n))
    assert np.allclose(O.dft(x, +1) / n, np.fft.ifft(x), rtol=0, atol=1e-12)


@pytest.mark.parametrize("p", list(range(1, 13)))
def test_radix2_fft_vs_direct_and_numpy(p):
    n = 1 << p
    x = synth.complex_gaussian(n, seed=100 + p)
    X = O.fft(x)
    ref = np.fft.fft(x)
    assert np.linalg.norm(X - ref) / np.linalg.norm(ref) < 1e-13
    if n <= 1024:
        D = O.dft(x)
        assert np.linalg.norm(X - D) / np.linalg.norm(D) < 1e-13
    assert np.linalg.norm(O.fft(X, +1) / n - x) / np.linalg.norm(x) < 1e-14


def test_radix2_fft_large_vs_numpy():
    n = 1 << 18
    x = synth.complex_gaussian(n, seed=7)
    X = O.fft(x)
    ref = np.fft.fft(x)
    assert np.linalg.norm(X - ref) / np.linalg.norm(ref) < 1e-12


# --------------------------------------------------------------------------- iono: Eq. 15 / Eq. 14
def test_bin_frequency_mapping():
    n, fs, fc = 16, 1.6e9, 0.0
    f = [O.bin_frequency(k, n, fs, fc) for k in range(n)]
    assert np.allclose(f, fc + np.fft.fftfreq(n, 1 / fs))  # numpy convention; Nyquist bin negative
    assert O.bin_frequency(8, 16, 16.0, 100.0) == 92.0


def test_iono_tec0_identity():
    x = synth.complex_gaussian(1024, seed=1)
    y = O.iono(x, 2.048e9, 0.0, 0.0)
    assert np.max(np.abs(y - x)) < 1e-14


def test_iono_golden_impulse(golden_dir):
    rows = read_golden(os.path.join(golden_dir, "G1_iono_impulse.txt"))
    p = [r for r in rows if r[0] == "params"][0]
    n, fs, fc, tec = int(p[1]), float(p[2]), float(p[3]), float(p[4])
    x = np.zeros(n, complex)
    x[0] = 1
    y = O.iono(x, fs, fc, tec)
    yd = O.iono(x, fs, fc, tec, direct=True)
    for r in rows:
        if r[0] == "nu":
            k = int(r[1])
            assert O.iono_phase_cycles(O.bin_frequency(k, n, fs, fc), tec) == pytest.approx(float(r[2]), abs=1e-8)
        if r[0] == "y":
            i = int(r[1])
            assert abs(y[i] - complex(float(r[2]), float(r[3]))) < 1e-11
            assert abs(yd[i] - complex(float(r[2]), float(r[3]))) < 1e-11
    assert np.linalg.norm(y) == pytest.approx(1.0, abs=1e-14)


def test_iono_golden_bin_tone(golden_dir):
    rows = read_golden(os.path.join(golden_dir, "G1b_iono_bin_tone.txt"))
    p = [r for r in rows if r[0] == "params"][0]
    n, fs, fc, tec = int(p[1]), float(p[2]), float(p[3]), float(p[4])
    k0 = int([r for r in rows if r[0] == "k0"][0][1])
    x = synth.bin_tone(n, k0)
    y = O.iono(x, fs, fc, tec)
    nu = float([r for r in rows if r[0] == "nu"][0][2])
    ratio = y / x
    assert np.ptp(ratio.real) < 1e-13 and np.ptp(ratio.imag) < 1e-13
    assert abs(ratio[0] - np.exp(-2j * np.pi * nu)) < 1e-9
    y0 = [r for r in rows if r[0] == "y"][0]
    assert abs(y[0] - complex(float(y0[2]), float(y0[3]))) < 1e-11


@pytest.mark.parametrize("k0", [1, 100, 511, 512, 700, 1023])
def test_iono_tone_is_eigenvector(k0):
    # A bin-centred tone is a DFT eigenvector, so Eq. 15 multiplies it by exp(-i 2 pi nu_k0) with
    # nu = 2 tau(f) f (two-way) at f = fc + fftfreq(k0) -- or by 1 if f <= 0.
    n, fs, fc, tec = 1024, 1.024e9, 0.0, 3e17
    x = synth.bin_tone(n, k0)
    y = O.iono(x, fs, fc, tec)
    f = np.fft.fftfreq(n, 1 / fs)[k0] + fc
    nu = 2 * O.group_delay(f, tec) * f if f > 0 else 0.0
    assert np.max(np.abs(y - x * np.exp(-2j * np.pi * (nu - np.rint(nu))))) < 1e-11


def test_iono_parseval_roundtrip_linearity():
    n, fs = 4096, 2.048e9
    x1 = synth.complex_gaussian(n, 11)
    x2 = synth.complex_gaussian(n, 12)
    y1 = O.iono(x1, fs, 0.0, 1e18)
    assert abs(np.linalg.norm(y1) / np.linalg.norm(x1) - 1) < 1e-14          # unit-modulus filter
    back = O.iono(y1, fs, 0.0, 1e18, distort=True)                            # Eq. 14 after Eq. 15
    assert np.linalg.norm(back - x1) / np.linalg.norm(x1) < 1e-14
    a, b = 0.3 - 1.2j, 2.0 + 0.5j
    lhs = O.iono(a * x1 + b * x2, fs, 0.0, 1e18)
    rhs = a * y1 + b * O.iono(x2, fs, 0.0, 1e18)
    assert np.linalg.norm(lhs - rhs) / np.linalg.norm(rhs) < 1e-14


def test_iono_fft_equals_direct_dft():
    x = synth.complex_gaussian(512, 5)
    a = O.iono(x, 51.2e6, 422e6, 7e17)
    b = O.iono(x, 51.2e6, 422e6, 7e17, direct=True)
    assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-13


@pytest.mark.parametrize("f_carrier", [400e6, 440e6])
def test_sign_gaussian_packet_group_delay(f_carrier):
    # Eq. 14 (distortion) delays the envelope by the two-way group delay 2 tau(f);
    # Eq. 15 (correction) advances it by the same amount.  Closed form: shift = 2 K2/(c f^2) fs samples.
    n, fs, tec, sigma = 1 << 15, 2.048e9, 1e18, 2000.0
    x = synth.gaussian_packet(n, fs, f_carrier, sigma, center=n / 2)
    expect = 2 * O.group_delay(f_carrier, tec) * fs
    assert expect == pytest.approx(3442.0 if f_carrier == 400e6 else 2844.6, abs=0.1)
    p0 = L.envelope_peak(x)
    dist = L.envelope_peak(O.iono(x, fs, 0.0, tec, distort=True)) - p0
    corr = L.envelope_peak(O.iono(x, fs, 0.0, tec)) - p0
    assert dist == pytest.approx(expect, abs=2.0)
    assert corr == pytest.approx(-expect, abs=2.0)


# --------------------------------------------------------------------------- Fig. 2 CUBIC pin
def test_cubic_closed_form_matches_newton_and_golden(golden_dir):
    rows = read_golden(os.path.join(golden_dir, "G3_cubic.txt"))
    p = [float(v) for v in [r for r in rows if r[0] == "params"][0][1:]]
    f0, B, T, tec = p
    k2 = O.k2_per_tec() * tec
    t = np.linspace(0, T, 1001)
    fc = L.cubic_frequency(t, f0, B, T, k2)
    fn = L.cubic_frequency_newton(t, f0, B, T, k2)
    assert np.max(np.abs(fc - fn)) < 1e-3                    # Eq. 9-12 vs Eq. 2 by Newton (Hz)
    assert np.all(np.diff(fc) > 0)
    for r in rows:
        if r[0] == "f":
            assert L.cubic_frequency(np.array([float(r[1])]), f0, B, T, k2)[0] == pytest.approx(float(r[2]), abs=2e-3)
    # k2 = 0 reduces Eq. 2 to the undistorted chirp f0 + B t / T
    assert np.allclose(L.cubic_frequency(t, f0, B, T, 0.0), f0 + B * t / T, rtol=0, atol=1e-6)


def test_fig2_fft_correction_vs_cubic_truth(golden_dir):
    # PAPER Fig. 2 caption / P:L305: "CUBIC (*) FFT ... lost < 0.01 dB SNR" at
    # f0 = 413 MHz, B = 18 MHz, fs = 2.048 GHz, E = 100e16, T = 100 us; N = 2^19.
    vals = dict((r[0], float(r[1])) for r in read_golden(os.path.join(golden_dir, "paper_values.txt")))
    f0, B, fs, tec, T = (vals["fig2_f0_hz"], vals["fig2_B_hz"], vals["fig2_fs_hz"], vals["fig2_tec"], vals["fig2_T_s"])
    n = 1 << 19
    x = synth.lfm(n, fs, f0, B, T, offset=1 << 17)
    cub = L.cubic_waveform(f0, B, T, O.k2_per_tec() * tec, fs)
    loss = L.matched_filter_loss_db(O.iono(x, fs, 0.0, tec), cub)
    assert loss < vals["fig2_fft_vs_cubic_loss_db_max"]
    assert loss == pytest.approx(0.00645, abs=5e-4)           # SURVEY 8c reproduction
    # the flipped sign (a plausible silent mistake) loses dB-scale SNR
    assert L.matched_filter_loss_db(O.iono(x, fs, 0.0, tec, distort=True), cub) > 5.0
    # uncorrected dispersion loss (context) ~1.31 dB
    assert 1.2 < L.matched_filter_loss_db(x, cub) < 1.4
    # same pin at baseband: fc = 422 MHz with fs = 204.8 MHz covering 413-431 MHz (reading R2)
    fsb, fcb, nb = 204.8e6, 422e6, 1 << 15
    xb = synth.lfm(nb, fsb, f0, B, T, offset=1000, fc=fcb)
    tb = np.arange(int(round(T * fsb))) / fsb
    fb = L.cubic_frequency(tb, f0, B, T, O.k2_per_tec() * tec) - fcb
    cycb = np.concatenate([[0.0], np.cumsum(0.5 * (fb[:-1] + fb[1:]) / fsb)])
    cubb = np.exp(2j * np.pi * (cycb - np.floor(cycb)))
    assert L.matched_filter_loss_db(O.iono(xb, fsb, fcb, tec), cubb) < vals["fig2_fft_vs_cubic_loss_db_max"]


# --------------------------------------------------------------------------- doppler: Eq. 16 + window
def test_doppler_alpha_one_bit_exact():
    x = synth.complex_gaussian(777, 3)
    for W in (2, 7, 16, 32):
        y = O.doppler(x, W, 2.048e9, 0.0, 1.0)
        assert np.array_equal(y, x)
    y = O.doppler(x, 16, 51.2e6, 422e6, 1.0)  # carrier term vanishes at beta = 1
    assert np.array_equal(y, x)


def test_doppler_golden(golden_dir):
    rows = read_golden(os.path.join(golden_dir, "G2_doppler.txt"))
    cases = {r[1]: (int(r[2]), float(r[3])) for r in rows if r[0] == "case"}
    x = np.arange(16) + 1j * (16 - np.arange(16))
    out = {name: O.doppler(x, W, 16e6, fc, 1.25) for name, (W, fc) in cases.items()}
    for r in rows:
        if r[0] == "y":
            assert abs(out[r[1]][int(r[2])] - complex(float(r[3]), float(r[4]))) < 1e-10


def test_doppler_integer_positions_direction():
    # alpha = 2 => beta = 1/2: output m samples the input at t = m/2 (resampling onto t/alpha,
    # undoing S(alpha t), Eq. 13).  At integer t the normalised sinc is a Kronecker delta.
    x = synth.complex_gaussian(64, 9)
    y = O.doppler(x, 8, 1.0, 0.0, 2.0)
    assert np.array_equal(y[0::2], x[:32])
    # alpha = 1/2 => beta = 2: y[m] = x[2m] inside the record, 0 past its end (zeros outside, R12)
    y = O.doppler(x, 8, 1.0, 0.0, 0.5)
    assert np.array_equal(y[:32], x[0::2]) and np.all(y[32:] == 0)


@pytest.mark.parametrize("n", [8, 33, 64])
def test_doppler_full_window_equals_exact(n):
    # With W/2 > max(t) + n the window covers the whole record: windowed Eq. 16 == exact Eq. 16.
    x = synth.complex_gaussian(n, n)
    for alpha in (1.0 + 3e-5, 0.93, 1.21):
        a = O.doppler(x, 3 * n + 2, 1e6, 0.0, alpha)
        b = O.doppler_exact(x, 1e6, 0.0, alpha)
        assert np.max(np.abs(a - b)) < 1e-12


def test_doppler_window_membership_odd_even():
    # odd W: the W samples nearest to t (centre = nearest sample);
    # even W: {k : -W/2 < k - t <= W/2}.
    n = 40
    x = np.zeros(n, complex)
    alpha = 1 / 1.3  # beta = 1.3
    for W in (4, 5):
        for k in range(n):
            x[:] = 0
            x[k] = 1
            y = O.doppler(x, W, 1.0, 0.0, alpha)
            for m in range(n):
                t = m * 1.3
                inside = (-W / 2 < k - t <= W / 2)
                if not inside:
                    assert y[m] == 0
                elif abs(t - round(t)) > 1e-9:
                    assert y[m] != 0


def test_doppler_recovers_dilated_lfm_and_error_falls_with_W():
    # Analytic truth (Table 2 "Analytical Resampling"): the echo S(alpha t) of a Tukey LFM, corrected
    # by resampling onto t/alpha, must approach the undilated chirp; error drops with W (Table 2
    # "O(N_window^-2)").  Resampling the wrong way (alpha -> 1/alpha) must be much worse.
    n, fs = 1 << 14, 2.048e9
    T = 0.8 * n / fs
    alpha = O.alpha_from_velocity(5000.0)
    t = np.arange(n) / fs
    truth = _tukey_at(t - (n // 10) / fs, T)
    echo = _tukey_at(alpha * t - (n // 10) / fs, T)     # S(alpha t)
    nrm = np.linalg.norm(truth)
    errs = [np.linalg.norm(O.doppler(echo, W, fs, 0.0, alpha) - truth) / nrm for W in (8, 16, 32)]
    unc = np.linalg.norm(echo - truth) / nrm
    wrong = np.linalg.norm(O.doppler(echo, 32, fs, 0.0, 1 / alpha) - truth) / nrm
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 0.02 and unc > 10 * errs[2] and wrong > unc


def _tukey_at(tau, T, f0=411e6, B=18e6, frac=0.1):
    inside = (tau >= 0) & (tau < T)
    cyc = f0 * tau + 0.5 * B * tau * tau / T
    x = np.exp(2j * np.pi * (cyc - np.floor(cyc)))
    u = np.clip(tau / T, 0, 1)
    env = np.ones_like(u)
    a = frac / 2
    lo, hi = u < a, u > 1 - a
    env[lo] = 0.5 * (1 - np.cos(np.pi * u[lo] / a))
    env[hi] = 0.5 * (1 - np.cos(np.pi * (1 - u[hi]) / a))
    x = x * env
    x[~inside] = 0
    return x


def test_doppler_carrier_term_baseband():
    # Baseband samples with an LO at fc: the echo of S_RF(alpha t) is s_bb(alpha t) exp(i 2 pi fc (alpha-1) t).
    # Resampling onto t/alpha must be followed by exp(-i 2 pi fc (1 - beta) t) (reading R10); without
    # it (fc passed as 0) the residual carrier costs a large loss.
    n, fs, fc, T = 4096, 51.2e6, 422e6, 40e-6
    alpha = O.alpha_from_velocity(5000.0)
    t = np.arange(n) / fs
    off = 48 / fs
    def sbb(tt):
        tau = tt - off
        inside = (tau >= 0) & (tau < T)
        cyc = (413e6 - fc) * tau + 0.5 * 18e6 * tau * tau / T
        v = np.exp(2j * np.pi * (cyc - np.floor(cyc)))
        v[~inside] = 0
        return v
    truth = sbb(t)
    cyc = fc * (alpha - 1) * t
    echo = sbb(alpha * t) * np.exp(2j * np.pi * (cyc - np.floor(cyc)))
    with_c = L.matched_filter_loss_db(O.doppler(echo, 32, fs, fc, alpha), truth)
    without = L.matched_filter_loss_db(O.doppler(echo, 32, fs, 0.0, alpha), truth)
    assert with_c < 0.01
    assert without > 0.1


def test_batch_entry_matches_single_and_is_thread_independent():
    n, batch, fs = 1024, 5, 2.048e9
    x = synth.complex_gaussian(n, 21, batch=batch).astype(np.complex64)
    tec, alpha = synth.pulse_params(batch)
    y1 = O.run_batch("correct", x, fs, 0.0, 16, tec, alpha, nthreads=1)
    y4 = O.run_batch("correct", x, fs, 0.0, 16, tec, alpha, nthreads=4)
    assert np.array_equal(y1, y4)
    for p in range(batch):
        ref = O.correct(x[p].astype(np.complex128), 16, fs, 0.0, tec[p], alpha[p])
        assert np.array_equal(y1[p], ref)
    yi = O.run_batch("iono", x, fs, 0.0, 16, tec, alpha)
    assert np.array_equal(yi[2], O.iono(x[2].astype(np.complex128), fs, 0.0, tec[2]))


# --------------------------------------------------------------------------- pulse compression (NEXT-2, reading R16)
def test_correlate_autocorrelation_peak_is_energy():
    # matched filter of the reference itself: z_0 = sum |r|^2 (closed form), |z_m| <= z_0 (Cauchy-Schwarz)
    n, Lr = 512, 200
    r = synth.complex_gaussian(Lr, seed=11)
    x = np.zeros(n, complex)
    x[:Lr] = r
    z = O.correlate(x, r)
    e = np.sum(np.abs(r) ** 2)
    assert abs(z[0] - e) < 1e-12 * e
    assert np.all(np.abs(z) <= e * (1 + 1e-12))
    assert np.argmax(np.abs(z)) == 0


@pytest.mark.parametrize("d", [0, 1, 37, 511])
def test_correlate_delayed_copy_peaks_at_delay(d):
    # x = r delayed circularly by d samples -> z_d = energy, argmax = d (sign of the lag fixed)
    n, Lr = 512, 64
    r = synth.complex_gaussian(Lr, seed=12)
    x = np.zeros(n, complex)
    x[(np.arange(Lr) + d) % n] = r
    z = O.correlate(x, r)
    assert np.argmax(np.abs(z)) == d
    assert abs(z[d] - np.sum(np.abs(r) ** 2)) < 1e-12 * np.sum(np.abs(r) ** 2)


def test_correlate_matches_numpy_fft_correlation():
    # independent library: IDFT(DFT(y) conj(DFT(r_padded))) with numpy.fft; also sampled outputs
    n, Lr = 256, 100
    y = synth.complex_gaussian(n, seed=13)
    r = synth.complex_gaussian(Lr, seed=14)
    rp = np.zeros(n, complex)
    rp[:Lr] = r
    ref = np.fft.ifft(np.fft.fft(y) * np.conj(np.fft.fft(rp)))
    z = O.correlate(y, r)
    assert np.max(np.abs(z - ref)) < 1e-12 * np.max(np.abs(ref))
    idx = np.array([0, 5, 255, 128])
    assert np.array_equal(O.correlate(y, r, idx), z[idx])


def test_compress_is_correlation_of_corrected_pulse():
    # compress(distort(x)) = correlate(x, r): the Eq. 15 correction undoes Eq. 14 before matching
    n = 1024
    x = synth.complex_gaussian(n, seed=15)
    r = synth.complex_gaussian(300, seed=16)
    fs, fc, tec = 51.2e6, 422e6, 1e18
    xd = O.iono(x, fs, fc, tec, distort=True)
    z = O.compress(xd, fs, fc, tec, r)
    ref = O.correlate(x, r)
    assert np.max(np.abs(z - ref)) < 1e-10 * np.max(np.abs(ref))
    # tec = 0: compress is the plain matched filter
    assert np.max(np.abs(O.compress(x, fs, fc, 0.0, r) - ref)) < 1e-12 * np.max(np.abs(ref))


def test_compress_lfm_peak_sidelobe_textbook():
    # large time-bandwidth LFM (TB = 18 MHz x 100 us = 1800): compressed peak = energy at lag 0 and
    # the first sidelobe sits near the sinc value -13.26 dB (textbook pulse-compression result);
    # a missing conj gives no compression at all
    fs, n = 204.8e6, 1 << 15
    T, B = 100e-6, 18e6
    ns = int(round(T * fs))
    t = np.arange(ns) / fs
    r = np.exp(1j * np.pi * (B / T) * (t - T / 2) ** 2)
    x = np.zeros(n, complex)
    x[:ns] = r
    z = np.abs(O.compress(x, fs, 0.0, 0.0, r))
    assert np.argmax(z) == 0 and abs(z[0] - ns) < 1e-9 * ns
    zz = np.concatenate([z[n // 2:], z[:n // 2]])
    c = n // 2
    # walk out of the main lobe to the first null, then take the highest sidelobe near it
    k = c + 1
    while zz[k + 1] < zz[k]:
        k += 1
    side = np.max(zz[k:k + int(3 * fs / B)])
    sll = 20 * np.log10(side / zz[c])
    assert -13.8 < sll < -12.8
    wrong = np.abs(np.fft.ifft(np.fft.fft(x) * np.fft.fft(np.pad(r, (0, n - ns)))))
    assert np.max(wrong) < 0.2 * ns


# ----------------------------------------------------------------------------- Kaiser taper (R17, NEXT-3)
def test_bessel_i0_matches_library():
    # the taper's I0 (power series) against an independent library implementation
    import scipy.special as sp
    for z in (0.0, 1e-3, 0.3, 1.0, 3.75, 8.0, 12.5, 20.0):
        assert abs(O.bessel_i0(z) / sp.i0(z) - 1) < 1e-14, z


def test_kaiser_taper_shape():
    L, kb = 16.0, 8.0
    assert O.kaiser(0.0, L, kb) == 1.0                                  # centre tap untouched: alpha = 1 stays exact
    assert O.kaiser(0.0, L, 0.0) == 1.0 and O.kaiser(15.5, L, 0.0) == 1.0   # kb = 0: rectangular (R11)
    for d in (0.3, 2.5, 7.0, 15.9):
        assert O.kaiser(d, L, kb) == O.kaiser(-d, L, kb)                 # symmetric
    assert abs(O.kaiser(L, L, kb) - 1 / 427.56411572180474) < 1e-15     # edge value 1/I0(kb)
    x = 0.5                                                              # closed form at d = L/2
    import scipy.special as sp
    assert abs(O.kaiser(x * L, L, kb) - sp.i0(kb * np.sqrt(1 - x * x)) / sp.i0(kb)) < 1e-14


def test_kaiser_alpha_one_identity_and_rect_reduction():
    x = synth.complex_gaussian(512, seed=3)
    assert np.array_equal(O.doppler(x, 32, 1e6, 0.0, 1.0, kaiser=8.0), x)         # exact at integer positions
    a = O.doppler(x, 16, 1e6, 0.0, 1 + 3e-5, kaiser=0.0)
    b = O.doppler(x, 16, 1e6, 0.0, 1 + 3e-5)
    assert np.array_equal(a, b)


def test_kaiser_taper_accuracy_vs_analytic_truth():
    # SURVEY 8(c) (independent FP64 scratch code): dilated Tukey LFM at 5 km/s, n = 2^14 (its table used
    # 2^16), rel-L2 vs the exact undilated chirp.  Rectangular W = 32: 7.3e-3; Kaiser kb = 8:
    # W = 16: 6.1e-5, W = 32: 3.2e-5.  The taper must reproduce those magnitudes.
    n, fs = 1 << 14, 2.048e9
    T = 0.8 * n / fs
    alpha = O.alpha_from_velocity(5000.0)
    t = np.arange(n) / fs
    truth = _tukey_at(t - (n // 10) / fs, T)
    echo = _tukey_at(alpha * t - (n // 10) / fs, T)
    nrm = np.linalg.norm(truth)
    err = lambda W, kb: np.linalg.norm(O.doppler(echo, W, fs, 0.0, alpha, kaiser=kb) - truth) / nrm
    rect32, k16, k32 = err(32, 0.0), err(16, 8.0), err(32, 8.0)
    assert 5e-3 < rect32 < 1e-2
    assert 4e-5 < k16 < 9e-5
    assert 2e-5 < k32 < 5e-5
    assert rect32 > 100 * k32


# ----------------------------------------------------------------------------- FFT P/Q resampling (R18, NEXT-4)
@pytest.mark.parametrize("n,M", [(64, 70), (64, 58), (63, 71), (65, 60), (100, 102), (101, 99), (256, 250)])
def test_pq_resample_matches_library(n, M):
    # independent library implementation of the same definition (FFT, box filter, IFFT, Nyquist split/fold)
    import scipy.signal as ss
    rng = np.random.default_rng(n * 1000 + M)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y = O.pq_resample(x, M)
    k = min(n, M)
    ref = ss.resample(x, M)[:k]
    assert np.abs(y[:k] - ref).max() < 1e-12 * np.abs(ref).max()
    assert not np.any(y[k:])                                  # outputs past M are zero (R12)


def test_pq_resample_identity_and_length_rule():
    x = synth.complex_gaussian(128, seed=11)
    assert np.allclose(O.pq_resample(x, 128), x, rtol=0, atol=1e-13)
    assert O.pq_length(1 << 19, 1.0) == 1 << 19
    a5 = O.alpha_from_velocity(5000.0)                      # n (alpha - 1) = 17.49 samples at 2^19
    assert O.pq_length(1 << 19, a5) == (1 << 19) + 18         # nearest even number of added samples
    assert O.pq_length(1 << 19, 1 / a5) == (1 << 19) - 18


@pytest.mark.parametrize("n,M", [(96, 100), (96, 90), (127, 131)])
def test_doppler_pq_exact_for_even_index_dilation(n, M):
    # Closed form ("exact when N - N/alpha is an even integer"): S(t) = sum_j a_j e^{i 2 pi f_j t / M}
    # (band-limited, period M) received as x_t = S(alpha t) with alpha = M / n; the correction must
    # return S(m) exactly.  The windowed sinc of Eq. 16 is not exact for the same input.
    rng = np.random.default_rng(n + M)
    f = np.array([0, 3, -5, 11, -17, 23])
    a = rng.standard_normal(f.size) + 1j * rng.standard_normal(f.size)
    t = np.arange(n)
    x = (a[None, :] * np.exp(2j * np.pi * np.outer(t, f) / n)).sum(1)        # S(alpha t), alpha = M / n
    m = np.arange(min(n, M))
    truth = (a[None, :] * np.exp(2j * np.pi * np.outer(m, f) / M)).sum(1)    # S(m)
    y = O.doppler_pq(x, 1e6, 0.0, M / n)
    assert O.pq_length(n, M / n) == M
    assert np.abs(y[:m.size] - truth).max() < 1e-11 * np.abs(truth).max()
    ws = O.doppler(x, 32, 1e6, 0.0, M / n)[:m.size]
    assert np.abs(ws - truth).max() > 1e-6 * np.abs(truth).max()


# ----------------------------------------------------------------------------- carrier term at fc != 0 (R10, R18)
def _baseband_echo_of_dilated_rf(g_hz, amp, fs, fc, alpha, n):
    """Received baseband samples r_k = S_bb(alpha t) e^{i 2 pi fc (alpha - 1) t}, t = k / fs: the echo
    S_RF(alpha t) (Eq. 13) of S_RF(t) = S_bb(t) e^{i 2 pi fc t}, mixed down by an LO at fc."""
    t = np.arange(n) / fs
    ph = np.outer(alpha * t, g_hz) + (fc * (alpha - 1.0) * t)[:, None]
    return (amp[None, :] * np.exp(2j * np.pi * (ph - np.floor(ph)))).sum(1)


@pytest.mark.parametrize("n,M", [(96, 100), (128, 122)])
def test_doppler_pq_carrier_recovers_transmitted_baseband(n, M):
    # Physical truth at fc != 0 (P:L294 exact case; reading R18 + R10): choose baseband tones g_j so the
    # received echo of S_RF(alpha_eff t), alpha_eff = M / n, is periodic in n and band-limited (every
    # component on an n-point bin).  P/Q resampling to M then samples the echo exactly at t = m n / M and
    # the carrier term (beta_eff = n / M, the grid actually resampled) must leave S_bb(m / fs) -- the
    # transmitted baseband -- for every m < min(n, M).  alpha passed to the method is NOT M / n exactly
    # (it only selects M), so a carrier computed from 1 / alpha, or with the wrong sign, fails.
    fs, fc = 51.2e6, 422e6
    a_eff = M / n
    f_bins = np.array([0, 2, -3, 7, -9, 13])
    rng = np.random.default_rng(7 * n + M)
    amp = rng.standard_normal(f_bins.size) + 1j * rng.standard_normal(f_bins.size)
    g = (f_bins * fs / n - fc * (a_eff - 1.0)) / a_eff          # a_eff g_j + fc (a_eff - 1) = f_j fs / n
    x = _baseband_echo_of_dilated_rf(g, amp, fs, fc, a_eff, n)
    alpha = a_eff * (1.0 + 0.6 / n)                              # rounds to the same M (pq_length)
    assert O.pq_length(n, alpha) == M
    m = np.arange(min(n, M))
    ph = np.outer(m / fs, g)
    truth = (amp[None, :] * np.exp(2j * np.pi * (ph - np.floor(ph)))).sum(1)   # S_bb(m / fs)
    y = O.doppler_pq(x, fs, fc, alpha)
    assert np.abs(y[:m.size] - truth).max() < 1e-9 * np.abs(truth).max()
    # the same input without the carrier term (fc passed as 0 shifts the bin grid, so compare the pure
    # resampling instead): the residual carrier exp(i 2 pi fc (1 - n/M) m / fs) is large
    y0 = O.pq_resample(x, M)[:m.size]
    assert np.abs(y0 - truth).max() > 0.1 * np.abs(truth).max()


def test_doppler_exact_carrier_term_baseband():
    # Eq. 16 over the whole record (orc_doppler_exact) with the R10 carrier at fc = 422 MHz: the
    # corrected echo of a dilated baseband LFM (the same physics as test_doppler_carrier_term_baseband)
    # matches the transmitted pulse; dropping the carrier (or flipping it: twice the residual) costs > 0.1 dB.
    n, fs, fc, T = 4096, 51.2e6, 422e6, 40e-6
    alpha = O.alpha_from_velocity(5000.0)
    t = np.arange(n) / fs
    off = 48 / fs

    def sbb(tt):
        tau = tt - off
        inside = (tau >= 0) & (tau < T)
        cyc = (413e6 - fc) * tau + 0.5 * 18e6 * tau * tau / T
        v = np.exp(2j * np.pi * (cyc - np.floor(cyc)))
        v[~inside] = 0
        return v

    truth = sbb(t)
    cyc = fc * (alpha - 1) * t
    echo = sbb(alpha * t) * np.exp(2j * np.pi * (cyc - np.floor(cyc)))
    with_c = L.matched_filter_loss_db(O.doppler_exact(echo, fs, fc, alpha), truth)
    without = L.matched_filter_loss_db(O.doppler_exact(echo, fs, 0.0, alpha), truth)
    assert with_c < 0.01
    assert without > 0.1


def test_doppler_at_equals_whole_pulse_outputs():
    # the sampled entry point (parity at 2^22..2^24) evaluates exactly the outputs of orc_doppler_win
    x = synth.complex_gaussian(2048, seed=19)
    idx = np.array([0, 1, 777, 1024, 2047])
    for a, kb in ((1 + 3.3e-5, 0.0), (0.93, 0.0), (1.0 - 2e-5, 8.0)):
        y = O.doppler(x, 32, 51.2e6, 422e6, a, kaiser=kb)
        assert np.array_equal(O.doppler_at(x, 32, 51.2e6, 422e6, a, idx, kaiser=kb), y[idx])
    with pytest.raises(RuntimeError):
        O.doppler_at(x, 32, 51.2e6, 0.0, 1.0, [2048])


# ----------------------------------------------------------------------------- P/Q at sampled outputs (R18)
@pytest.mark.parametrize("n,M", [(64, 70), (64, 58), (256, 250), (256, 264), (1024, 1024), (512, 2)])
def test_pq_resample_at_matches_full(n, M):
    # the sampled-output form (radix-2 forward FFT + the length-M inverse DFT sum per output) equals the
    # full O(n^2) definition, which is pinned to scipy.signal.resample above
    rng = np.random.default_rng(n + 3 * M)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    idx = np.arange(n)
    full = O.pq_resample(x, M)
    at = O.pq_resample_at(x, M, idx)
    assert np.abs(at - full).max() < 1e-12 * np.abs(full).max()


@pytest.mark.parametrize("n,M", [(128, 122), (128, 134)])
def test_doppler_pq_at_matches_full_with_carrier(n, M):
    fs, fc = 51.2e6, 422e6
    rng = np.random.default_rng(M)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    alpha = M / n * (1.0 + 0.3 / n)
    assert O.pq_length(n, alpha) == M
    idx = np.array([0, 1, 5, 63, 64, 100, n - 1])
    full = O.doppler_pq(x, fs, fc, alpha)[idx]
    at = O.doppler_pq_at(x, fs, fc, alpha, idx)
    assert np.abs(at - full).max() < 1e-12 * np.abs(full).max()


# ----------------------------------------------------------------------------- Hann taper (R17, NEXT-3)
def test_hann_taper_shape():
    L = 16.0
    assert O.hann(0.0, L) == 1.0                              # centre tap untouched: alpha = 1 stays exact
    assert abs(O.hann(L, L)) < 1e-16 and abs(O.hann(-L, L)) < 1e-16   # zero at the window edges
    assert abs(O.hann(L / 2, L) - 0.5) < 1e-15               # cos^2(pi/4)
    for d in (0.3, 2.5, 7.0, 15.9):
        assert O.hann(d, L) == O.hann(-d, L)
        assert abs(O.hann(d, L) - np.cos(np.pi * d / (2 * L)) ** 2) < 1e-15   # cos^2(pi d / 2L) identity


def test_hann_alpha_one_identity_and_accuracy():
    x = synth.complex_gaussian(512, seed=3)
    assert np.array_equal(O.doppler(x, 32, 1e6, 0.0, 1.0, kaiser=O.HANN), x)
    # dilated Tukey LFM (as the Kaiser pin): the Hann taper beats the rectangular window at W = 32
    n, fs = 1 << 14, 2.048e9
    T = 0.8 * n / fs
    alpha = O.alpha_from_velocity(5000.0)
    t = np.arange(n) / fs
    truth = _tukey_at(t - (n // 10) / fs, T)
    echo = _tukey_at(alpha * t - (n // 10) / fs, T)
    nrm = np.linalg.norm(truth)
    err = lambda W, kb: np.linalg.norm(O.doppler(echo, W, fs, 0.0, alpha, kaiser=kb) - truth) / nrm
    rect32, h32 = err(32, 0.0), err(32, O.HANN)
    assert h32 < rect32 / 5
