"""GPU parity: the CUDA path through the C ABI vs the FP64 oracle on identical complex64 inputs.

Bar (north_star): per-pulse relative L2 error <= 1e-5; alpha = 1 bit-exact;
TEC = 0 within the FP32 FFT round trip.  Sizes span several tiles and ragged tails; the
full-size configurations are checked on sampled pulses the oracle computes one by one.
"""
import numpy as np
import pytest

import synth
from oracle import lfm as L
from oracle import oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(scope="module")
def dc():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2508_04951_b200 as dcmod
    from paper_2508_04951_b200 import build
    build.build()
    dcmod.load()
    return dcmod


def to_dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex64)).cuda()


def from_dev(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


def rel_l2(a, b):
    a = np.atleast_2d(a)
    b = np.atleast_2d(b)
    num = np.linalg.norm(a - b, axis=1)
    den = np.maximum(np.linalg.norm(b, axis=1), 1e-300)
    return num / den


def gpu_iono(dc, x, fs, fc, tec, distort=False):
    p = dc.Plan(x.shape[-1], fs, fc, taps=min(8, x.shape[-1]))
    t = to_dev(x)
    (p.iono_distort if distort else p.iono)(t, tec)
    return from_dev(t)


# ----------------------------------------------------------------------------- iono (Eq. 15)
@pytest.mark.parametrize("log2n", list(range(1, 14)))
def test_iono_small_regime_vs_oracle(dc, log2n):
    n = 1 << log2n
    batch = 3 if n >= 1024 else 37   # ragged: fewer pulses than a CTA tile holds, or not a multiple
    x = synth.complex_gaussian(n, seed=log2n, batch=batch).astype(np.complex64)
    tec = np.linspace(0, 2e18, batch)
    for fs, fc in ((2.048e9, 0.0), (51.2e6, 422e6)):
        y = gpu_iono(dc, x, fs, fc, tec)
        ref = O.run_batch("iono", x, fs, fc, 8, tec)
        err = rel_l2(y, ref)
        assert err.max() < TOL, (n, fs, fc, err.max())


@pytest.mark.parametrize("log2n", [14, 15, 16, 17, 18, 19, 20])
def test_iono_fourstep_regime_vs_oracle(dc, log2n):
    n = 1 << log2n
    batch = 2
    x = synth.complex_gaussian(n, seed=100 + log2n, batch=batch).astype(np.complex64)
    tec = np.array([1e18, 3.7e17])
    for fs, fc in ((2.048e9, 0.0), (204.8e6, 422e6)):
        y = gpu_iono(dc, x, fs, fc, tec)
        ref = O.run_batch("iono", x, fs, fc, 8, tec)
        err = rel_l2(y, ref)
        assert err.max() < TOL, (n, fs, fc, err.max())


@pytest.mark.slow
@pytest.mark.parametrize("log2n", [21, 22, 23, 24])
def test_iono_largest_pulses_vs_oracle(dc, log2n):
    n = 1 << log2n
    x = synth.complex_gaussian(n, seed=log2n, batch=1).astype(np.complex64)
    y = gpu_iono(dc, x, 2.048e9, 0.0, [1e18])
    ref = O.run_batch("iono", x, 2.048e9, 0.0, 8, [1e18])
    assert rel_l2(y, ref).max() < TOL


@pytest.mark.parametrize("log2n", [10, 13, 16, 20])
def test_iono_tec_zero_and_roundtrip(dc, log2n):
    n = 1 << log2n
    x = synth.complex_gaussian(n, seed=7, batch=2).astype(np.complex64)
    y0 = gpu_iono(dc, x, 2.048e9, 0.0, [0.0, 0.0])
    assert rel_l2(y0, x).max() < 2e-6                       # FFT round trip only
    d = gpu_iono(dc, x, 2.048e9, 0.0, [1e18, 5e17], distort=True)
    refd = np.stack([O.iono(x[i].astype(np.complex128), 2.048e9, 0.0, t, distort=True) for i, t in enumerate([1e18, 5e17])])
    assert rel_l2(d, refd).max() < TOL                      # Eq. 14 path
    back = gpu_iono(dc, d.astype(np.complex64), 2.048e9, 0.0, [1e18, 5e17])
    assert rel_l2(back, x).max() < 5e-6                     # Eq. 15 inverts Eq. 14


def test_iono_c2_tec_sweep_sampled(dc):
    # C2: 256 x 2^16 phase-coded pulses, TEC_p = p TECU; parity on sampled pulses, identity at p = 0
    cfg = synth.c2_batch()
    x, tec = cfg["x"], cfg["tec"]
    y = gpu_iono(dc, x, cfg["fs"], 0.0, tec)
    idx = [0, 1, 17, 128, 255]
    ref = O.run_batch("iono", x[idx], cfg["fs"], 0.0, 8, tec[idx])
    assert rel_l2(y[idx], ref).max() < TOL
    assert rel_l2(y[0], x[0]).max() < 2e-6


def test_iono_fig2_cubic_pin_on_gpu(dc):
    # PAPER Fig. 2: FFT correction vs CUBIC truth loses < 0.01 dB at 2^19 samples
    n, fs, tec = 1 << 19, 2.048e9, 1e18
    x = synth.lfm(n, fs, 413e6, 18e6, 100e-6, offset=1 << 17).astype(np.complex64)
    y = gpu_iono(dc, x[None], fs, 0.0, [tec])[0]
    cub = L.cubic_waveform(413e6, 18e6, 100e-6, O.k2_per_tec() * tec, fs)
    assert L.matched_filter_loss_db(y, cub) < 0.01


def test_iono_sign_gaussian_packet_on_gpu(dc):
    n, fs, tec = 1 << 15, 2.048e9, 1e18
    x = synth.gaussian_packet(n, fs, 400e6, 2000.0, n / 2).astype(np.complex64)
    y = gpu_iono(dc, x[None], fs, 0.0, [tec])[0]
    shift = L.envelope_peak(y) - L.envelope_peak(x)
    assert shift == pytest.approx(-2 * O.group_delay(400e6, tec) * fs, abs=2.0)


# ----------------------------------------------------------------------------- doppler (Eq. 16 windowed)
def gpu_doppler(dc, x, W, fs, fc, alpha):
    import torch
    p = dc.Plan(x.shape[-1], fs, fc, taps=W)
    t = to_dev(x)
    y = torch.empty_like(t)
    p.doppler(t, y, alpha)
    return from_dev(y)


ALPHA_CASES = {
    "fast1": [1 + 3.3e-5, 1 - 3.3e-5, 1 + 1e-5],      # |v| <= 5 km/s: first-order path
    "fast2": [1 + 4e-4, 1 - 4.5e-4, 1 + 1e-4],        # second-order path
    "exact": [1.05, 0.93, 1.0 + 2e-3],                # exact-tap path
}


@pytest.mark.parametrize("case", list(ALPHA_CASES))
@pytest.mark.parametrize("W", [2, 3, 8, 16, 25, 32, 64, 128])
def test_doppler_vs_oracle(dc, case, W):
    n = 4096
    alphas = np.array(ALPHA_CASES[case])
    x = synth.complex_gaussian(n, seed=W, batch=len(alphas)).astype(np.complex64)
    for fs, fc in ((2.048e9, 0.0), (51.2e6, 422e6)):
        y = gpu_doppler(dc, x, W, fs, fc, alphas)
        ref = O.run_batch("doppler", x, fs, fc, W, None, alphas)
        err = rel_l2(y, ref)
        assert err.max() < TOL, (case, W, fs, fc, err.max())


@pytest.mark.parametrize("log2n", [4, 11, 16, 20])
def test_doppler_sizes_vs_oracle(dc, log2n):
    n = 1 << log2n
    alphas = np.array([1 + 3.3e-5, 1 - 2e-5])
    x = synth.complex_gaussian(n, seed=log2n, batch=2).astype(np.complex64)
    y = gpu_doppler(dc, x, 32 if n >= 32 else n, 2.048e9, 0.0, alphas)
    ref = O.run_batch("doppler", x, 2.048e9, 0.0, 32 if n >= 32 else n, None, alphas)
    assert rel_l2(y, ref).max() < TOL


@pytest.mark.parametrize("W", [8, 32, 128])
def test_doppler_alpha_one_bit_exact(dc, W):
    x = synth.complex_gaussian(8192, seed=3, batch=3).astype(np.complex64)
    y = gpu_doppler(dc, x, W, 51.2e6, 422e6, [1.0, 1.0, 1.0])
    assert np.array_equal(y, x)


def test_doppler_full_window_equals_exact_eq16(dc):
    # W = n = 128 and a signal supported on [56, 72): every output whose window (t - 64, t + 64]
    # covers the support equals the exact (unwindowed) Eq. 16 sum.
    n, W = 128, 128
    x = np.zeros((2, n), np.complex64)
    x[:, 56:72] = synth.complex_gaussian(16, seed=5, batch=2)
    alphas = [1 + 3e-5, 1.0 + 1e-3]
    y = gpu_doppler(dc, x, W, 1e6, 0.0, alphas)
    for i, a in enumerate(alphas):
        ref = O.doppler_exact(x[i].astype(np.complex128), 1e6, 0.0, a)
        t = np.arange(n) / a
        sel = (t - 64 < 56) & (t + 64 >= 71)
        assert sel.sum() > 100
        assert rel_l2(y[i][sel], ref[sel]).max() < TOL


# ----------------------------------------------------------------------------- correct (both stages)
def gpu_correct(dc, x, W, fs, fc, tec, alpha):
    import torch
    p = dc.Plan(x.shape[-1], fs, fc, taps=W)
    t = to_dev(x)
    y = torch.empty_like(t)
    p.correct(t, y, tec, alpha)
    xt = from_dev(t)
    assert np.array_equal(xt, x)                  # x untouched
    return from_dev(y)


@pytest.mark.parametrize("variant", ["a", "b"])
def test_correct_c1(dc, variant):
    c = synth.c1_pulse(variant)
    y = gpu_correct(dc, c["x"][None], c["W"], c["fs"], c["fc"], [c["tec"]], [c["alpha"]])
    ref = O.run_batch("correct", c["x"][None], c["fs"], c["fc"], c["W"], [c["tec"]], [c["alpha"]])
    assert rel_l2(y, ref).max() < TOL


@pytest.mark.parametrize("log2n", [12, 16, 20])
def test_correct_pulse_train_sampled(dc, log2n):
    n = 1 << log2n
    batch = 24 if log2n == 20 else 64
    bank = synth.waveform_bank(n, count=8, T=min(100e-6, 0.4 * n / 2.048e9))
    tec, alpha = synth.pulse_params(batch)
    x = bank[np.arange(batch) % 8]
    y = gpu_correct(dc, x, 32, 2.048e9, 0.0, tec, alpha)
    idx = [0, 1, batch // 2, batch - 1]
    ref = O.run_batch("correct", x[idx], 2.048e9, 0.0, 32, tec[idx], alpha[idx])
    assert rel_l2(y[idx], ref).max() < TOL


def test_correct_host_matches_device(dc):
    import torch
    n, batch = 1 << 14, 40
    x = synth.complex_gaussian(n, seed=11, batch=batch).astype(np.complex64)
    tec, alpha = synth.pulse_params(batch)
    p = dc.Plan(n, 2.048e9, 0.0, taps=32)
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    p.correct_host(xh, yh, tec, alpha)
    yd = gpu_correct(dc, x, 32, 2.048e9, 0.0, tec, alpha)
    assert np.array_equal(yh.numpy(), yd)
    y_np = np.empty_like(x)
    p.correct_host(x, y_np, tec, alpha)            # pageable numpy buffers too
    assert np.array_equal(y_np, yd)


# ----------------------------------------------------------------------------- errors through the ABI
def test_abi_errors_on_gpu(dc):
    import torch
    p = dc.Plan(1024, 1e6, 0.0, taps=8)
    x = torch.zeros(4, 1024, dtype=torch.complex64, device="cuda")
    y = torch.zeros(4, 1024, dtype=torch.complex64, device="cuda")
    with pytest.raises(dc.DispCorrError) as e:
        p.iono(x, [1.0, -1.0, 0, 0])
    assert e.value.name == "DC_ERR_INVALID_VALUE"
    with pytest.raises(dc.DispCorrError) as e:
        p.doppler(x, y, [1.0, 0.0, 1, 1])
    assert e.value.name == "DC_ERR_INVALID_VALUE"
    with pytest.raises(dc.DispCorrError) as e:
        p.doppler(x, x, [1.0] * 4)
    assert e.value.name == "DC_ERR_ALIASING"
    flat = torch.zeros(4 * 1024 + 1, dtype=torch.complex64, device="cuda")
    with pytest.raises(dc.DispCorrError) as e:
        lib = dc.load()
        import ctypes
        arr = (ctypes.c_double * 1)(0.0)
        st = lib.dc_iono(p._h, ctypes.c_void_p(flat.data_ptr() + 8), 1, arr)
        dc._check(st)
    assert e.value.name == "DC_ERR_MISALIGNED"
    host = torch.zeros(1024, dtype=torch.complex64)
    with pytest.raises(dc.DispCorrError) as e:
        lib = dc.load()
        import ctypes
        arr = (ctypes.c_double * 1)(0.0)
        dc._check(lib.dc_iono(p._h, ctypes.c_void_p(host.data_ptr()), 1, arr))
    assert e.value.name == "DC_ERR_NOT_DEVICE_MEMORY"
    p.sync()
    info = p.info()
    assert info["regime"] == 0 and info["n"] == 1024


# ----------------------------------------------------------------------------- pulse compression (NEXT-2)
def gpu_compress(dc, x, r, fs, fc, tec, inplace=False):
    p = dc.Plan(x.shape[-1], fs, fc, taps=min(8, x.shape[-1]))
    p.set_reference(to_dev(r))
    t = to_dev(x)
    z = t if inplace else to_dev(np.zeros_like(x))
    p.compress(t, z, tec)
    return from_dev(z)


@pytest.mark.parametrize("log2n,L", [(1, 1), (5, 7), (8, 256), (10, 300), (10, 1024), (11, 2048), (12, 1000),
                                     (13, 5000), (14, 500), (16, 2000), (17, 8192), (18, 1000), (21, 4096),
                                     (22, 3000), (23, 100000), (24, 4096)])
def test_compress_vs_oracle(dc, log2n, L):
    # z = circular matched filter of iono(x) against r (oracle: the direct-sum definition)
    n = 1 << log2n
    rng = np.random.default_rng(log2n + L)
    r = (rng.standard_normal(L) + 1j * rng.standard_normal(L)).astype(np.complex64)
    x = synth.complex_gaussian(n, seed=200 + log2n, batch=2).astype(np.complex64)
    tec = np.array([1e18, 0.0])
    fs, fc = (2.048e9, 0.0) if log2n not in (12, 18, 22) else (204.8e6, 422e6)
    z = gpu_compress(dc, x, r, fs, fc, tec)
    if n <= (1 << 17):
        ref = np.stack([O.compress(x[i], fs, fc, tec[i], r) for i in range(2)])
        assert rel_l2(z, ref).max() < TOL
    else:  # sampled outputs, computed one by one by the oracle
        idx = np.sort(np.random.default_rng(5).choice(n, 300, replace=False))
        ref = np.stack([O.compress(x[i], fs, fc, tec[i], r, idx=idx) for i in range(2)])
        assert rel_l2(z[:, idx], ref).max() < TOL


def test_compress_lfm_echo_c3_sampled(dc):
    # C3 geometry: a dispersed (Eq. 14), delayed LFM echo compressed against the transmitted LFM;
    # the compressed peak sits at the echo delay, and sampled outputs around it match the oracle
    n, fs, T, delay = 1 << 20, 2.048e9, 100e-6, 123457
    L = int(T * fs)
    r = synth.lfm(L, fs, 413e6, 18e6, T).astype(np.complex64)
    echo = np.roll(np.concatenate([r, np.zeros(n - L, np.complex64)]), delay)
    x = O.iono(echo.astype(np.complex128), fs, 0.0, 1e18, distort=True).astype(np.complex64)[None]
    z = gpu_compress(dc, x, r, fs, 0.0, [1e18], inplace=True)[0]
    assert int(np.argmax(np.abs(z))) == delay
    idx = np.unique(np.concatenate([np.arange(delay - 64, delay + 64), np.random.default_rng(9).choice(n, 200)]))
    ref = O.compress(x[0], fs, 0.0, 1e18, r, idx=idx)
    assert rel_l2(z[idx], ref).max() < TOL
    # matched-filter gain: the peak equals the reference energy (Cauchy-Schwarz bound attained)
    assert abs(abs(z[delay]) / np.sum(np.abs(r.astype(np.complex128)) ** 2) - 1) < 1e-4


def test_compress_errors(dc):
    import torch
    p = dc.Plan(1 << 17, 2.048e9, 0.0, taps=8)
    x = torch.zeros(1, 1 << 17, dtype=torch.complex64, device="cuda")
    with pytest.raises(dc.DispCorrError) as e:
        p.compress(x, x, [1e18])          # no reference yet
    assert e.value.name == "DC_ERR_INVALID_VALUE"
    with pytest.raises(dc.DispCorrError) as e:
        p.set_reference(torch.zeros((1 << 17) + 1, dtype=torch.complex64, device="cuda"))   # L > n
    assert e.value.name == "DC_ERR_INVALID_VALUE"
    p.set_reference(torch.ones(16, dtype=torch.complex64, device="cuda"))
    buf = torch.zeros(2 << 17, dtype=torch.complex64, device="cuda")
    import ctypes
    arr = (ctypes.c_double * 1)(0.0)
    st = dc.load().dc_compress(p._h, ctypes.c_void_p(buf.data_ptr()), ctypes.c_void_p(buf.data_ptr() + 4096), 1, arr)
    assert dc.STATUS[st] == "DC_ERR_ALIASING"      # partial overlap of x and z
    p.compress(x, x, [1e18])                       # in place is allowed
    p.sync()


# ----------------------------------------------------------------------------- Kaiser taper (R17, NEXT-3)
def gpu_doppler_taper(dc, x, W, fs, fc, alpha, kaiser):
    import torch
    p = dc.Plan(x.shape[-1], fs, fc, taps=W)
    p.set_taper(kaiser)
    t = to_dev(x)
    y = torch.empty_like(t)
    p.doppler(t, y, alpha)
    return from_dev(y)


@pytest.mark.parametrize("case", ["fast1", "exact"])
@pytest.mark.parametrize("W,kb", [(8, 4.0), (16, 8.0), (25, 6.0), (32, 8.0), (64, 10.0), (128, 12.0)])
def test_doppler_kaiser_vs_oracle(dc, case, W, kb):
    n = 4096
    alphas = np.array(ALPHA_CASES[case])
    x = synth.complex_gaussian(n, seed=W + 7, batch=len(alphas)).astype(np.complex64)
    for fs, fc in ((2.048e9, 0.0), (51.2e6, 422e6)):
        y = gpu_doppler_taper(dc, x, W, fs, fc, alphas, kb)
        ref = O.run_batch("doppler", x, fs, fc, W, None, alphas, kaiser=kb)
        err = rel_l2(y, ref)
        assert err.max() < TOL, (case, W, kb, fs, fc, err.max())


def gpu_doppler_window(dc, x, W, fs, fc, alpha, kind, param=0.0):
    import torch
    p = dc.Plan(x.shape[-1], fs, fc, taps=W)
    p.set_window(kind, param)
    t = to_dev(x)
    y = torch.empty_like(t)
    p.doppler(t, y, alpha)
    return from_dev(y)


@pytest.mark.parametrize("case", ["fast1", "fast2", "exact"])
@pytest.mark.parametrize("W", [8, 16, 25, 32, 64, 128, 7])
def test_doppler_hann_vs_oracle(dc, case, W):
    # Hann taper (R17): first-order fast path, the second-order drift range (tapered: exact path) and the
    # exact-tap kernel; compile-time and runtime W
    n = 4096
    alphas = np.array(ALPHA_CASES[case])
    x = synth.complex_gaussian(n, seed=W + 17, batch=len(alphas)).astype(np.complex64)
    for fs, fc in ((2.048e9, 0.0), (51.2e6, 422e6)):
        y = gpu_doppler_window(dc, x, W, fs, fc, alphas, "hann")
        ref = O.run_batch("doppler", x, fs, fc, W, None, alphas, kaiser=O.HANN)
        assert rel_l2(y, ref).max() < TOL, (case, W, fs, fc)


def test_doppler_hann_alpha_one_bit_exact_and_window_switch(dc):
    import torch
    x = synth.complex_gaussian(8192, seed=5, batch=2).astype(np.complex64)
    assert np.array_equal(gpu_doppler_window(dc, x, 32, 51.2e6, 422e6, [1.0, 1.0], "hann"), x)
    # switching windows on one plan: hann -> rect -> kaiser reproduce the oracle of each
    p = dc.Plan(8192, 2.048e9, 0.0, taps=16)
    xd = to_dev(x)
    a = [1 + 2e-5, 1 - 3e-5]
    for kind, param, kb in (("hann", 0.0, O.HANN), ("rect", 0.0, 0.0), ("kaiser", 6.0, 6.0)):
        p.set_window(kind, param)
        yd = torch.empty_like(xd)
        p.doppler(xd, yd, a)
        ref = O.run_batch("doppler", x, 2.048e9, 0.0, 16, None, a, kaiser=kb)
        assert rel_l2(from_dev(yd), ref).max() < TOL, kind
    with pytest.raises(dc.DispCorrError):
        dc.load()
        import ctypes
        dc._check(dc.load().dc_set_window(p._h, 7, 0.0))


def test_doppler_kaiser_second_order_drift_takes_exact_path(dc):
    # |beta - 1| beyond the first-order range: the tapered weights run on the exact-tap path
    alphas = np.array(ALPHA_CASES["fast2"])
    x = synth.complex_gaussian(4096, seed=77, batch=3).astype(np.complex64)
    y = gpu_doppler_taper(dc, x, 32, 2.048e9, 0.0, alphas, 8.0)
    ref = O.run_batch("doppler", x, 2.048e9, 0.0, 32, None, alphas, kaiser=8.0)
    assert rel_l2(y, ref).max() < TOL


def test_doppler_kaiser_alpha_one_bit_exact_and_accuracy(dc):
    x = synth.complex_gaussian(8192, seed=3, batch=2).astype(np.complex64)
    assert np.array_equal(gpu_doppler_taper(dc, x, 32, 51.2e6, 422e6, [1.0, 1.0], 8.0), x)
    # the GPU path reproduces the taper's accuracy gain against the analytic dilated LFM (R17)
    from test_oracle_pins import _tukey_at
    n, fs = 1 << 14, 2.048e9
    T = 0.8 * n / fs
    alpha = O.alpha_from_velocity(5000.0)
    t = np.arange(n) / fs
    truth = _tukey_at(t - (n // 10) / fs, T)
    echo = _tukey_at(alpha * t - (n // 10) / fs, T).astype(np.complex64)[None]
    yk = gpu_doppler_taper(dc, echo, 32, fs, 0.0, [alpha], 8.0)[0]
    yr = gpu_doppler(dc, echo, 32, fs, 0.0, [alpha])[0]
    nrm = np.linalg.norm(truth)
    assert np.linalg.norm(yk - truth) / nrm < 5e-5 < 5e-3 < np.linalg.norm(yr - truth) / nrm


def test_correct_kaiser_train_sampled(dc):
    import torch
    n, batch = 1 << 16, 6
    bank = synth.waveform_bank(n, count=3)
    x = bank[np.arange(batch) % 3]
    tec, alpha = synth.pulse_params(batch)
    p = dc.Plan(n, 2.048e9, 0.0, taps=32)
    p.set_taper(8.0)
    xd = to_dev(x)
    yd = torch.empty_like(xd)
    p.correct(xd, yd, tec, alpha)
    y = from_dev(yd)
    idx = [0, 4, 5]
    ref = O.run_batch("correct", x[idx], 2.048e9, 0.0, 32, tec[idx], alpha[idx], kaiser=8.0)
    assert rel_l2(y[idx], ref).max() < TOL
    with pytest.raises(dc.DispCorrError) as e:
        p.set_taper(-1.0)
    assert e.value.name == "DC_ERR_INVALID_VALUE"
    with pytest.raises(dc.DispCorrError) as e:
        p.set_taper(float("nan"))
    assert e.value.name == "DC_ERR_INVALID_VALUE"


def test_correct_c4_bench_workload_sampled(dc):
    # The bench's exact workload and launch configuration: the full C4 train (1024 x 2^20, W = 32,
    # 16 launch groups of 64 pulses), built the way bench.py builds it; parity on the SURVEY 8(d)
    # sample {0, 64, ..., 960} u {1, 511, 1023}, computed one pulse at a time by the oracle.
    import torch
    n, pulses = 1 << 20, 1024
    cfg = synth.pulse_train(pulses, n)
    bank_d = torch.from_numpy(cfg["bank"]).cuda()
    x = bank_d[torch.from_numpy(cfg["index"]).cuda()].contiguous()
    del bank_d
    y = torch.empty_like(x)
    p = dc.Plan(n, cfg["fs"], 0.0, taps=cfg["W"])
    p.correct(x, y, cfg["tec"], cfg["alpha"])
    p.sync()
    idx = sorted(set(range(0, pulses, 64)) | {1, 511, 1023})
    ys = y[torch.tensor(idx, device="cuda")].cpu().numpy()
    ref = O.run_batch("correct", cfg["bank"][cfg["index"][idx]], cfg["fs"], 0.0, cfg["W"], cfg["tec"][idx],
                      cfg["alpha"][idx])
    assert rel_l2(ys, ref).max() < TOL


def test_large_batch_device_param_expansion_is_bit_identical(dc):
    # batches above 4096 pulses stage raw tec / alpha and derive the per-pulse parameters on the
    # device; the result must equal the host-derived path bit for bit (same binary64 operations)
    import torch
    n, batch = 256, 5000
    x = torch.from_numpy(synth.complex_gaussian(n, seed=21, batch=batch).astype(np.complex64)).cuda()
    tec, alpha = synth.pulse_params(batch)
    p = dc.Plan(n, 2.048e9, 0.0, taps=16)
    y_big = torch.empty_like(x)
    p.correct(x, y_big, tec, alpha)                              # one call: device expansion
    y_small = torch.empty_like(x)
    for lo in range(0, batch, 2500):                             # two calls: host derivation
        p.correct(x[lo:lo + 2500], y_small[lo:lo + 2500], tec[lo:lo + 2500], alpha[lo:lo + 2500])
    p.sync()
    assert torch.equal(y_big, y_small)
    xi = x.clone()
    p.iono(xi, tec)                                              # tec only
    xs = x.clone()
    for lo in range(0, batch, 2500):
        p.iono(xs[lo:lo + 2500], tec[lo:lo + 2500])
    yd = torch.empty_like(x)
    p.doppler(x, yd, alpha)                                      # alpha only
    yd2 = torch.empty_like(x)
    for lo in range(0, batch, 2500):
        p.doppler(x[lo:lo + 2500], yd2[lo:lo + 2500], alpha[lo:lo + 2500])
    p.sync()
    assert torch.equal(xi, xs) and torch.equal(yd, yd2)
    idx = [0, 4097, 4999]
    ref = O.run_batch("correct", x[idx].cpu().numpy(), 2.048e9, 0.0, 16, tec[idx], alpha[idx])
    assert rel_l2(y_big[idx].cpu().numpy(), ref).max() < TOL


@pytest.mark.parametrize("alpha", [1.25, 0.8, 1.0 + 2.0 ** -20, 1.0 - 2.0 ** -22, 4.0 / 3.0])
def test_doppler_window_boundaries_match_oracle(dc, alpha):
    # alphas whose positions m beta land on or next to integers and half-integers, where a fused
    # multiply-add (one rounding) and the oracle's fl(fl(m beta) - W/2) (two roundings) can disagree
    # on window membership (R9); every path must take the oracle's decisions
    n = 4096
    x = synth.complex_gaussian(n, seed=31, batch=1).astype(np.complex64)
    for W in (4, 16, 25, 32):
        y = gpu_doppler(dc, x, W, 2.048e9, 0.0, [alpha])
        ref = O.run_batch("doppler", x, 2.048e9, 0.0, W, None, [alpha])
        assert rel_l2(y, ref).max() < TOL, (alpha, W)


def test_iono_c3_geometry_cubic_pin_on_gpu(dc):
    # f0 = 411 MHz, B = 18 MHz, T = 500 us (1,024,000 samples) in a 2^20 window at
    # 2.048 GHz, 100 TECU: the GPU's Eq. 15 correction vs the CUBIC truth loses ~0.00135 dB (the
    # uncorrected echo ~1.347 dB), reproducing the survey's FP64 numbers on the GPU output
    n, fs, tec, T = 1 << 20, 2.048e9, 1e18, 500e-6
    x = synth.lfm(n, fs, 411e6, 18e6, T, offset=8192).astype(np.complex64)
    y = gpu_iono(dc, x[None], fs, 0.0, [tec])[0]
    cub = L.cubic_waveform(411e6, 18e6, T, O.k2_per_tec() * tec, fs)
    loss = L.matched_filter_loss_db(y, cub)
    assert loss < 0.01 and loss == pytest.approx(0.00135, abs=5e-4)
    assert 1.2 < L.matched_filter_loss_db(x, cub) < 1.5


def test_correct_c3_physics_dilated_dispersed_echo(dc):
    # C3 end to end: the echo of a 411 MHz / 500 us LFM from a target at +5 km/s through 100 TECU is
    # S(alpha t) (analytic dilation) dispersed by Eq. 14; dc_correct (iono then Doppler, W = 32) must
    # recover the transmitted chirp up to the windowed-sinc error and the order-of-operations residue
    # (SURVEY Q15), while the uncorrected echo loses > 1 dB
    import torch
    n, fs, tec, T, off = 1 << 20, 2.048e9, 1e18, 500e-6, 8192
    alpha = O.alpha_from_velocity(5000.0)
    tx = synth.lfm(n, fs, 411e6, 18e6, T, offset=off)
    dil = synth.lfm(n, fs, 411e6, 18e6, T, offset=off / alpha, time_scale=alpha)        # S(alpha t)
    echo = O.iono(dil, fs, 0.0, tec, distort=True).astype(np.complex64)                    # Eq. 14
    p = dc.Plan(n, fs, 0.0, taps=32)
    xd = to_dev(echo[None])
    yd = torch.empty_like(xd)
    p.correct(xd, yd, [tec], [alpha])
    y = from_dev(yd)[0]
    ref = tx[off:off + int(T * fs)]
    loss = L.matched_filter_loss_db(y, ref)
    unc = L.matched_filter_loss_db(echo, ref)
    iono_only = L.matched_filter_loss_db(from_dev(p.iono(xd.clone(), [tec]))[0], ref)
    # FP64 oracle on the same input: 1.0e-4 dB corrected, 0.093 dB iono-only, 2.15 dB uncorrected
    assert loss < 1e-3 and iono_only > 0.05 and unc > 2.0, (loss, iono_only, unc)


# ----------------------------------------------------------------------------- fused single-round-trip dc_correct (NEXT-1)
@pytest.mark.parametrize("log2n", [10, 11, 12, 13, 14])
@pytest.mark.parametrize("W", [16, 32])
@pytest.mark.parametrize("case", ["fast1", "second"])
def test_correct_fused_small_vs_oracle(dc, log2n, W, case):
    # n = 2^10 .. 2^14 with W = 16 / 32 and a first/second-order alpha run iono + Doppler in ONE kernel
    # (the ionospheric result stays in shared memory); parity with the oracle's Doppler(iono(x))
    import torch
    n = 1 << log2n
    # drift |1/alpha - 1| (R/2 + 1/2) within the first-order (<= 2e-4) or second-order (<= 2e-3) range
    alphas = np.array(ALPHA_CASES["fast1"] if case == "fast1" else [1 + 2e-4, 1 - 3e-4, 1 + 1e-4])
    alphas = np.append(alphas, 1.0)
    batch = len(alphas) + 2                       # ragged: not a multiple of the tile's pulses
    alphas = np.resize(alphas, batch)
    x = synth.complex_gaussian(n, seed=log2n * 7 + W, batch=batch).astype(np.complex64)
    tec = np.linspace(0.0, 2e18, batch)
    for fs, fc in ((2.048e9, 0.0), (51.2e6, 422e6)):
        p = dc.Plan(n, fs, fc, taps=W)
        p.profile_enable(True)
        xd = to_dev(x)
        yd = torch.empty_like(xd)
        p.correct(xd, yd, tec, alphas)
        prof = p.profile_read()
        assert prof["correct_fused"]["launches"] >= 1 and prof["doppler"]["launches"] == 0
        ref = O.run_batch("correct", x, fs, fc, W, tec, alphas)
        assert rel_l2(from_dev(yd), ref).max() < TOL, (fs, fc)


def test_correct_fused_falls_back_outside_its_range(dc):
    # taper, W = 25 and the exact-tap alpha range take the two-kernel path (and still match the oracle)
    import torch
    n = 4096
    x = synth.complex_gaussian(n, seed=5, batch=3).astype(np.complex64)
    tec = [1e18, 0.0, 5e17]
    for W, kaiser, alphas in ((25, 0.0, [1 + 3e-5, 1.0, 1 - 2e-5]), (32, 8.0, [1 + 3e-5, 1.0, 1 - 2e-5]),
                              (32, 0.0, [1.05, 0.97, 1.0])):
        p = dc.Plan(n, 2.048e9, 0.0, taps=W)
        if kaiser:
            p.set_taper(kaiser)
        p.profile_enable(True)
        xd = to_dev(x)
        yd = torch.empty_like(xd)
        p.correct(xd, yd, tec, alphas)
        prof = p.profile_read()
        assert prof["correct_fused"]["launches"] == 0 and prof["doppler"]["launches"] >= 1
        ref = O.run_batch("correct", x, 2.048e9, 0.0, W, tec, alphas, kaiser=kaiser)
        assert rel_l2(from_dev(yd), ref).max() < TOL, (W, kaiser)


def test_correct_host_fused_small_matches_device(dc):
    # dc_correct_host runs the same fused kernel per transfer chunk: bit-identical to the device path
    import torch
    n, batch = 4096, 37
    x = synth.complex_gaussian(n, seed=77, batch=batch).astype(np.complex64)
    tec, alpha = synth.pulse_params(batch, seed=5)
    p = dc.Plan(n, 2.048e9, 0.0, taps=32)
    xd = to_dev(x)
    yd = torch.empty_like(xd)
    p.correct(xd, yd, tec, alpha)
    yh = np.empty_like(x)
    p.correct_host(x, yh, tec, alpha)
    assert np.array_equal(from_dev(yd), yh)


def test_doppler_hann_full_size_sampled(dc):
    # Hann window on the C3/C4 pulse length, sampled outputs (the taper path of the T = 256 kernel)
    import torch
    n = 1 << 20
    x = synth.complex_gaussian(n, seed=93, batch=2).astype(np.complex64)
    alphas = [O.alpha_from_velocity(4000.0), O.alpha_from_velocity(-2500.0)]
    p = dc.Plan(n, 2.048e9, 0.0, taps=32)
    p.set_window("hann")
    xd = to_dev(x)
    yd = torch.empty_like(xd)
    p.doppler(xd, yd, alphas)
    y = from_dev(yd)
    idx = np.unique(np.concatenate([[0, 1, n - 1], np.random.default_rng(4).integers(0, n, 200)]))
    for i, a in enumerate(alphas):
        ref = O.doppler_at(x[i].astype(np.complex128), 32, 2.048e9, 0.0, a, idx, kaiser=O.HANN)
        assert rel_l2(y[i][idx], ref).max() < TOL


# ----------------------------------------------------------------------------- long-pulse Doppler kernels (R = 13)
# n >= 2^16 runs doppler_pipe_kernel at 256 / 512 threads with R = 13 outputs per thread for W <= 32; the
# first-order path holds up to drift |beta - 1| (R + 1) / 2 = 5e-4 (|beta - 1| ~ 7.1e-5): "edge" sits just
# inside it, "fast2" on the second-order path
LONG_ALPHAS = {
    "fast1": [1 + 3.3e-5, 1 - 3.3e-5, 1.0],
    "edge": [1 + 7.0e-5, 1 - 7.1e-5, 1 + 2e-6],
    "fast2": [1 + 2.5e-4, 1 - 2.0e-4, 1 + 1e-4],
}


@pytest.mark.parametrize("case", list(LONG_ALPHAS))
@pytest.mark.parametrize("W", [8, 16, 25, 32, 64])
def test_doppler_long_pulse_kernels_vs_oracle(dc, case, W):
    n = 1 << 16
    alphas = np.array(LONG_ALPHAS[case])
    x = synth.complex_gaussian(n, seed=W + 31, batch=len(alphas)).astype(np.complex64)
    for fs, fc in ((2.048e9, 0.0), (51.2e6, 422e6)):
        y = gpu_doppler(dc, x, W, fs, fc, alphas)
        ref = O.run_batch("doppler", x, fs, fc, W, None, alphas)
        assert rel_l2(y, ref).max() < TOL, (case, W, fs, fc, rel_l2(y, ref).max())
        if case == "fast1":
            assert np.array_equal(y[2], x[2])  # alpha = 1 bit-exact on the R = 13 kernels too
    if case != "fast2":  # tapered: first-order path only
        y = gpu_doppler_taper(dc, x, W, 2.048e9, 0.0, alphas, 8.0)
        ref = O.run_batch("doppler", x, 2.048e9, 0.0, W, None, alphas, kaiser=8.0)
        assert rel_l2(y, ref).max() < TOL, (case, W, "kaiser", rel_l2(y, ref).max())
