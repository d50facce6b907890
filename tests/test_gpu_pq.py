"""GPU parity of the FFT P/Q resampler (dc_doppler_pq; NEXT-4, reading R18)
against the FP64 oracle (orc_doppler_pq / orc_doppler_pq_at) on identical complex64 inputs.

Bar: per-pulse relative L2 <= 1e-5 (the north_star tolerance) and element-wise max |y - ref| / rms(ref)
<= 1e-4; M == n (no samples added or removed) returns x bit-exactly ("no work was done").
Full outputs up to n = 2^14 (O(n^2) oracle); 2^19 (the paper's E4 pulse) and 2^20 on sampled outputs.
"""
import numpy as np
import pytest

import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-5
TOL_ELEM = 1e-4


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


def check(y, ref):
    y = np.asarray(y, np.complex128)
    rms = np.sqrt(np.mean(np.abs(ref) ** 2))
    rel = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    elem = np.abs(y - ref).max() / rms
    assert rel <= TOL and elem <= TOL_ELEM, (rel, elem)


def alpha_for(n, d, frac=0.3):
    """an alpha whose P/Q length is M = n + d (d even), off the exact grid by `frac` samples"""
    a = (n + d + frac) / n
    assert O.pq_length(n, a) == n + d
    return a


def gpu_pq(dc, x, alphas, fs=2.048e9, fc=0.0):
    n = x.shape[-1]
    p = dc.Plan(n, fs, fc, taps=2)
    xd = to_dev(x)
    yd = to_dev(np.zeros_like(x))
    p.doppler_pq(xd, yd, alphas)
    out = from_dev(yd)
    p.close()
    return out


@pytest.mark.parametrize("log2n", [2, 4, 6, 8, 10, 11, 12, 13, 14])
def test_pq_full_vs_oracle(dc, log2n):
    n = 1 << log2n
    ds = [2, -2, 4, 0] + ([-6, 2 * (n // 8)] if n >= 16 else [])
    x = synth.complex_gaussian(n, seed=100 + log2n, batch=len(ds)).astype(np.complex64)
    alphas = [alpha_for(n, d) for d in ds]
    y = gpu_pq(dc, x, alphas)
    for i, (d, a) in enumerate(zip(ds, alphas)):
        if d == 0:
            assert np.array_equal(y[i], x[i])  # M == n: bit-exact identity
            continue
        check(y[i], O.doppler_pq(x[i].astype(np.complex128), 2.048e9, 0.0, a))


@pytest.mark.parametrize("log2n", [8, 12, 14])
def test_pq_full_vs_oracle_baseband_carrier(dc, log2n):
    # fc = 422 MHz at fs = 51.2 MHz: the R10 carrier term with beta_eff = n / M (reading R18)
    n = 1 << log2n
    ds = [2, -4, 8]
    x = synth.complex_gaussian(n, seed=200 + log2n, batch=len(ds)).astype(np.complex64)
    alphas = [alpha_for(n, d, frac=-0.4) for d in ds]
    y = gpu_pq(dc, x, alphas, fs=51.2e6, fc=422e6)
    for i, a in enumerate(alphas):
        check(y[i], O.doppler_pq(x[i].astype(np.complex128), 51.2e6, 422e6, a))


def test_pq_large_truncation_and_padding(dc):
    # far from the Doppler regime: M = n/2 and M = 3n/2 (the Nyquist fold / split and the zero tail)
    n = 2048
    ds = [-n // 2, n // 2, -(n - 2), 6 * n]
    x = synth.complex_gaussian(n, seed=7, batch=len(ds)).astype(np.complex64)
    alphas = [(n + d + 0.2) / n for d in ds]
    y = gpu_pq(dc, x, alphas)
    for i, a in enumerate(alphas):
        ref = O.doppler_pq(x[i].astype(np.complex128), 2.048e9, 0.0, a)
        M = O.pq_length(n, a)
        if M < n:
            assert not np.any(y[i][M:])  # zero tail (R12)
        check(y[i], ref)


@pytest.mark.parametrize("log2n", [19, 20])
def test_pq_full_size_sampled(dc, log2n):
    # the paper's E4 pulse (f0 = 420 MHz, B = 18 MHz, T = 500 us, N = 2^19, v ~ U(0, 5 km/s)) and
    # the C3/C4 length; v both signs, |v| up to 5 km/s, plus v = 0 (M == n)
    n = 1 << log2n
    fs = 2.048e9 if log2n == 20 else 1.048576e9  # T = 500 us fits in 2^19 samples
    vs = [4000.0, -1500.0, 2600.0, -4999.0, 0.0]
    T = min(500e-6, 0.95 * n / fs)
    x = synth.complex_gaussian(n, seed=log2n, batch=len(vs)).astype(np.complex64)
    x[0] = synth.lfm(n, fs, 420e6, 18e6, T, offset=int(0.02 * n)).astype(np.complex64)
    alphas = [O.alpha_from_velocity(v) for v in vs]
    y = gpu_pq(dc, x, alphas, fs=fs)
    rng = np.random.default_rng(log2n)
    idx = np.unique(np.concatenate([[0, 1, 2, n // 2, n - 2, n - 1], rng.integers(0, n, 120)]))
    for i, a in enumerate(alphas):
        if O.pq_length(n, a) == n:
            assert np.array_equal(y[i], x[i])
            continue
        ref = O.doppler_pq_at(x[i].astype(np.complex128), fs, 0.0, a, idx)
        M = O.pq_length(n, a)
        tail = idx >= M
        assert not np.any(y[i][idx[tail]])
        check(y[i][idx[~tail]], ref[~tail])


def test_pq_many_distinct_lengths_groups_and_cache(dc):
    # more distinct M than the plan's table cache holds (8 tables of 2n at n = 2^23 is 1 GiB): the call
    # runs in groups with LRU table reuse; repeated M values and identity pulses interleaved
    n = 1 << 23
    ds = [2, 4, 6, 8, 10, 12, 14, 16, 18, 0, 2, 20, -2, 4]
    x0 = synth.complex_gaussian(n, seed=31, batch=1).astype(np.complex64)[0]
    x = np.stack([np.roll(x0, 977 * i) for i in range(len(ds))])
    alphas = [alpha_for(n, d) for d in ds]
    y = gpu_pq(dc, x, alphas)
    idx = np.array([0, 3, 1 << 20, n // 2 + 5, n - 7])
    for i in (0, 8, 9, 10, 11, 13):
        if ds[i] == 0:
            assert np.array_equal(y[i], x[i])
            continue
        ref = O.pq_resample_at(x[i].astype(np.complex128), n + ds[i], idx)
        check(y[i][idx], ref)


def test_pq_errors(dc):
    import torch
    p = dc.Plan(1 << 10, 2.048e9, 0.0, taps=8)
    x = to_dev(np.zeros((2, 1024), np.complex64))
    with pytest.raises(dc.DispCorrError) as e:
        p.doppler_pq(x, x, [1.0, 1.0])
    assert e.value.name == "DC_ERR_ALIASING"
    y = torch.empty_like(x)
    with pytest.raises(dc.DispCorrError) as e:
        p.doppler_pq(x, y, [9.0, 1.0])          # M > 8n
    assert e.value.name == "DC_ERR_INVALID_VALUE"
    with pytest.raises(dc.DispCorrError) as e:
        p.doppler_pq(x, y, [1.0, -1.0])
    assert e.value.name == "DC_ERR_INVALID_VALUE"
    big = dc.Plan(1 << 24, 2.048e9, 0.0, taps=8)
    xb = torch.zeros((1, 1 << 24), dtype=torch.complex64, device="cuda")
    with pytest.raises(dc.DispCorrError) as e:
        big.doppler_pq(xb, torch.empty_like(xb), [1.0])
    assert e.value.name == "DC_ERR_INVALID_VALUE"


def test_pq_all_identity_batch_is_a_copy(dc):
    # |n alpha - n| < 1 for every pulse: M == n, nothing added or removed ("no work was done")
    n = 1 << 16
    x = synth.complex_gaussian(n, seed=41, batch=5).astype(np.complex64)
    alphas = [1.0, 1 + 0.4 / n, 1 - 0.9 / n, 1.0, 1 + 0.99 / n]
    assert all(O.pq_length(n, a) == n for a in alphas)
    p = dc.Plan(n, 2.048e9, 0.0, taps=8)
    xd = to_dev(x)
    yd = to_dev(np.zeros_like(x))
    l0 = p.info()["kernel_launches"]
    p.doppler_pq(xd, yd, alphas)
    assert np.array_equal(from_dev(yd), x)
    assert p.info()["kernel_launches"] == l0  # a device copy, no kernels


def test_pq_full_size_baseband_carrier_sampled(dc):
    # 2^20 samples at fs = 204.8 MHz around fc = 422 MHz: the R10 carrier with beta_eff = n / M on sampled
    # outputs, M = n +- 2j for |v| up to 5 km/s
    n, fs, fc = 1 << 20, 204.8e6, 422e6
    vs = [4800.0, -3000.0]
    x = synth.complex_gaussian(n, seed=91, batch=len(vs)).astype(np.complex64)
    alphas = [O.alpha_from_velocity(v) for v in vs]
    assert all(O.pq_length(n, a) != n for a in alphas)
    y = gpu_pq(dc, x, alphas, fs=fs, fc=fc)
    idx = np.unique(np.concatenate([[0, 1, n // 3, n - 40], np.random.default_rng(3).integers(0, n - 40, 60)]))
    for i, a in enumerate(alphas):
        ref = O.doppler_pq_at(x[i].astype(np.complex128), fs, fc, a, idx)
        M = O.pq_length(n, a)
        keep = idx < min(n, M)
        check(y[i][idx[keep]], ref[keep])


def test_pq_plan_reuse_and_stream_order(dc):
    # one plan, consecutive calls with different M sets (table cache hits and rebuilds), results equal a
    # fresh plan's
    import torch
    n = 1 << 14
    x = synth.complex_gaussian(n, seed=92, batch=3).astype(np.complex64)
    sets = [[alpha_for(n, 2), alpha_for(n, -4), 1.0], [alpha_for(n, 6), alpha_for(n, 2), alpha_for(n, -4)]]
    p = dc.Plan(n, 2.048e9, 0.0, taps=8)
    xd = to_dev(x)
    for al in sets:
        yd = torch.empty_like(xd)
        p.doppler_pq(xd, yd, al)
        fresh = gpu_pq(dc, x, al)
        assert np.array_equal(from_dev(yd), fresh)
