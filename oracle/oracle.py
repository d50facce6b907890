"""ctypes front end of the FP64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` leg.  The product package
(``paper_2508_04951_b200``) never imports this module and shares no code with it.

Every function follows the paper step by step; see the citations in oracle.c
(Eq. 15 P:L231-236 for the ionospheric correction, Eq. 16 P:L285-288 with the
window of P:L533 for the Doppler resampler) and the readings R1..R12 in
DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# overridable only for the mutation check in tools/mutate_oracle.py
_SRC = os.environ.get("DISPCORR_ORACLE_SRC", os.path.join(_HERE, "oracle.c"))
_LIB = os.environ.get("DISPCORR_ORACLE_LIB", os.path.join(_HERE, "liboracle.so"))

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with plain -O2 (no fast-math) into liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-fno-fast-math",
               "-ffp-contract=off", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        d, i64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_int
        p = ctypes.c_void_p
        lib.orc_k2_per_tec.restype = d
        lib.orc_speed_of_light.restype = d
        lib.orc_group_delay.restype = d
        lib.orc_group_delay.argtypes = [d, d]
        lib.orc_alpha_from_velocity.restype = d
        lib.orc_alpha_from_velocity.argtypes = [d]
        lib.orc_dft.argtypes = [i64, p, p, i32]
        lib.orc_fft.argtypes = [i64, p, i32]
        lib.orc_bin_frequency.restype = d
        lib.orc_bin_frequency.argtypes = [i64, i64, d, d]
        lib.orc_iono_phase_cycles.restype = d
        lib.orc_iono_phase_cycles.argtypes = [d, d]
        lib.orc_iono_dir.restype = i32
        lib.orc_iono_dir.argtypes = [i64, d, d, d, i32, i32, p, p]
        lib.orc_sinc.restype = d
        lib.orc_sinc.argtypes = [d]
        lib.orc_doppler.restype = i32
        lib.orc_doppler.argtypes = [i64, i32, d, d, d, p, p]
        lib.orc_doppler_win.restype = i32
        lib.orc_doppler_win.argtypes = [i64, i32, d, d, d, d, p, p]
        lib.orc_doppler_at.restype = i32
        lib.orc_doppler_at.argtypes = [i64, i32, d, d, d, d, p, i64, p, p]
        lib.orc_bessel_i0.restype = d
        lib.orc_bessel_i0.argtypes = [d]
        lib.orc_kaiser.restype = d
        lib.orc_kaiser.argtypes = [d, d, d]
        lib.orc_hann.restype = d
        lib.orc_hann.argtypes = [d, d]
        lib.orc_run_batch_win.restype = i32
        lib.orc_run_batch_win.argtypes = [i32, i64, i64, d, d, i32, d, p, p, p, p, i32, i32]
        lib.orc_pq_resample.restype = i32
        lib.orc_pq_resample.argtypes = [i64, i64, p, p]
        lib.orc_pq_length.restype = i64
        lib.orc_pq_length.argtypes = [i64, d]
        lib.orc_doppler_pq.restype = i32
        lib.orc_doppler_pq.argtypes = [i64, d, d, d, p, p]
        lib.orc_pq_resample_at.restype = i32
        lib.orc_pq_resample_at.argtypes = [i64, i64, p, i64, p, p]
        lib.orc_doppler_pq_at.restype = i32
        lib.orc_doppler_pq_at.argtypes = [i64, d, d, d, p, i64, p, p]
        lib.orc_doppler_exact.restype = i32
        lib.orc_doppler_exact.argtypes = [i64, d, d, d, p, p]
        lib.orc_run_batch.restype = i32
        lib.orc_correlate.argtypes = [i64, p, i64, p, i64, p, p]
        lib.orc_compress.argtypes = [i64, d, d, d, p, i64, p, i64, p, p]
        lib.orc_run_batch.argtypes = [i32, i64, i64, d, d, i32, p, p, p, p, i32, i32]
        lib.orc_max_threads.restype = i32
        _lib = lib
    return _lib


def _c128(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.complex128))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ----------------------------------------------------------------------------- constants
def k2_per_tec() -> float:
    """K2/E = q_e^2/(8 pi^2 m_e eps0), Eq. 1, CODATA 2018."""
    return _load().orc_k2_per_tec()


def speed_of_light() -> float:
    return _load().orc_speed_of_light()


def group_delay(f_hz: float, tec: float) -> float:
    """One-way tau(f) = K2/(c f^2), Eq. 1."""
    return _load().orc_group_delay(f_hz, tec)


def alpha_from_velocity(v_mps: float) -> float:
    """alpha = (1+v/c)/(1-v/c)."""
    return _load().orc_alpha_from_velocity(v_mps)


def bin_frequency(k: int, n: int, fs: float, fc: float) -> float:
    return _load().orc_bin_frequency(k, n, fs, fc)


def iono_phase_cycles(f_hz: float, tec: float) -> float:
    """nu = 2 K2/(c f) cycles (0 for f <= 0)."""
    return _load().orc_iono_phase_cycles(f_hz, tec)


def sinc(d: float) -> float:
    return _load().orc_sinc(d)


# ----------------------------------------------------------------------------- transforms
def dft(x, sign: int = -1) -> np.ndarray:
    x = _c128(x)
    X = np.empty_like(x)
    _load().orc_dft(x.size, _ptr(x), _ptr(X), sign)
    return X


def fft(x, sign: int = -1) -> np.ndarray:
    X = _c128(x).copy()
    n = X.size
    if n & (n - 1):
        raise ValueError("radix-2 oracle FFT needs a power of two")
    _load().orc_fft(n, _ptr(X), sign)
    return X


# ----------------------------------------------------------------------------- method
def iono(x, fs: float, fc: float, tec: float, direct: bool = False, distort: bool = False) -> np.ndarray:
    """Eq. 15 correction (distort=False) or Eq. 14 distortion (distort=True) of one pulse."""
    x = _c128(x)
    y = np.empty_like(x)
    n = x.size
    if not direct and (n & (n - 1)):
        raise ValueError("radix-2 path needs a power of two; use direct=True")
    rc = _load().orc_iono_dir(n, fs, fc, tec, +1 if distort else -1, 1 if direct else 0,
                              _ptr(x), _ptr(y))
    if rc:
        raise RuntimeError(f"orc_iono_dir failed ({rc})")
    return y


def doppler(x, W: int, fs: float, fc: float, alpha: float, kaiser: float = 0.0) -> np.ndarray:
    """Windowed Whittaker-Shannon resampling onto t/alpha, Eq. 16 + window; optional
    Kaiser taper of shape `kaiser` (reading R17; 0 = rectangular, R11)."""
    x = _c128(x)
    y = np.empty_like(x)
    rc = _load().orc_doppler_win(x.size, int(W), fs, fc, alpha, float(kaiser), _ptr(x), _ptr(y))
    if rc:
        raise RuntimeError(f"orc_doppler_win failed ({rc})")
    return y


def doppler_at(x, W: int, fs: float, fc: float, alpha: float, idx, kaiser: float = 0.0) -> np.ndarray:
    """The outputs of doppler() at the sample positions idx only (same arithmetic per output)."""
    x = _c128(x)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    y = np.empty(idx.size, np.complex128)
    rc = _load().orc_doppler_at(x.size, int(W), fs, fc, alpha, float(kaiser), _ptr(x), idx.size,
                                idx.ctypes.data_as(ctypes.c_void_p), _ptr(y))
    if rc:
        raise RuntimeError(f"orc_doppler_at failed ({rc})")
    return y


def bessel_i0(z: float) -> float:
    """Modified Bessel function I0 by its power series (the taper's definition, R17)."""
    return _load().orc_bessel_i0(float(z))


HANN = -1.0  # pass as `kaiser` to select the Hann taper (oracle.c ORC_HANN)


def hann(d: float, L: float) -> float:
    """Hann taper (1 + cos(pi d / L)) / 2 (R17)."""
    return _load().orc_hann(float(d), float(L))


def kaiser(d: float, L: float, kb: float) -> float:
    """Kaiser taper I0(kb sqrt(1 - (d/L)^2)) / I0(kb) (R17)."""
    return _load().orc_kaiser(float(d), float(L), float(kb))


def pq_resample(x, M: int) -> np.ndarray:
    """FFT P/Q resampling of x (length n) to M samples (reading R18), first min(n, M) outputs, zero-padded to n."""
    x = _c128(x)
    y = np.empty_like(x)
    rc = _load().orc_pq_resample(x.size, int(M), _ptr(x), _ptr(y))
    if rc:
        raise RuntimeError(f"orc_pq_resample failed ({rc})")
    return y


def pq_length(n: int, alpha: float) -> int:
    """M = n + 2 round((n alpha - n) / 2): an even number of samples added or removed (R18)."""
    return _load().orc_pq_length(int(n), float(alpha))


def doppler_pq(x, fs: float, fc: float, alpha: float) -> np.ndarray:
    """Doppler correction by FFT P/Q resampling onto t n / M (+ carrier term, R10/R18)."""
    x = _c128(x)
    y = np.empty_like(x)
    rc = _load().orc_doppler_pq(x.size, fs, fc, alpha, _ptr(x), _ptr(y))
    if rc:
        raise RuntimeError(f"orc_doppler_pq failed ({rc})")
    return y


def pq_resample_at(x, M: int, idx) -> np.ndarray:
    """pq_resample(x, M) at the output indices idx only (radix-2 FFT forward; n a power of two)."""
    x = _c128(x)
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
    y = np.empty(idx.size, dtype=np.complex128)
    rc = _load().orc_pq_resample_at(x.size, int(M), _ptr(x), idx.size, idx.ctypes.data, _ptr(y))
    if rc:
        raise RuntimeError(f"orc_pq_resample_at failed ({rc})")
    return y


def doppler_pq_at(x, fs: float, fc: float, alpha: float, idx) -> np.ndarray:
    """doppler_pq(x, fs, fc, alpha) at the output indices idx only."""
    x = _c128(x)
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
    y = np.empty(idx.size, dtype=np.complex128)
    rc = _load().orc_doppler_pq_at(x.size, fs, fc, alpha, _ptr(x), idx.size, idx.ctypes.data, _ptr(y))
    if rc:
        raise RuntimeError(f"orc_doppler_pq_at failed ({rc})")
    return y


def doppler_exact(x, fs: float, fc: float, alpha: float) -> np.ndarray:
    """Unwindowed Eq. 16 (O(n^2)) -- brute-force pin only."""
    x = _c128(x)
    y = np.empty_like(x)
    _load().orc_doppler_exact(x.size, fs, fc, alpha, _ptr(x), _ptr(y))
    return y


def correct(x, W: int, fs: float, fc: float, tec: float, alpha: float) -> np.ndarray:
    """dc_correct = doppler(iono(x)), iono first (reading R7)."""
    return doppler(iono(x, fs, fc, tec), W, fs, fc, alpha)


def correlate(y, r, idx=None) -> np.ndarray:
    """Circular matched filter z_m = sum_s y[(s+m) mod n] conj(r_s) (direct sum), at outputs idx."""
    y, r = _c128(y), _c128(r)
    n, L = y.size, r.size
    ix = None if idx is None else np.ascontiguousarray(idx, dtype=np.int64)
    z = np.empty(n if ix is None else ix.size, dtype=np.complex128)
    rc = _load().orc_correlate(n, _ptr(y), L, _ptr(r), 0 if ix is None else ix.size,
                               None if ix is None else _ptr(ix), _ptr(z))
    if rc:
        raise RuntimeError(f"orc_correlate failed ({rc})")
    return z


def compress(x, fs: float, fc: float, tec: float, r, idx=None) -> np.ndarray:
    """Pulse compression of the iono-corrected pulse: correlate(iono(x), r) (reading R16)."""
    x, r = _c128(x), _c128(r)
    n, L = x.size, r.size
    ix = None if idx is None else np.ascontiguousarray(idx, dtype=np.int64)
    z = np.empty(n if ix is None else ix.size, dtype=np.complex128)
    rc = _load().orc_compress(n, fs, fc, tec, _ptr(x), L, _ptr(r), 0 if ix is None else ix.size,
                              None if ix is None else _ptr(ix), _ptr(z))
    if rc:
        raise RuntimeError(f"orc_compress failed ({rc})")
    return z


STAGES = {"iono": 1, "doppler": 2, "correct": 3}


def run_batch(stage: str, x64: np.ndarray, fs: float, fc: float, W: int,
              tec=None, alpha=None, nthreads: int = 0, direct: bool = False, kaiser: float = 0.0) -> np.ndarray:
    """Batched oracle on complex64 input [batch, n] (upcast exactly), complex128 output."""
    x64 = np.ascontiguousarray(x64, dtype=np.complex64)
    if x64.ndim == 1:
        x64 = x64[None]
    batch, n = x64.shape
    tec_a = np.ascontiguousarray(np.zeros(batch) if tec is None else np.broadcast_to(tec, (batch,)), dtype=np.float64)
    alpha_a = np.ascontiguousarray(np.ones(batch) if alpha is None else np.broadcast_to(alpha, (batch,)), dtype=np.float64)
    y = np.empty((batch, n), dtype=np.complex128)
    rc = _load().orc_run_batch_win(STAGES[stage], n, batch, fs, fc, int(W), float(kaiser), _ptr(tec_a),
                                   _ptr(alpha_a), _ptr(x64), _ptr(y), int(nthreads), 1 if direct else 0)
    if rc:
        raise RuntimeError(f"orc_run_batch failed ({rc})")
    return y


def max_threads() -> int:
    return _load().orc_max_threads()
