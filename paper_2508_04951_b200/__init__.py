"""paper_2508_04951_b200 -- B200-native per-pulse dispersion correction (arXiv 2508.04951).

Thin ctypes binding over the C ABI of ``libdispcorr`` (include/libdispcorr.h).  This
module only marshals arguments: every step of the hot path (FFT, ionospheric phase,
inverse FFT, windowed-sinc resampling) runs in the CUDA kernels of the library.  There
is no CPU fallback: if the shared library is missing or a call fails, an exception is
raised.

    import torch, paper_2508_04951_b200 as dc
    plan = dc.Plan(n=1 << 20, fs=2.048e9, fc=0.0, taps=32)
    plan.iono(x, tec)                 # x: torch.complex64 [batch, n] on cuda, in place (Eq. 15)
    plan.doppler(x, y, alpha)         # y = resampled onto t/alpha (Eq. 16, windowed)
    plan.correct(x, y, tec, alpha)    # both stages, iono first
    plan.set_reference(r); plan.compress(x, z, tec)   # iono correction + matched filter (fused)
    plan.doppler_pq(x, y, alpha)      # FFT P/Q resampling (the paper's second Doppler method)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["Plan", "DispCorrError", "alpha_from_velocity", "k2_per_tec", "library_path", "load", "use_library", "STATUS"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "lib", "libdispcorr.so")
_lib = None

STATUS = {
    0: "DC_OK", 1: "DC_ERR_INVALID_VALUE", 2: "DC_ERR_NULL_POINTER", 3: "DC_ERR_MISALIGNED",
    4: "DC_ERR_ALIASING", 5: "DC_ERR_OUT_OF_MEMORY", 6: "DC_ERR_CUDA", 7: "DC_ERR_UNSUPPORTED_DEVICE",
    8: "DC_ERR_NOT_DEVICE_MEMORY",
}


class DispCorrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


KERNEL_CLASSES = ("iono_small", "fourstep_A", "fourstep_B", "fourstep_C", "doppler", "pq", "correct_fused")


class Profile(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64 * 7), ("ms", ctypes.c_double * 7), ("samples", ctypes.c_int64 * 7)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("log2n", ctypes.c_int), ("taps", ctypes.c_int), ("regime", ctypes.c_int),
                ("n1", ctypes.c_int64), ("n2", ctypes.c_int64), ("chunk_pulses", ctypes.c_int64),
                ("scratch_bytes", ctypes.c_int64), ("sm_count", ctypes.c_int), ("kernel_launches", ctypes.c_int64)]


def library_path() -> str:
    return _LIB_PATH


def use_library(path: str):
    """Kernel-tuning tools only: load an alternative in-tree build (e.g. one compiled with extra -D
    flags by ``build.build(out=...)``) instead of lib/libdispcorr.so.  Must precede the first load()."""
    global _LIB_PATH
    if _lib is not None:
        raise RuntimeError("libdispcorr is already loaded")
    _LIB_PATH = os.path.abspath(path)


def load():
    """Load libdispcorr.so (built by ``python -m paper_2508_04951_b200.build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"libdispcorr.so not built ({_LIB_PATH}); run `python -m paper_2508_04951_b200.build`")
    lib = ctypes.CDLL(_LIB_PATH)
    i64, i32, d, p = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
    pd = ctypes.POINTER(ctypes.c_double)
    sigs = {
        "dc_plan": ([ctypes.POINTER(p), i64, d, d, i32, i32, p], i32),
        "dc_plan_destroy": ([p], i32),
        "dc_set_stream": ([p, p], i32),
        "dc_sync": ([p], i32),
        "dc_iono": ([p, p, i64, pd], i32),
        "dc_iono_distort": ([p, p, i64, pd], i32),
        "dc_doppler": ([p, p, p, i64, pd], i32),
        "dc_doppler_pq": ([p, p, p, i64, pd], i32),
        "dc_set_reference": ([p, p, i64], i32),
        "dc_set_taper": ([p, d], i32),
        "dc_set_window": ([p, i32, d], i32),
        "dc_compress": ([p, p, p, i64, pd], i32),
        "dc_correct": ([p, p, p, i64, pd, pd], i32),
        "dc_correct_host": ([p, p, p, i64, pd, pd], i32),
        "dc_plan_info": ([p, ctypes.POINTER(PlanInfo)], i32),
        "dc_profile_enable": ([p, i32], i32),
        "dc_profile_read": ([p, ctypes.POINTER(Profile)], i32),
        "dc_status_string": ([i32], ctypes.c_char_p),
        "dc_last_error_message": ([], ctypes.c_char_p),
        "dc_alpha_from_velocity": ([d], d),
        "dc_k2_per_tec": ([], d),
        "dc_version": ([], i32),
    }
    for name, (args, res) in sigs.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _check(status: int):
    if status != 0:
        raise DispCorrError(status, load().dc_last_error_message().decode())


def alpha_from_velocity(v_mps: float) -> float:
    """alpha = (1 + v/c)/(1 - v/c), v > 0 approaching."""
    return load().dc_alpha_from_velocity(float(v_mps))


def k2_per_tec() -> float:
    """K2 / TEC = q_e^2 / (8 pi^2 m_e eps0) (Eq. 1)."""
    return load().dc_k2_per_tec()


def _f64(a, batch: int, name: str):
    arr = np.ascontiguousarray(np.broadcast_to(np.asarray(a, dtype=np.float64), (batch,)))
    return arr, arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _dev_ptr(t, name: str, n: int):
    """(pointer, batch) of a complex64 CUDA tensor shaped [batch, n] or [n]."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor on a CUDA device")
    if t.dtype != torch.complex64:
        raise TypeError(f"{name} must be complex64 (got {t.dtype})")
    if not t.is_cuda:
        raise TypeError(f"{name} must be on a CUDA device")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.numel() % n:
        raise ValueError(f"{name} has {t.numel()} samples, not a multiple of n = {n}")
    return ctypes.c_void_p(t.data_ptr()), t.numel() // n


def _host_ptr(a, name: str, n: int):
    import torch
    if isinstance(a, torch.Tensor):
        if a.is_cuda or a.dtype != torch.complex64 or not a.is_contiguous():
            raise TypeError(f"{name} must be a contiguous complex64 CPU tensor")
        return ctypes.c_void_p(a.data_ptr()), a.numel() // n
    if not (isinstance(a, np.ndarray) and a.dtype == np.complex64 and a.flags.c_contiguous):
        raise TypeError(f"{name} must be a contiguous complex64 numpy array or CPU tensor")
    return ctypes.c_void_p(a.ctypes.data), a.size // n


class Plan:
    """A libdispcorr plan for pulses of n samples (power of two, 2..2^24) at fs Hz whose DFT
    bin k maps to fc + fftfreq(k) Hz, with a `taps`-sample sinc window."""

    def __init__(self, n: int, fs: float, fc: float = 0.0, taps: int = 32, device: int | None = None,
                 stream=None):
        import torch
        lib = load()
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        explicit_stream = stream is not None
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.n, self.fs, self.fc, self.taps = int(n), float(fs), float(fc), int(taps)
        h = ctypes.c_void_p()
        _check(lib.dc_plan(ctypes.byref(h), self.n, self.fs, self.fc, self.taps, self.device,
                           ctypes.c_void_p(stream.cuda_stream)))
        self._h = h
        self._stream = stream
        # an explicit stream pins the plan to it; otherwise calls follow torch's current stream
        self.follow_current_stream = not explicit_stream

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            load().dc_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_stream(self, stream):
        """Pin the plan to `stream` (it stops following torch's current stream); later work on
        `stream` is ordered after the plan's earlier work (dc_set_stream)."""
        self._retarget(stream)
        self.follow_current_stream = False

    def _retarget(self, stream):
        _check(load().dc_set_stream(self._h, ctypes.c_void_p(stream.cuda_stream)))
        self._stream = stream

    def _follow_stream(self):
        # enqueue on torch's current stream of the plan's device (like a torch op), with the
        # plan's earlier work ordered before it (dc_set_stream)
        if not self.follow_current_stream:
            return
        import torch
        cur = torch.cuda.current_stream(self.device)
        if cur.cuda_stream != self._stream.cuda_stream:
            self._retarget(cur)

    def sync(self):
        _check(load().dc_sync(self._h))

    def info(self) -> dict:
        inf = PlanInfo()
        _check(load().dc_plan_info(self._h, ctypes.byref(inf)))
        return {f: getattr(inf, f) for f, _ in PlanInfo._fields_}

    def profile_enable(self, on: bool = True):
        """Bracket every kernel launch with CUDA events (resets the counters)."""
        _check(load().dc_profile_enable(self._h, 1 if on else 0))

    def profile_read(self) -> dict:
        """{class: {"launches", "ms", "samples"}} since the last profile_enable()."""
        pr = Profile()
        _check(load().dc_profile_read(self._h, ctypes.byref(pr)))
        return {name: {"launches": pr.launches[i], "ms": pr.ms[i], "samples": pr.samples[i]}
                for i, name in enumerate(KERNEL_CLASSES)}

    # -- hot path
    def iono(self, x, tec):
        """Eq. 15 ionospheric correction of x [batch, n] in place; tec in el/m^2 per pulse."""
        px, batch = _dev_ptr(x, "x", self.n)
        tec_a, pt = _f64(tec, batch, "tec")
        self._follow_stream()
        _check(load().dc_iono(self._h, px, batch, pt))
        return x

    def iono_distort(self, x, tec):
        """Eq. 14 forward ionospheric model of x [batch, n] in place."""
        px, batch = _dev_ptr(x, "x", self.n)
        tec_a, pt = _f64(tec, batch, "tec")
        self._follow_stream()
        _check(load().dc_iono_distort(self._h, px, batch, pt))
        return x

    def set_taper(self, kaiser: float = 0.0):
        """Kaiser taper (shape `kaiser`, 0 = rectangular) of the Doppler sinc window (reading R17)."""
        _check(load().dc_set_taper(self._h, float(kaiser)))
        return self

    WINDOWS = {"rect": 0, "kaiser": 1, "hann": 2}

    def set_window(self, kind: str = "rect", param: float = 0.0):
        """Window of the Doppler sinc taps: "rect", "kaiser" (shape `param`) or "hann" (reading R17)."""
        _check(load().dc_set_window(self._h, self.WINDOWS[kind], float(param)))
        return self

    def set_reference(self, r):
        """Matched-filter reference r (complex64 CUDA tensor of L <= n samples) for compress()."""
        import torch
        if not isinstance(r, torch.Tensor) or r.dtype != torch.complex64 or not r.is_cuda or not r.is_contiguous():
            raise TypeError("r must be a contiguous complex64 CUDA tensor")
        self._follow_stream()
        _check(load().dc_set_reference(self._h, ctypes.c_void_p(r.data_ptr()), int(r.numel())))
        self._ref = r  # keep alive until the plan stream has consumed it
        return self

    def compress(self, x, z, tec):
        """z = circular matched filter of iono(x) against the reference (z may be x)."""
        px, batch = _dev_ptr(x, "x", self.n)
        pz, bz = _dev_ptr(z, "z", self.n)
        if bz != batch:
            raise ValueError("x and z batch sizes differ")
        tec_a, pt = _f64(tec, batch, "tec")
        self._follow_stream()
        _check(load().dc_compress(self._h, px, pz, batch, pt))
        return z

    def doppler(self, x, y, alpha):
        """Windowed-sinc resampling of x onto t/alpha into y (distinct buffers)."""
        px, batch = _dev_ptr(x, "x", self.n)
        py, by = _dev_ptr(y, "y", self.n)
        if by != batch:
            raise ValueError("x and y batch sizes differ")
        alpha_a, pa = _f64(alpha, batch, "alpha")
        self._follow_stream()
        _check(load().dc_doppler(self._h, px, py, batch, pa))
        return y

    def doppler_pq(self, x, y, alpha):
        """FFT P/Q resampling of x (M = n + 2 round((n alpha - n)/2) samples, reading R18) into y."""
        px, batch = _dev_ptr(x, "x", self.n)
        py, by = _dev_ptr(y, "y", self.n)
        if by != batch:
            raise ValueError("x and y batch sizes differ")
        alpha_a, pa = _f64(alpha, batch, "alpha")
        self._follow_stream()
        _check(load().dc_doppler_pq(self._h, px, py, batch, pa))
        return y

    def correct(self, x, y, tec, alpha):
        """y = doppler(iono(x)); x is left unchanged."""
        px, batch = _dev_ptr(x, "x", self.n)
        py, by = _dev_ptr(y, "y", self.n)
        if by != batch:
            raise ValueError("x and y batch sizes differ")
        tec_a, pt = _f64(tec, batch, "tec")
        alpha_a, pa = _f64(alpha, batch, "alpha")
        self._follow_stream()
        _check(load().dc_correct(self._h, px, py, batch, pt, pa))
        return y

    def correct_host(self, x_host, y_host, tec, alpha):
        """dc_correct on host buffers (numpy complex64 or CPU tensors, pinned for overlap); synchronous."""
        px, batch = _host_ptr(x_host, "x_host", self.n)
        py, by = _host_ptr(y_host, "y_host", self.n)
        if by != batch:
            raise ValueError("x and y batch sizes differ")
        tec_a, pt = _f64(tec, batch, "tec")
        alpha_a, pa = _f64(alpha, batch, "alpha")
        self._follow_stream()
        _check(load().dc_correct_host(self._h, px, py, batch, pt, pa))
        return y_host
