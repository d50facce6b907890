"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol that
include/libdispcorr.h declares, and host-side validation rejects bad plans before any CUDA call."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "libdispcorr.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dc_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import paper_2508_04951_b200 as dc
    from paper_2508_04951_b200 import build
    build.build()
    return dc.load()


def test_header_declares_the_hot_path_calls():
    names = declared_functions()
    for required in ("dc_plan", "dc_iono", "dc_doppler", "dc_correct", "dc_plan_destroy", "dc_status_string",
                     "dc_alpha_from_velocity", "dc_k2_per_tec", "dc_correct_host", "dc_doppler_pq", "dc_compress",
                     "dc_set_reference", "dc_set_taper", "dc_iono_distort"):
        assert required in names


def test_every_declared_symbol_is_exported(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_exports_are_only_the_abi(lib):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2508_04951_b200", "lib", "libdispcorr.so")],
                         capture_output=True, text=True).stdout
    exported = sorted(set(l.split()[-1] for l in out.splitlines() if " T " in l))
    assert set(exported) == set(declared_functions())


def test_library_reads_no_environment(lib):
    # no tuning knob reaches the product path: none of libdispcorr's own objects imports getenv (the
    # statically linked CUDA runtime reads CUDA_* variables itself; that is not library behaviour)
    import glob
    import subprocess
    objs = glob.glob(os.path.join(ROOT, "paper_2508_04951_b200", "lib", "obj", "*.o"))
    assert objs
    for o in objs:
        out = subprocess.run(["nm", "--undefined-only", o], capture_output=True, text=True).stdout
        assert "getenv" not in out, o


def test_status_strings(lib):
    assert lib.dc_status_string(0) == b"DC_OK"
    assert lib.dc_status_string(4) == b"DC_ERR_ALIASING"
    assert lib.dc_status_string(99) == b"DC_ERR_UNKNOWN"
    assert lib.dc_version() == 100


def test_host_constants(lib):
    import math
    assert abs(lib.dc_k2_per_tec() - 40.308193022) < 1e-8          # Eq. 1, CODATA 2018
    assert lib.dc_alpha_from_velocity(0.0) == 1.0
    assert abs(lib.dc_alpha_from_velocity(5000.0) - 1 - 3.33569658541e-5) < 1e-14
    assert abs(lib.dc_alpha_from_velocity(-7e3) * lib.dc_alpha_from_velocity(7e3) - 1) < 1e-15
    assert math.isnan(lib.dc_alpha_from_velocity(3e8))
    assert math.isnan(lib.dc_alpha_from_velocity(float("inf")))


@pytest.mark.parametrize("n,fs,fc,taps,what", [
    (3, 1e6, 0.0, 4, "n = 3"),
    (0, 1e6, 0.0, 4, "n = 0"),
    (1, 1e6, 0.0, 2, "n = 1"),
    ((1 << 24) * 2, 1e6, 0.0, 4, "n = 2^25"),
    (1024, 0.0, 0.0, 4, "fs"),
    (1024, float("nan"), 0.0, 4, "fs"),
    (1024, 1e6, -1.0, 4, "fc"),
    (1024, 1e6, float("inf"), 4, "fc"),
    (1024, 1e6, 0.0, 1, "taps"),
    (1024, 1e6, 0.0, 129, "taps"),
    (4, 1e6, 0.0, 8, "taps"),
])
def test_plan_validation_rejects_before_touching_cuda(lib, n, fs, fc, taps, what):
    h = ctypes.c_void_p(123)
    st = lib.dc_plan(ctypes.byref(h), n, fs, fc, taps, 0, None)
    assert st == 1, (what, st)                      # DC_ERR_INVALID_VALUE
    assert h.value is None
    assert lib.dc_last_error_message()


def test_null_pointers(lib):
    assert lib.dc_plan(None, 1024, 1e6, 0.0, 8, 0, None) == 2
    assert lib.dc_plan_destroy(None) == 2
    assert lib.dc_iono(None, None, 1, None) == 2
    assert lib.dc_sync(None) == 2


def test_binding_fails_loudly_without_library(monkeypatch, tmp_path):
    import importlib
    import paper_2508_04951_b200 as dc
    monkeypatch.setattr(dc, "_LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(dc, "_lib", None)
    with pytest.raises(ImportError):
        dc.load()


def test_product_does_not_import_oracle():
    # the product package and the C sources must not reference oracle/ (independence)
    pkg = os.path.join(ROOT, "paper_2508_04951_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.c" not in txt, f
