"""Device-side bounds checks in lieu of compute-sanitizer (disabled on this GPU pool): a build of libdispcorr
with -DDC_DEBUG_CHECKS traps if any Doppler tile reads outside its staged / resident shared-memory span or
stages a span larger than its buffer; tools/debug_checks_driver.py runs the fused and two-kernel dc_correct
and dc_doppler paths (n = 2^10 .. 2^20, W = 16 / 32, first-order edge, second order, alpha = 1, fc = 0 and a
baseband carrier) on that build and checks sampled outputs against the oracle."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_debug_bounds_checks_clean():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_04951_b200 import build
    build.build()
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "tune", "build_variants.py"),
                        "doppler_kernel.cu+iono_small.cu", "dbgchk:-DDC_DEBUG_CHECKS"], cwd=ROOT, capture_output=True,
                       text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    lib = os.path.join(build.LIB_DIR, "variants", "dbgchk.so")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "debug_checks_driver.py"), lib], cwd=ROOT,
                       capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "debug checks done" in out, out[-3000:]
