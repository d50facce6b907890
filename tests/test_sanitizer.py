"""compute-sanitizer tier (tier 4): memcheck, racecheck, synccheck and initcheck over one small
launch of every libdispcorr kernel (tools/sanitize_driver.py) must report zero errors.  The kernels
rely on TMA + transaction mbarriers, full/empty mbarrier pipelines, bulk async stores, cp.async and
warp-private shared-memory exchanges; racecheck / synccheck check those hazards."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COMPONENTS = ["iono7", "iono8", "iono9", "iono10", "iono12", "iono14", "iono20", "iono22", "iono24", "doppler", "expand", "compress",
              "fused", "pq", "host"]


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_compute_sanitizer_clean(tool):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not installed")
    from paper_2508_04951_b200 import build
    build.build()
    # initcheck does not track writes made by the bulk-async (TMA) copy engine: every sample the Doppler
    # kernel stores with cp.async.bulk reads back as "uninitialized" (measured: the host-path D2H of 3 x 2^14
    # outputs gives exactly 3 * 2^14 * 8 / 32 = 12288 flagged sectors).  The driver's other components
    # never read a TMA-written buffer back through the runtime; the host pipeline runs under the other
    # three tools.
    comps = [c for c in COMPONENTS if not (tool == "initcheck" and c == "host")]
    r = subprocess.run([exe, "--tool", tool, "--print-limit", "10", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_driver.py"), *comps], cwd=ROOT, capture_output=True,
                       text=True, timeout=1200)
    out = r.stdout + r.stderr
    if "closed on this pool" in out:
        # the GPU pool disabled compute-sanitizer in round 2 (runs under it left GPUs needing a reset); the
        # clean logs of the earlier runs are kept in profiles/ (r2_sanitizer_fused.log, r2b_initcheck_components.log)
        pytest.skip("compute-sanitizer is disabled on this GPU pool: " + out.strip().splitlines()[0][:200])
    assert "sanitize driver done" in out, out[-3000:]
    summary = [ln for ln in out.splitlines() if "ERROR SUMMARY" in ln or "RACECHECK SUMMARY" in ln]
    assert summary, out[-3000:]
    m = re.search(r"(\d+) errors", summary[-1])
    assert m and int(m.group(1)) == 0, "\n".join(summary) + "\n" + out[-3000:]
