"""Run the Doppler-bearing paths of a DC_DEBUG_CHECKS build of libdispcorr (device-side bounds traps on every
shared-memory window the Doppler tile code reads, and on every staged span against its buffer) over the
configurations the product dispatches, and compare sampled outputs with the FP64 oracle.
    python tools/debug_checks_driver.py LIB.so    -> prints 'debug checks done' (a trap is a CUDA error)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_04951_b200 as dc  # noqa: E402
import synth  # noqa: E402
from oracle import oracle as O  # noqa: E402

dc.use_library(sys.argv[1])
# first-order edge, second order, alpha < 1 and > 1, alpha = 1
ALPHAS = [1 + 7.0e-5, 1 - 7.1e-5, 1 + 2.5e-4, 1 - 2.0e-4, 1.0]
worst = 0.0
for log2n in (10, 11, 12, 13, 14, 16, 20):
    n = 1 << log2n
    x = synth.complex_gaussian(n, seed=log2n, batch=len(ALPHAS)).astype(np.complex64)
    tec = np.linspace(0.0, 2e18, len(ALPHAS))
    for W in (16, 32):
        for fs, fc in ((2.048e9, 0.0), (51.2e6, 422e6)):
            p = dc.Plan(n, fs, fc, taps=W)
            xd = torch.from_numpy(x).cuda()
            yd = torch.empty_like(xd)
            for i, a in enumerate(ALPHAS):  # one call per alpha: each takes its own path (first / second order)
                p.correct(xd[i:i + 1], yd[i:i + 1], tec[i:i + 1], [a])
                p.doppler(xd[i:i + 1], yd[i:i + 1], [a])
            torch.cuda.synchronize()
            idx = np.r_[0:64, n // 2 - 32:n // 2 + 32, n - 64:n]
            for i, a in enumerate(ALPHAS):
                ref = O.doppler_at(x[i], W, fs, fc, a, idx)
                got = yd[i].cpu().numpy()[idx]
                worst = max(worst, float(np.linalg.norm(got - ref) / np.linalg.norm(ref)))
            p.close()
assert worst < 1e-5, worst
print("debug checks done: worst sampled rel-L2", worst, flush=True)
