"""One small launch of every libdispcorr kernel, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  Run:  compute-sanitizer --tool memcheck python tools/sanitize_driver.py
Kernels exercised (by plan regime / path): warp_tiny (n = 128 .. 512), tile_fft, warp_row SMALL (n = 1024), warp_small
(n = 4096), thread_col + warp_row ROWB (n = 2^14), warp_col3 + warp_row ROWB (n = 2^20), warp_col3 +
tile_fft ROWB (n = 2^22), tile_fft for all passes (n = 2^24), doppler_pipe (first / second order,
Kaiser), doppler_exact, expand_params (batch > 4096), pulse compression (reference + compress),
the host pipeline."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_04951_b200 as dc  # noqa: E402
import synth  # noqa: E402

FS = 2.048e9
only = sys.argv[1:]


def want(name):
    return not only or name in only


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex64)).cuda()


def run_correct(n, batch, W=32, alphas=None, kaiser=0.0, fc=0.0):
    x = dev(synth.complex_gaussian(n, seed=n % 97, batch=batch))
    tec, alpha = synth.pulse_params(batch, seed=3)
    if alphas is not None:
        alpha = np.resize(np.asarray(alphas, float), batch)
    p = dc.Plan(n, FS, fc, taps=min(W, n))
    if kaiser:
        p.set_taper(kaiser)
    y = torch.empty_like(x)
    p.correct(x, y, tec, alpha)
    p.sync()
    return p


for log2n, batch in ((7, 9), (8, 3), (9, 5), (10, 3), (12, 3), (14, 2), (20, 1), (22, 1), (24, 1)):
    if want(f"iono{log2n}"):
        run_correct(1 << log2n, batch)
if want("doppler"):
    run_correct(1 << 14, 2, alphas=[1 + 3e-5, 1 - 3e-5])           # first-order pipe
    run_correct(1 << 14, 2, alphas=[1 + 4e-4, 1 - 4e-4])           # second-order pipe
    run_correct(1 << 14, 2, alphas=[1.05, 0.93])                   # exact kernel
    run_correct(1 << 14, 2, alphas=[1 + 3e-5, 1.0], kaiser=8.0)    # tapered pipe
    run_correct(4096, 2, W=25, alphas=[1 + 3e-5, 1 - 1e-5], fc=422e6)  # runtime-W path? (25 is compiled) + carrier
    run_correct(4096, 2, W=7, alphas=[1 + 3e-5, 1 - 1e-5])         # runtime W
if want("expand"):
    run_correct(256, 4100, W=16)                                   # device-side parameter expansion
if want("compress"):
    for n in (1024, 1 << 16):
        p = dc.Plan(n, 51.2e6, 422e6, taps=8)
        p.set_reference(dev(synth.complex_gaussian(n // 4, seed=5)))
        x = dev(synth.complex_gaussian(n, seed=6, batch=2))
        z = torch.empty_like(x)
        p.compress(x, z, [1e17, 2e17])
        p.compress(x, x, [1e17, 2e17])
        p.sync()
if want("fused"):
    run_correct(1 << 12, 5, W=32)                                  # fused single-round-trip dc_correct
    run_correct(1 << 10, 7, W=32)                                  # fused, warp-level FFT (n = 1024)
    run_correct(1 << 13, 2, W=16, alphas=[1 + 4e-4, 1 - 4e-4], fc=422e6)
if want("pq"):
    for n in (256, 1 << 14, 1 << 20):                              # tile / four-step regimes of n and 2n
        p = dc.Plan(n, FS, 422e6 if n == 256 else 0.0, taps=8)
        x = dev(synth.complex_gaussian(n, seed=12, batch=3))
        y = torch.empty_like(x)
        p.doppler_pq(x, y, [(n + 2.3) / n, 1.0, (n - 4.2) / n])     # M = n + 2, identity, M = n - 4
        p.sync()
if want("host"):
    n = 1 << 14
    p = dc.Plan(n, FS, 0.0, taps=32)
    # pageable numpy buffers: host writes into pinned memory are invisible to initcheck
    xh = synth.complex_gaussian(n, seed=9, batch=3).astype(np.complex64)
    yh = np.empty_like(xh)
    tec, alpha = synth.pulse_params(3, seed=9)
    p.correct_host(xh, yh, tec, alpha)
torch.cuda.synchronize()
print("sanitize driver done")
