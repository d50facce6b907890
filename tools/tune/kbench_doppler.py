"""Device-timed dc_doppler throughput of one library build (tuning; not the benchmark of record).
    python tools/tune/kbench_doppler.py [lib.so]   -> one JSON line"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_04951_b200 as dc  # noqa: E402
import synth  # noqa: E402

if len(sys.argv) > 1:
    dc.use_library(sys.argv[1])
out = {"lib": os.path.basename(dc.library_path())}


def rate(n, batch, W, reps=5, kaiser=0.0, check=None):
    x = torch.from_numpy(synth.complex_gaussian(n, seed=1, batch=min(batch, 4)).astype(np.complex64)).cuda()
    x = x.repeat((batch + 3) // 4, 1)[:batch].contiguous()
    y = torch.empty_like(x)
    _, alpha = synth.pulse_params(batch, seed=2)
    p = dc.Plan(n, 2.048e9, 0.0, taps=W, stream=torch.cuda.current_stream())
    if kaiser:
        p.set_taper(kaiser)
    p.doppler(x, y, alpha)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        p.doppler(x, y, alpha)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    if check is not None:
        from oracle import oracle as O
        idx = np.arange(0, n, max(1, n // 4096))
        ref = O.doppler_at(x[0].cpu().numpy(), W, 2.048e9, 0.0, alpha[0], idx, kaiser=kaiser)
        ys = y[0, torch.from_numpy(idx).cuda()].cpu().numpy()
        out[check] = float(np.linalg.norm(ys - ref) / np.linalg.norm(ref))
    p.close()
    return round(batch * n / ms / 1e6, 1)  # G samples/s


out["w32_2e20"] = rate(1 << 20, 256, 32, check="err_w32")
out["w64_2e20"] = rate(1 << 20, 128, 64, check="err_w64")
out["w128_2e20"] = rate(1 << 20, 128, 128, check="err_w128")
out["w16_2e20"] = rate(1 << 20, 256, 16)
out["w32_4096"] = rate(4096, 65536, 32)
out["w32_2e24"] = rate(1 << 24, 16, 32)
out["w32_k8"] = rate(1 << 20, 128, 32, kaiser=8.0, check="err_k8")
print(json.dumps(out), flush=True)
