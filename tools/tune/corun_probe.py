"""Feasibility probe (tuning, not a benchmark of record): does a memory-bound kernel co-run with the
FP32-bound Doppler kernel on the same SMs?  Times dc_doppler alone, a 2 GiB torch copy alone, and the
two launched concurrently on two streams (max of both, CUDA events).
    python tools/tune/corun_probe.py [lib.so]"""
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
n, batch = 1 << 20, 64
x = torch.from_numpy(synth.complex_gaussian(n, seed=1, batch=4).astype(np.complex64)).cuda().repeat(batch // 4, 1)
y = torch.empty_like(x)
_, alpha = synth.pulse_params(batch, seed=2)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
p = dc.Plan(n, 2.048e9, 0.0, taps=32, stream=s1)
a = torch.empty(1 << 27, dtype=torch.complex64, device="cuda")
b = torch.empty_like(a)


def timed(do_d, do_c, reps=5):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    ev[0].record()
    s1.wait_event(ev[0])
    s2.wait_event(ev[0])
    for _ in range(reps):
        if do_d:
            p.doppler(x, y, alpha)
        if do_c:
            with torch.cuda.stream(s2):
                b.copy_(a)
    ev[1].record(s1)
    ev[2].record(s2)
    torch.cuda.synchronize()
    return max(ev[0].elapsed_time(ev[1]) if do_d else 0, ev[0].elapsed_time(ev[2]) if do_c else 0) / reps


timed(True, True)
out = {"lib": os.path.basename(dc.library_path()), "doppler_ms": timed(True, False), "copy_ms": timed(False, True),
       "both_ms": timed(True, True)}
out["doppler_gsps"] = batch * n / out["doppler_ms"] / 1e6
out["copy_gbs"] = 2 * a.numel() * 8 / out["copy_ms"] / 1e6
print(json.dumps(out))
