"""Device-timed dc_doppler throughput at n = 2^20 for W = 8 / 16 / 25 / 32 (tuning; best of 3 x 5 calls).
    python tools/tune/kbench_doppler_w.py [lib.so]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_04951_b200 as dc  # noqa: E402
import synth  # noqa: E402

if len(sys.argv) > 1:
    dc.use_library(sys.argv[1])
out = {"lib": os.path.basename(dc.library_path())}
n, batch = 1 << 20, 256
x = torch.from_numpy(synth.complex_gaussian(n, seed=1, batch=4).astype(np.complex64)).cuda().repeat(batch // 4, 1)
y = torch.empty_like(x)
_, alpha = synth.pulse_params(batch, seed=2)
for W in (8, 16, 25, 32):
    p = dc.Plan(n, 2.048e9, 0.0, taps=W, stream=torch.cuda.current_stream())
    p.doppler(x, y, alpha)
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            p.doppler(x, y, alpha)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 5)
    out[f"w{W}"] = round(batch * n / best / 1e6, 1)
    p.close()
print(json.dumps(out))
