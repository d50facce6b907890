"""dc_iono / dc_correct throughput vs launch-group size (tuning): C2 (256 x 2^16), 2^16 x 4096, 2^20 x 256.
    python tools/tune/kbench_groups.py lib.so"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_04951_b200 as dc  # noqa: E402
import synth  # noqa: E402

dc.use_library(sys.argv[1])
out = {"lib": os.path.basename(sys.argv[1])}
for log2n, batch, what in ((16, 256, "iono"), (16, 4096, "iono"), (20, 256, "correct"), (16, 256, "correct")):
    n = 1 << log2n
    x = torch.from_numpy(synth.complex_gaussian(n, seed=1, batch=4).astype(np.complex64)).cuda().repeat(batch // 4, 1)
    y = torch.empty_like(x)
    tec, alpha = synth.pulse_params(batch, seed=2)
    p = dc.Plan(n, 2.048e9, 0.0, taps=32, stream=torch.cuda.current_stream())
    f = (lambda: p.iono(x, tec)) if what == "iono" else (lambda: p.correct(x, y, tec, alpha))
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    out[f"{what}_2e{log2n}x{batch}"] = round(batch * n * 20 / e0.elapsed_time(e1) / 1e6, 1)
    p.close()
print(json.dumps(out), flush=True)
