"""Device-timed dc_iono / dc_correct throughput of one library build (tuning; not the benchmark of record).
    python tools/tune/kbench_iono.py [lib.so]   -> one JSON line (G samples/s)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_04951_b200 as dc  # noqa: E402
import synth  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):
    dc.use_library(sys.argv[1])
out = {"lib": os.path.basename(dc.library_path())}


def rate(log2n, total_log2=28, reps=5, what="iono"):
    n = 1 << log2n
    batch = max(1, (1 << total_log2) >> log2n)
    x = torch.from_numpy(synth.complex_gaussian(n, seed=1, batch=min(batch, 4)).astype(np.complex64)).cuda()
    x = x.repeat((batch + 3) // 4, 1)[:batch].contiguous()
    y = torch.empty_like(x)
    tec, alpha = synth.pulse_params(batch, seed=2)
    p = dc.Plan(n, 2.048e9, 0.0, taps=32, stream=torch.cuda.current_stream())
    f = (lambda: p.iono(x, tec)) if what == "iono" else (lambda: p.correct(x, y, tec, alpha))
    f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    p.profile_enable(True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    prof = p.profile_read()
    ms = e0.elapsed_time(e1) / reps
    p.close()
    kern = {k: round(v["samples"] / v["ms"] / 1e6, 1) for k, v in prof.items() if v["launches"]}
    return {"gsps": round(batch * n / ms / 1e6, 1), "kernels": kern}


for l in [int(a) for a in os.environ.get("KB_IONO_N", "8,10,12,13,14,16,18,20,22,24").split(",")]:
    out[f"iono_2e{l}"] = rate(l)
out["correct_2e20"] = rate(20, what="correct")
for l in (10, 11, 12, 13, 14):  # the fused single-round-trip dc_correct (n = 2^10 .. 2^14, W = 32)
    out[f"correct_2e{l}"] = rate(l, what="correct")
print(json.dumps(out), flush=True)
