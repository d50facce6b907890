import sys, os, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2508_04951_b200 as dc, synth
dc.use_library(sys.argv[1])
out = {"lib": os.path.basename(sys.argv[1])}
for W in (16, 32):
    for l in (12, 13, 14, 15):
        n = 1 << l; batch = (1 << 28) // n
        x = torch.from_numpy(synth.complex_gaussian(n, seed=1, batch=4).astype(np.complex64)).cuda().repeat(batch // 4, 1)
        y = torch.empty_like(x); _, alpha = synth.pulse_params(batch, seed=2)
        p = dc.Plan(n, 2.048e9, 0.0, taps=W, stream=torch.cuda.current_stream())
        p.doppler(x, y, alpha)
        best = 1e9
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            for _ in range(5): p.doppler(x, y, alpha)
            e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1) / 5)
        out[f"w{W}_2e{l}"] = round(batch * n / best / 1e6, 1)
        p.close(); del x, y
print(json.dumps(out))
