"""Doppler-stage throughput with and without the Kaiser taper (n = 2^20 x 128 pulses, W = 32)."""
import sys, json
sys.path.insert(0, '.')
import numpy as np, torch
import synth
import paper_2508_04951_b200 as dc
n, batch = 1 << 20, 128
x = torch.from_numpy(synth.waveform_bank(n, count=4)[np.arange(batch) % 4]).cuda()
y = torch.empty_like(x)
_, alpha = synth.pulse_params(batch)
out = {}
for W in (16, 32, 64):
    for kb in (0.0, 8.0):
        p = dc.Plan(n, 2.048e9, 0.0, taps=W)
        p.set_taper(kb)
        for _ in range(3):
            p.doppler(x, y, alpha)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            p.doppler(x, y, alpha)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        out[f"W{W}_kaiser{kb:g}"] = round(batch * n / ms / 1e6, 1)
        p.close()
print(json.dumps({"doppler_GS_per_s": out}))
