"""Small dc_correct driver for ncu captures: C4-style pulses (2^20, W=32), `pulses` per call."""
import sys
import numpy as np
sys.path.insert(0, '.')
import torch
import synth
import paper_2508_04951_b200 as dc

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
pulses = int(sys.argv[2]) if len(sys.argv) > 2 else 12
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
n = 1 << log2n
bank = synth.waveform_bank(n, count=4, T=min(100e-6, 0.4 * n / 2.048e9))
x = torch.from_numpy(bank[np.arange(pulses) % 4]).cuda()
y = torch.empty_like(x)
tec, alpha = synth.pulse_params(pulses)
p = dc.Plan(n, 2.048e9, 0.0, taps=32)
for _ in range(reps):
    p.correct(x, y, tec, alpha)
p.sync()
print("ok", p.info())
