import sys
sys.path.insert(0, '.')
import numpy as np, torch, synth
import paper_2508_04951_b200 as dc
log2n = int(sys.argv[1]); pulses = int(sys.argv[2])
n = 1 << log2n
x = torch.from_numpy(synth.complex_gaussian(n, seed=1, batch=pulses).astype(np.complex64)).cuda()
tec, alpha = synth.pulse_params(pulses)
p = dc.Plan(n, 2.048e9, 0.0, taps=32)
for _ in range(3):
    p.iono(x, tec)
p.sync(); print("ok")
