"""Run one small dc_doppler call (W from argv) and compare with the oracle."""
import sys
import numpy as np
sys.path.insert(0, '.')
import torch
import synth
from oracle import oracle as O
import paper_2508_04951_b200 as dc
W = int(sys.argv[1]) if len(sys.argv) > 1 else 32
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
alphas = np.array([1 + 3.3e-5, 1 - 3.3e-5, 1 + 1e-5])
x = synth.complex_gaussian(n, seed=W, batch=len(alphas)).astype(np.complex64)
p = dc.Plan(n, 2.048e9, 0.0, taps=W)
t = torch.from_numpy(x).cuda()
y = torch.empty_like(t)
p.doppler(t, y, alphas)
p.sync()
ref = O.run_batch("doppler", x, 2.048e9, 0.0, W, None, alphas)
err = np.linalg.norm(y.cpu().numpy() - ref, axis=1) / np.linalg.norm(ref, axis=1)
print("W", W, "rel-L2", err)
