"""Small dc_doppler driver for ncu captures: `pulses` x 2^log2n, W taps, C4-style alphas."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_04951_b200 as dc  # noqa: E402
import synth  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
pulses = int(sys.argv[2]) if len(sys.argv) > 2 else 64
W = int(sys.argv[3]) if len(sys.argv) > 3 else 32
if len(sys.argv) > 4:
    dc.use_library(sys.argv[4])
n = 1 << log2n
x = torch.from_numpy(synth.complex_gaussian(n, seed=1, batch=4).astype(np.complex64)).cuda()
x = x.repeat(pulses // 4, 1).contiguous()
y = torch.empty_like(x)
_, alpha = synth.pulse_params(pulses, seed=2)
p = dc.Plan(n, 2.048e9, 0.0, taps=W)
for _ in range(2):
    p.doppler(x, y, alpha)
p.sync()
print("ok", p.info()["kernel_launches"])
