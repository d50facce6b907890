"""Small dc_correct driver for ncu captures of the short-pulse fused kernels:
    python tools/correct_driver.py LOG2N PULSES [W]"""
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_04951_b200 as dc  # noqa: E402
import synth  # noqa: E402

log2n, pulses = int(sys.argv[1]), int(sys.argv[2])
W = int(sys.argv[3]) if len(sys.argv) > 3 else 32
n = 1 << log2n
x = torch.from_numpy(synth.complex_gaussian(n, seed=1, batch=pulses).astype(np.complex64)).cuda()
y = torch.empty_like(x)
tec, alpha = synth.pulse_params(pulses)
p = dc.Plan(n, 2.048e9, 0.0, taps=W)
for _ in range(3):
    p.correct(x, y, tec, alpha)
p.sync()
print("ok", p.info())
