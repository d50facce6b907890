"""dc_iono driver for ncu captures: `batch` pulses of 2^log2n samples, `reps` calls."""
import sys
import numpy as np
sys.path.insert(0, '.')
import torch
import synth
import paper_2508_04951_b200 as dc

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
n = 1 << log2n
x = torch.from_numpy(synth.complex_gaussian(n, seed=1).astype(np.complex64)).cuda().expand(batch, n).contiguous()
tec = 1e16 * (np.arange(batch) % 200).astype(np.float64)
p = dc.Plan(n, 2.048e9, 0.0, taps=8)
for _ in range(reps):
    p.iono(x, tec)
p.sync()
print("ok", p.info())
