"""One process of the two-processes-on-one-GPU diagnostic: dc_correct on a 512-pulse C4 shard, `reps` calls.
    python tools/debug/one_proc.py rank [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_04951_b200 as dc  # noqa: E402
import synth  # noqa: E402

rank = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
n, pulses = 1 << 20, 512
bank = synth.waveform_bank(n, count=16)
x = torch.from_numpy(bank[(np.arange(pulses) + pulses * rank) % 16]).cuda()
y = torch.empty_like(x)
tec, alpha = synth.pulse_params(2 * pulses)
tec, alpha = tec[pulses * rank:pulses * (rank + 1)].copy(), alpha[pulses * rank:pulses * (rank + 1)].copy()
p = dc.Plan(n, 2.048e9, 0.0, taps=32, stream=torch.cuda.current_stream())
for _ in range(reps):
    p.correct(x, y, tec, alpha)
torch.cuda.synchronize()
print("rank", rank, "ok", flush=True)
