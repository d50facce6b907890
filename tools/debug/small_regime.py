"""Debug driver: small-regime iono parity per log2n (prints rel-L2), optional subset via argv."""
import sys
import numpy as np
sys.path.insert(0, '.')
import torch
import synth
from oracle import oracle as O
import paper_2508_04951_b200 as dc

ps = [int(a) for a in sys.argv[1:]] or list(range(1, 14))
for P in ps:
    n = 1 << P
    batch = 3 if n >= 1024 else 37
    x = synth.complex_gaussian(n, seed=P, batch=batch).astype(np.complex64)
    tec = np.linspace(0, 2e18, batch)
    for fs, fc in ((2.048e9, 0.0), (51.2e6, 422e6)):
        p = dc.Plan(n, fs, fc, taps=min(8, n))
        t = torch.from_numpy(x).cuda()
        p.iono(t, tec)
        p.sync()
        y = t.cpu().numpy()
        ref = O.run_batch("iono", x, fs, fc, 8, tec)
        err = np.linalg.norm(y - ref, axis=1) / np.linalg.norm(ref, axis=1)
        print(P, fs, fc, "max rel-L2", err.max(), "argmax", err.argmax(), flush=True)
        p.close()
