for v in splitwide; do
 DISPCORR_LIB=paper_2508_04951_b200/lib/variants/libdispcorr_$v.so timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch, synth, paper_2508_04951_b200 as dc
from oracle import oracle as O
for log2n in (21, 22):
    n = 1 << log2n; b = (1 << 27) // n
    x = torch.from_numpy(synth.complex_gaussian(n, seed=1).astype(np.complex64)).cuda().expand(b, n).contiguous()
    x0 = x[:1].cpu().numpy()
    tec = 1e16 * (np.arange(b) % 200).astype(np.float64)
    p = dc.Plan(n, 2.048e9, 0.0, taps=8)
    xs = x.clone(); p.iono(xs, tec); torch.cuda.synchronize()
    ref = O.run_batch('iono', x0, 2.048e9, 0.0, 8, tec[:1])
    err = np.linalg.norm(xs[:1].cpu().numpy() - ref) / np.linalg.norm(ref)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2): p.iono(xs, tec)
    e0.record()
    for _ in range(5): p.iono(xs, tec)
    e1.record(); torch.cuda.synchronize()
    print(log2n, 'GS/s', round(b * n * 5 / e0.elapsed_time(e1) / 1e6, 1), 'relL2', err)
"
done > gpurun_out/s42.log 2>&1
