"""Per-kernel-class timing of dc_correct for the library named by DISPCORR_LIB."""
import os, sys, json
sys.path.insert(0, '.')
import numpy as np, torch
import synth
import paper_2508_04951_b200 as dc
log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
pulses = int(sys.argv[2]) if len(sys.argv) > 2 else 96
n = 1 << log2n
bank = synth.waveform_bank(n, count=4, T=min(100e-6, 0.4 * n / 2.048e9))
x = torch.from_numpy(bank[np.arange(pulses) % 4]).cuda()
y = torch.empty_like(x)
tec, alpha = synth.pulse_params(pulses)
p = dc.Plan(n, 2.048e9, 0.0, taps=32)
for _ in range(2):
    p.correct(x, y, tec, alpha)
p.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); p.correct(x, y, tec, alpha); p.correct(x, y, tec, alpha); e1.record(); torch.cuda.synchronize()
tot = e0.elapsed_time(e1) / 2
p.profile_enable(True)
p.correct(x, y, tec, alpha)
pr = p.profile_read()
out = {"lib": os.path.basename(dc.library_path()), "fused_env": os.environ.get("DISPCORR_FUSED", "1"), "pg": os.environ.get("DISPCORR_FUSED_PG"), "depth": os.environ.get("DISPCORR_FUSED_DEPTH"), "log2n": log2n, "pulses": pulses, "ms_per_call": tot,
       "GS/s": pulses * n / tot / 1e6}
for k, v in pr.items():
    if v["launches"]:
        out[k] = round(v["samples"] / (v["ms"] / 1e3) / 1e9, 1)
print(json.dumps(out))
