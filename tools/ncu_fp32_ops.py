"""Counter-based FP32 roofline of each kernel in an ncu report: executed SASS instructions per opcode (the
source page of the capture) -> FP32 lane-operations per sample (FFMA2/FADD2/FMUL2 count twice, FFMA/FADD/FMUL
once) -> the FMA-pipe ceiling in samples/s (148 SMs x 128 lanes x clock / lane-ops per sample).
    python tools/ncu_fp32_ops.py REPORT SAMPLES_PER_LAUNCH [CLOCK_GHZ]  -> JSON on stdout"""
import csv
import json
import subprocess
import sys
from collections import defaultdict

rep, spl = sys.argv[1], int(sys.argv[2])
clk = float(sys.argv[3]) if len(sys.argv) > 3 else 1.965
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
hdr = raw[0]
names = []
tunit = raw[1][hdr.index("gpu__time_duration.sum")]
tscale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(tunit.strip(), 1.0)
for r in raw[2:]:
    nm = r[hdr.index("Kernel Name")]
    names.append((nm[:nm.index("(")] if "(" in nm else nm, float(r[hdr.index("gpu__time_duration.sum")]) * tscale,
                  float(r[hdr.index("smsp__inst_executed.sum")])))
LANES = {"FFMA2": 2, "FADD2": 2, "FMUL2": 2, "FFMA": 1, "FADD": 1, "FMUL": 1}
out = {}
for i, (nm, us, winst) in enumerate(names):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(i), "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    h = None
    ops = defaultdict(float)
    tot_warp = 0.0
    for r in rows:
        if "Address" in r and "Source" in r:
            h = r
            continue
        if not h or len(r) != len(h):
            continue
        d = dict(zip(h, r))
        op = d["Source"].strip().split()
        if not op:
            continue
        mnem = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        base = mnem.split(".")[0]
        thr = d.get("Thread Instructions Executed") or "0"
        try:
            ops[base] += float(thr.replace(",", ""))
            tot_warp += float((d.get("Instructions Executed") or "0").replace(",", ""))
        except ValueError:
            pass
    # the source page aggregates every captured launch of functions sharing a base name (warp_col3_kernel<0>
    # and <1>): take this launch's share of their executed instructions (same opcode mix assumed)
    base_nm = nm.split("<")[0]
    same = [w for (n2, _, w) in names if n2.split("<")[0] == base_nm]
    scale = winst / sum(same) if len(same) > 1 else 1.0
    lane_ops = scale * sum(ops[k] * v for k, v in LANES.items())
    per = lane_ops / spl if spl else 0.0
    key = f"{i}:{nm}"
    out[key] = {"us": round(us, 2), "fp32_lane_ops_per_sample": round(per, 2), "source_page_scale": round(scale, 3),
                "ffma2_share": round(2 * ops["FFMA2"] / lane_ops, 3) if lane_ops else 0,
                "fma_pipe_ceiling_gsps": round(148 * 128 * clk / per, 1) if per else None,
                "achieved_gsps_under_ncu": round(spl / us / 1e3, 1)}
stage = [v for k, v in out.items() if "doppler" not in k]
if stage:
    per = sum(v["fp32_lane_ops_per_sample"] for v in stage)
    out["fft_stage"] = {"fp32_lane_ops_per_sample": round(per, 2), "fma_pipe_ceiling_gsps": round(148 * 128 * clk / per, 1)}
print(json.dumps(out, indent=1))
