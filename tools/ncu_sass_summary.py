"""Summarise an ncu --page source --csv (SASS) export: executed warp-instructions and stall
samples per opcode, plus the hottest instructions.  Usage: ncu -i rep --page source --csv
--kernel-name regex:K | python tools/ncu_sass_summary.py"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(sys.stdin))
hdr = None
data = []
for r in rows:
    if "Address" in r and "Source" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
ops = defaultdict(lambda: [0, 0])
tot_i = tot_s = 0
for d in data:
    src = d["Source"].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    try:
        ie = int(float(d["Instructions Executed"] or 0))
        ss = int(float(d["Warp Stall Sampling (All Samples)"] or 0))
    except ValueError:
        continue
    ops[op][0] += ie
    ops[op][1] += ss
    tot_i += ie
    tot_s += ss
print(f"total warp-instructions {tot_i}, stall samples {tot_s}")
for op, (i, s) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{op:10s} inst {i:12d} ({100*i/max(tot_i,1):5.1f}%)  stall {100*s/max(tot_s,1):5.1f}%")
hot = sorted(data, key=lambda d: -float(d["Warp Stall Sampling (All Samples)"] or 0))[:15]
print("hottest (stall samples):")
for d in hot:
    print(f"  {d['Address']} {d['Source'][:60]:60s} stall {d['Warp Stall Sampling (All Samples)']} inst {d['Instructions Executed']}")
